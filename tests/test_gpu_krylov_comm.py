"""GPU tier: the FGMRES orthogonalization options and the library's own NCCL
communicator.

* CGS2 (classical Gram-Schmidt twice, two batched all-reduces per iteration)
  against the reference's MGS (solver.cpp:146-152): the same Krylov space, so
  iteration counts within +-1 and solutions within the solve tolerance of the
  oracle (relative L2 <= 1e-8), in 2D (time-marched gmres and the all-at-once
  solve), in 3D, with more than kMultiMax = 16 basis vectors (chunked batched
  passes), and over a 2-rank loopback partition (the batched all-reduce
  carries j+1 values per pass).
* stmg_comm_nccl_*: the C++ NCCL communicator at one rank (NCCL cannot pair
  two ranks on one GPU): the callbacks run NCCL on device memory, and an
  installed communicator leaves the solve unchanged.
"""
import ctypes
import threading

import numpy as np
import pytest
import torch

import oracle3_ctypes as o3
import oracle_ctypes as oc

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def consistent(lv, r_fine, seed, n):
    npc = (r_fine + 1) * (r_fine + 2) // 2
    v = oc.seeded(n * lv.size, seed)
    return oc.make_consistent(v, lv.n_slots, lv.n_scalar, lv.grid_x, lv.n_pressure, lv.n_pressure // npc, npc, n)


@pytest.mark.parametrize("c,r,k,kind,n_steps", [(3, 1, 1, 0, 8), (2, 2, 2, 0, 4), (3, 1, 1, 1, 4)])
def test_cgs2_all_at_once_matches_mgs_and_oracle(ctx, stmg, c, r, k, kind, n_steps):
    ref = oc.OracleSolver(c, r, k, n_steps=n_steps, nu=1.0, gamma=1.0, smoother=kind, nu1=2, nu2=2, rtol=1e-12)
    its = {}
    for ortho in (stmg.ORTHO_MGS, stmg.ORTHO_CGS2):
        sol = stmg.Solver(ctx, c, r, k, n_steps=n_steps, nu=1.0, gamma=1.0, smoother=kind, nu1=2, nu2=2,
                          rtol=1e-12)
        sol.set_krylov(ortho)
        F = consistent(sol.finest, r, 17, n_steps)
        X = torch.zeros(n_steps * sol.finest.size, dtype=torch.float64, device="cuda")
        its[ortho], _ = sol.solve_all_at_once(dev(F), X, n_steps)
        Xr, _, _ = ref.time_march(F)
        assert np.linalg.norm(host(X) - Xr) <= 1e-8 * np.linalg.norm(Xr)
    assert abs(its[stmg.ORTHO_MGS] - its[stmg.ORTHO_CGS2]) <= 1, its


def test_cgs2_gmres_beyond_one_batch(ctx, stmg):
    """A weak preconditioner (V(1,1), one smoothing sweep) and a tight
    tolerance run more than 16 Arnoldi steps: the batched passes chunk."""
    sol = stmg.Solver(ctx, 3, 1, 1, n_steps=4, nu=1.0, gamma=1.0, nu1=1, nu2=1, omega=0.5, rtol=1e-14, atol=0.0)
    rs = oc.OracleSolver(3, 1, 1, n_steps=4, nu=1.0, gamma=1.0, nu1=1, nu2=1, omega=0.5, rtol=1e-14, atol=0.0)
    lv = sol.finest
    b = consistent(lv, 1, 5, 1)
    xr, itr, _ = rs.gmres(b)
    for ortho in (stmg.ORTHO_MGS, stmg.ORTHO_CGS2):
        sol.set_krylov(ortho)
        x = torch.zeros(lv.size, dtype=torch.float64, device="cuda")
        it, _ = sol.gmres(dev(b), x)
        assert abs(it - itr) <= 1, (ortho, it, itr)
        assert np.linalg.norm(host(x) - xr) <= 1e-8 * np.linalg.norm(xr)
    assert itr > 16, itr  # the case must exercise more than one batch


def test_cgs2_3d(ctx, stmg):
    """3D all-at-once FGMRES: CGS2 vs MGS iterations +-1, both equal to the
    oracle's direct time march of the same system (<= 1e-8)."""
    nx, r, k, N = 4, 1, 1, 4
    ref = o3.OracleLevel3(nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, smoother=False)
    b = o3.make_consistent3(np.random.default_rng(9).uniform(-1, 1, N * ref.size), ref, N)
    xd = ref.direct_time_march(b, N)
    its = {}
    for ortho in (stmg.ORTHO_MGS, stmg.ORTHO_CGS2):
        S = stmg.Solver3(ctx, nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, n_hcoarse=2, time_coarsen=False, k_min=1,
                         rtol=1e-11)
        S.set_krylov(ortho)
        X = torch.zeros(N * ref.size, dtype=torch.float64, device="cuda")
        its[ortho], _ = S.solve_all_at_once(dev(b), X, N)
        assert np.linalg.norm(host(X) - xd) <= 1e-8 * np.linalg.norm(xd)
    assert abs(its[0] - its[1]) <= 1, its


def test_cgs2_loopback_partition(stmg):
    from paper_2502_09159_b200 import timeslab

    world, c, r, k, n_local = 2, 3, 1, 1, 2
    n_global = world * n_local
    tau = 1.0 / n_global
    ctx0 = stmg.Context(0)
    full = stmg.Solver(ctx0, c, r, k, n_steps=n_global, t_end=1.0, nu=1.0, gamma=1.0, nu1=2, nu2=2, rtol=1e-11)
    lv = full.finest
    F = dev(consistent(lv, r, 31, n_global))
    X1 = torch.zeros_like(F)
    it1, _ = full.solve_all_at_once(F, X1, n_global)
    torch.cuda.synchronize()
    hub = timeslab.LoopbackHub(world, timeout=120.0)
    Xp = torch.zeros_like(F)
    results, errors = {}, []
    m = n_local * lv.size

    def run(rank):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                sol = stmg.Solver(stmg.Context(0, stream=stream), c, r, k, n_steps=n_local, t_end=n_local * tau,
                                  nu=1.0, gamma=1.0, nu1=2, nu2=2, rtol=1e-11)
                sol.set_krylov(stmg.ORTHO_CGS2)
                sol.set_comm(timeslab.LoopbackComm(hub, rank))
                Fr = F[rank * m:(rank + 1) * m].clone()
                Xr = torch.zeros_like(Fr)
                stream.synchronize()
                it, _ = sol.solve_all_at_once(Fr, Xr, n_local)
                stream.synchronize()
                Xp[rank * m:(rank + 1) * m].copy_(Xr)
                stream.synchronize()
                results[rank] = it
        except BaseException as exc:
            errors.append(exc)
            hub.barrier.abort()

    threads = [threading.Thread(target=run, args=(q,)) for q in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(300)
    assert not errors, errors
    assert len(set(results.values())) == 1 and abs(results[0] - it1) <= 1, (results, it1)
    assert float((Xp - X1).norm() / X1.norm()) <= 1e-9


def test_nccl_comm_single_rank(ctx, stmg):
    uid = stmg.NcclComm.unique_id()
    assert len(uid) == 128
    comm = stmg.NcclComm(0, 1, 0, uid)
    ops = comm.ops()
    assert (ops.rank, ops.world) == (0, 1)
    stream = torch.cuda.Stream()
    buf = torch.arange(6, dtype=torch.float64, device="cuda")
    src = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64, device="cuda")
    out = torch.zeros(3, dtype=torch.float64, device="cuda")
    recv = torch.full((3,), -1.0, dtype=torch.float64, device="cuda")
    torch.cuda.synchronize()
    s = ctypes.c_void_p(stream.cuda_stream)
    assert ops.allreduce_sum(ops.user, buf.data_ptr(), 6, s) == 0
    assert ops.allgather(ops.user, src.data_ptr(), out.data_ptr(), 3, s) == 0
    assert ops.exchange_halo(ops.user, src.data_ptr(), recv.data_ptr(), 3, s) == 0
    stream.synchronize()
    assert torch.equal(buf, torch.arange(6, dtype=torch.float64, device="cuda"))
    assert torch.equal(out, src)
    assert bool((recv == -1.0).all())  # rank 0 of 1: nothing to receive
    sol = stmg.Solver(ctx, 3, 1, 1, n_steps=4, nu=1.0, nu1=2, nu2=2, rtol=1e-10)
    lv = sol.finest
    F = dev(consistent(lv, 1, 9, 4))
    X0 = torch.zeros_like(F)
    it0, _ = sol.solve_all_at_once(F, X0, 4)
    sol.set_comm(comm)
    sol.set_krylov(stmg.ORTHO_CGS2)
    X1 = torch.zeros_like(F)
    it1, _ = sol.solve_all_at_once(F, X1, 4)
    assert abs(it0 - it1) <= 1
    assert float((X1 - X0).norm() / X0.norm()) <= 1e-9
    S3 = stmg.Solver3(ctx, 2, 2, 2, 1, 1, 0.125, 1.0, 1.0, n_hcoarse=1, time_coarsen=False, k_min=1)
    S3.set_comm(comm)
    S3.set_comm(None)
    sol.set_comm(None)
