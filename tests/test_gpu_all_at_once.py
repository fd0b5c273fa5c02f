"""GPU tier: the all-at-once space-time solve (Eq. GloSys)
and its time-slab partition.

The reference only time-marches (solver.cpp:204-325), so the all-at-once
path is pinned by the identity SURVEY §8c names: the converged all-at-once
solution equals the time-marched solution of the same system (relative L2
<= 1e-8), here checked against the oracle's time marching. The time-slab
partition is checked on one GPU with in-process loopback ranks
(host-synchronised exchanges, no kernel waits on another rank) against the
unpartitioned solve."""
import threading

import numpy as np
import pytest
import torch

import oracle_ctypes as oc

pytestmark = pytest.mark.gpu

SOLVE_TOL = 1e-8


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def consistent(lv, r_fine, seed, n_intervals):
    npc = (r_fine + 1) * (r_fine + 2) // 2
    ncell = lv.n_pressure // npc
    v = oc.seeded(n_intervals * lv.size, seed)
    return oc.make_consistent(v, lv.n_slots, lv.n_scalar, lv.grid_x, lv.n_pressure, ncell, npc, n_intervals)


CASES = [
    # refinements, r, k, nu, gamma, smoother, nu1, nu2, n_steps
    (3, 1, 1, 1.0, 1.0, 0, 2, 2, 8),    # C1-like: Q2/P1, DG(1), V(2,2)
    (2, 2, 2, 0.1, 1.0, 0, 1, 1, 4),    # Q3/P2, DG(2): p_space + p_time levels
    (3, 1, 1, 1.0, 1.0, 1, 1, 1, 4),    # vertex-star Vanka
    (4, 1, 1, 1.0, 0.0, 0, 2, 2, 8),    # C1 discretisation, gamma = 0
]


@pytest.mark.parametrize("c,r,k,nu,gamma,kind,nu1,nu2,n_steps", CASES)
def test_all_at_once_equals_time_march(ctx, stmg, c, r, k, nu, gamma, kind, nu1, nu2, n_steps):
    sol = stmg.Solver(ctx, c, r, k, n_steps=n_steps, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2,
                      rtol=1e-12)
    ref = oc.OracleSolver(c, r, k, n_steps=n_steps, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2,
                          rtol=1e-12)
    F = consistent(sol.finest, r, 17, n_steps)
    X = torch.zeros(n_steps * sol.finest.size, dtype=torch.float64, device="cuda")
    it, hist = sol.solve_all_at_once(dev(F), X, n_steps)
    Xr, _, _ = ref.time_march(F)
    Xs = host(X)
    assert np.linalg.norm(Xs - Xr) <= SOLVE_TOL * np.linalg.norm(Xr)
    assert hist[-1] <= 1e-12 * hist[0] * (1 + 1e-9)
    err = np.linalg.norm(Xs - Xr) / np.linalg.norm(Xr)
    print(f"all-at-once iterations {it}, rel L2 vs oracle time march {err:.2e} "
          f"(c={c} r={r} k={k} smoother={kind} N={n_steps})")
    assert 1 <= it <= 60, it


def test_all_at_once_vcycle_is_linear_and_contracting(ctx, stmg):
    """V-cycle with zero initial guess is a linear map (solver.cpp:69-93,
    tests/test_solver.cpp:209-224), and one all-at-once cycle reduces the
    residual of a consistent right-hand side."""
    n = 4
    sol = stmg.Solver(ctx, 3, 1, 1, n_steps=n, nu=1.0, gamma=1.0, nu1=2, nu2=2)
    lv = sol.finest
    b1 = dev(consistent(lv, 1, 3, n))
    b2 = dev(consistent(lv, 1, 4, n))
    x1, x2, x12 = (torch.zeros_like(b1) for _ in range(3))
    sol.vcycle_all_at_once(b1, x1, n)
    sol.vcycle_all_at_once(b2, x2, n)
    sol.vcycle_all_at_once(b1 + 2.5 * b2, x12, n)
    lin = x1 + 2.5 * x2
    assert float((x12 - lin).abs().max() / lin.abs().max()) <= 1e-11
    r = torch.empty_like(b1)
    lv.residual(b1, x1, r, n, None, coupled=True)
    assert float(r.norm()) <= 0.75 * float(b1.norm())


def test_macro_steps_hand_off(ctx, stmg):
    """Two consecutive all-at-once slabs coupled through v_init (macro steps,
    PAPER.md:494-514) reproduce the time-marched trajectory."""
    n_steps, half = 8, 4
    sol = stmg.Solver(ctx, 3, 1, 1, n_steps=n_steps, nu=1.0, gamma=1.0, nu1=2, nu2=2, rtol=1e-12)
    ref = oc.OracleSolver(3, 1, 1, n_steps=n_steps, nu=1.0, gamma=1.0, nu1=2, nu2=2, rtol=1e-12)
    lv = sol.finest
    F = consistent(lv, 1, 23, n_steps)
    Fd = dev(F)
    X = torch.zeros_like(Fd)
    m = half * lv.size
    sol.solve_all_at_once(Fd[:m], X[:m], half)
    v = X[(half - 1) * lv.size + (lv.n_slots - 1) * lv.n_velocity:(half - 1) * lv.size + lv.n_slots * lv.n_velocity]
    sol.solve_all_at_once(Fd[m:], X[m:], half, v_init=v.contiguous())
    Xr, _, _ = ref.time_march(F)
    assert np.linalg.norm(host(X) - Xr) <= SOLVE_TOL * np.linalg.norm(Xr)


@pytest.mark.parametrize("world", [2, 4])
def test_time_slab_partition_loopback(stmg, world):
    """World ranks of n_local intervals each (threads sharing the GPU,
    host-synchronised exchanges) solve the same global system as one rank:
    halo exchange, all-reduced Krylov dots and the all-gathered coarse
    forward substitution reproduce the unpartitioned solve."""
    from paper_2502_09159_b200 import timeslab

    c, r, k, n_local = 3, 1, 1, 2
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
                ctx_r = stmg.Context(0, stream=stream)
                sol = stmg.Solver(ctx_r, c, r, k, n_steps=n_local, t_end=n_local * tau, nu=1.0, gamma=1.0,
                                  nu1=2, nu2=2, rtol=1e-11)
                sol.set_comm(timeslab.LoopbackComm(hub, rank))
                Fr = F[rank * m:(rank + 1) * m].clone()
                Xr = torch.zeros_like(Fr)
                stream.synchronize()
                it, _ = sol.solve_all_at_once(Fr, Xr, n_local)
                stream.synchronize()
                Xp[rank * m:(rank + 1) * m].copy_(Xr)
                stream.synchronize()
                results[rank] = it
        except BaseException as exc:  # surfaced below
            errors.append(exc)
            hub.barrier.abort()

    threads = [threading.Thread(target=run, args=(q,)) for q in range(world)]
    for t in threads:
        t.start()
    for t in threads:
        t.join(300)
    assert not errors, errors
    assert sorted(results) == list(range(world))
    assert len(set(results.values())) == 1  # every rank ran the same Krylov iterations
    assert abs(results[0] - it1) <= 1, (results, it1)
    torch.cuda.synchronize()
    assert float((Xp - X1).norm() / X1.norm()) <= 1e-9


def test_torch_comm_over_nccl_single_rank(stmg):
    """The NCCL flavour of the communicator on real device memory (one rank:
    NCCL cannot pair two ranks on one GPU): raw-pointer views, the library's
    stream, all-reduce and all-gather through torch.distributed/NCCL, and a
    partitioned solve object with the communicator installed."""
    import os
    import socket

    import torch.distributed as dist

    from paper_2502_09159_b200 import timeslab

    sock = socket.socket()
    sock.bind(("127.0.0.1", 0))
    port = sock.getsockname()[1]
    sock.close()
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        comm = timeslab.TorchComm(device="cuda:0")
        stream = torch.cuda.Stream()
        buf = torch.arange(6, dtype=torch.float64, device="cuda")
        recv = torch.full((4,), -1.0, dtype=torch.float64, device="cuda")
        out = torch.zeros(3, dtype=torch.float64, device="cuda")
        src = torch.tensor([1.0, 2.0, 3.0], dtype=torch.float64, device="cuda")
        torch.cuda.synchronize()
        comm.allreduce_sum(buf.data_ptr(), 6, stream.cuda_stream)
        comm.allgather(src.data_ptr(), out.data_ptr(), 3, stream.cuda_stream)
        comm.exchange_halo(src.data_ptr(), recv.data_ptr(), 3, stream.cuda_stream)  # single rank: no-op
        stream.synchronize()
        assert torch.equal(buf, torch.arange(6, dtype=torch.float64, device="cuda"))
        assert torch.equal(out, src)
        assert bool((recv == -1.0).all())
        # the solver accepts it and solves exactly as without a communicator
        ctx = stmg.Context(0)
        sol = stmg.Solver(ctx, 3, 1, 1, n_steps=4, nu=1.0, nu1=2, nu2=2, rtol=1e-10)
        lv = sol.finest
        F = torch.from_numpy(oc.make_consistent(oc.seeded(4 * lv.size, 9), lv.n_slots, lv.n_scalar, lv.grid_x,
                                                lv.n_pressure, 64, 3, 4)).cuda()
        X0 = torch.zeros_like(F)
        it0, _ = sol.solve_all_at_once(F, X0, 4)
        sol.set_comm(comm)
        X1 = torch.zeros_like(F)
        it1, _ = sol.solve_all_at_once(F, X1, 4)
        assert it0 == it1 and torch.equal(X0, X1)
    finally:
        dist.destroy_process_group()
