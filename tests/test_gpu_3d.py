"""GPU tier, 3D (BASELINE C3 / C5): the sm_100a 3D path through the C ABI
against the oracle's 3D restatement (oracle/src/st3d.cpp) on the same seeded
inputs: vmult / residual (relative max-norm <= 1e-12), the cell-Vanka smoother
step (<= 1e-10), transfers with time coarsening, the exact coarse forward
substitution, the all-at-once V-cycle (<= 1e-10) and the FGMRES solve
(iterations +-1 against the oracle's FGMRES; solution against the oracle's
time-marched direct solve <= 1e-8), on Cartesian and deformed meshes."""
import threading

import numpy as np
import pytest
import torch

import oracle3_ctypes as o3

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


CASES = [  # nx, ny, nz, r, k, gamma, amp
    (2, 2, 2, 1, 1, 1.0, 0.0),
    (3, 2, 4, 1, 0, 0.0, 0.0),
    (2, 3, 2, 1, 2, 0.7, 0.0),
    (2, 2, 2, 2, 2, 1.0, 0.0),
    (3, 2, 2, 2, 1, 0.0, 0.0),
    (3, 3, 2, 1, 1, 1.0, 0.1),
    (2, 2, 3, 2, 2, 1.0, 0.1),
    # several 16-cell blocks with a ragged last one, blocks straddling
    # intervals (cell-minor thread maps of the r = 1 kernels)
    (5, 4, 3, 1, 1, 1.0, 0.0),
    (4, 3, 3, 1, 2, 0.5, 0.1),
]


@pytest.mark.parametrize("nx,ny,nz,r,k,gamma,amp", CASES)
def test_vmult3_matches_oracle(stmg, ctx, oracle, nx, ny, nz, r, k, gamma, amp):
    verts = o3.vertices(nx, ny, nz, amp, seed=11) if amp else None
    tau = 1.0 / 8
    ref = o3.OracleLevel3(nx, ny, nz, r, k, tau, 1.0, gamma, vertices=verts, smoother=False)
    lvl = stmg.Level3(ctx, nx, ny, nz, r, k, tau, 1.0, gamma, stmg.SMOOTHER_NONE, vertices=verts)
    assert (lvl.size, lvl.n_velocity, lvl.n_pressure) == (ref.size, ref.mv, ref.mp)
    rng = np.random.default_rng(1)
    n = 3
    x = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.mv)
    b = rng.uniform(-1, 1, n * ref.size)
    for raw in (False, True):
        y = torch.zeros(ref.size, dtype=torch.float64, device="cuda")
        lvl.apply_block(_cuda(x[:ref.size]), y, 1, raw=raw)
        assert _rel(y.cpu().numpy(), ref.apply_block(x[:ref.size], raw=raw)) <= 1e-12
    y = torch.zeros(n * ref.size, dtype=torch.float64, device="cuda")
    lvl.vmult(_cuda(x), y, n, _cuda(halo))
    yr = ref.vmult_all(x, n, halo)
    assert _rel(y.cpu().numpy(), yr) <= 1e-12
    r_ = torch.zeros_like(y)
    lvl.residual(_cuda(b), _cuda(x), r_, n, _cuda(halo), coupled=True)
    assert _rel(r_.cpu().numpy(), b - yr) <= 1e-12


@pytest.mark.parametrize("nx,ny,nz,r,k,gamma,amp", [c for c in CASES if c[3] == 1] + [(2, 2, 2, 2, 2, 1.0, 0.0),
                                                                                     (2, 2, 2, 2, 1, 1.0, 0.1)])
def test_smooth_step3_matches_oracle(stmg, ctx, oracle, nx, ny, nz, r, k, gamma, amp):
    verts = o3.vertices(nx, ny, nz, amp, seed=11) if amp else None
    tau = 1.0 / 8
    ref = o3.OracleLevel3(nx, ny, nz, r, k, tau, 1.0, gamma, vertices=verts)
    lvl = stmg.Level3(ctx, nx, ny, nz, r, k, tau, 1.0, gamma, stmg.SMOOTHER_CELL, vertices=verts)
    rng = np.random.default_rng(2)
    n = 2
    u = rng.uniform(-1, 1, n * ref.size)
    b = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.mv)
    ug = _cuda(u)
    lvl.smooth_step(_cuda(b), ug, 0.8, n, _cuda(halo), coupled=True)
    ur = ref.smooth_step_all(b, u, 0.8, n, halo)
    assert _rel(ug.cpu().numpy(), ur) <= 1e-10


def test_single_cell_whole_domain_patch3(stmg, ctx, oracle):
    """The 1x1x1 patch is singular (pressure constant): pseudo-inverse, as the
    reference's COD fall-back (vanka.cpp:167-176)."""
    ref = o3.OracleLevel3(1, 1, 1, 1, 1, 0.5, 1.0, 1.0)
    lvl = stmg.Level3(ctx, 1, 1, 1, 1, 1, 0.5, 1.0, 1.0, stmg.SMOOTHER_CELL)
    b = o3.make_consistent3(np.random.default_rng(3).uniform(-1, 1, ref.size), ref)
    u = torch.zeros(ref.size, dtype=torch.float64, device="cuda")
    lvl.smooth_step(_cuda(b), u, 1.0, 1)
    assert _rel(u.cpu().numpy(), ref.smooth_step_all(b, np.zeros(ref.size), 1.0, 1)) <= 1e-10


HIER = [  # nx, r, k, N, n_hcoarse, amp, time_coarsen, k_min
    (2, 1, 1, 2, 1, 0.0, True, 0),
    (4, 1, 1, 4, 2, 0.0, True, 0),
    (2, 2, 2, 2, 1, 0.0, True, 0),
    (4, 1, 1, 2, 1, 0.1, True, 0),
    (4, 1, 1, 3, 2, 0.0, False, 1),
    (2, 2, 2, 2, 1, 0.1, False, 2),
]


def _pair(stmg, ctx, nx, r, k, N, nh, amp, tc, kmin, rtol=1e-8):
    verts = o3.vertices(nx, nx, nx, amp, seed=4) if amp else None
    H = o3.OracleHier3(nx, nx, nx, r, k, N, t_end=N / 8.0, n_hcoarse=nh, time_coarsen=tc, vertices=verts, k_min=kmin)
    S = stmg.Solver3(ctx, nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, n_hcoarse=nh, time_coarsen=tc, k_min=kmin,
                     vertices=verts, rtol=rtol)
    assert [(l["nx"], l["r"], l["k"], l["tshift"], l["size"]) for l in S.level_info] == \
        [(l["nx"], l["r"], l["k"], l["tshift"], l["size"]) for l in H.levels]
    return H, S


def _project_all(lvl_ref, x, n, residual=False):
    x = x.copy()
    proj = lvl_ref.project_residual if residual else lvl_ref.project_mean_zero
    for t in range(n):
        for a in range(lvl_ref.S):
            p0 = t * lvl_ref.size + lvl_ref.S * lvl_ref.mv + a * lvl_ref.mp
            x[p0:p0 + lvl_ref.mp] = proj(np.ascontiguousarray(x[p0:p0 + lvl_ref.mp]))
    return x


def _zero_bnd(lvl_ref, x, n):
    x = x.reshape(n, lvl_ref.size).copy()
    bnd = o3.boundary_mask3(lvl_ref.gx, lvl_ref.gy, lvl_ref.gz)
    for t in range(n):
        for a in range(lvl_ref.S):
            for c in range(3):
                seg = x[t, a * lvl_ref.mv + c * lvl_ref.nsc: a * lvl_ref.mv + (c + 1) * lvl_ref.nsc]
                seg[bnd] = 0.0
    return x.reshape(-1)


@pytest.mark.parametrize("nx,r,k,N,nh,amp,tc,kmin", HIER)
def test_transfers3_match_oracle(stmg, ctx, oracle, nx, r, k, N, nh, amp, tc, kmin):
    H, S = _pair(stmg, ctx, nx, r, k, N, nh, amp, tc, kmin)
    rng = np.random.default_rng(5)
    nI = N
    for l in range(H.n_levels - 1, 0, -1):
        fine, coarse = H.levels[l], H.levels[l - 1]
        ht = coarse["tshift"] > fine["tshift"]
        nc = nI // 2 if ht else nI
        xf = rng.uniform(-1, 1, nI * fine["size"])
        xc = rng.uniform(-1, 1, nc * coarse["size"])
        # restrict_residual = R, zero constrained, project (transfer.cpp:117-132)
        want = _project_all(H.level[l - 1], _zero_bnd(H.level[l - 1], H.restrict(l, xf, nc), nc), nc, True)
        got = torch.zeros(nc * coarse["size"], dtype=torch.float64, device="cuda")
        S.restrict_residual(l, _cuda(xf), got, nc)
        assert _rel(got.cpu().numpy(), want) <= 1e-12, ("restrict", l)
        want = _project_all(H.level[l], _zero_bnd(H.level[l], H.prolongate(l, xc, nc), nI), nI)
        got = torch.zeros(nI * fine["size"], dtype=torch.float64, device="cuda")
        S.prolongate_correction(l, _cuda(xc), got, nc)
        assert _rel(got.cpu().numpy(), want) <= 1e-12, ("prolongate", l)
        nI = nc


@pytest.mark.parametrize("nx,r,k,N,nh,amp,tc,kmin", HIER)
def test_coarse_forward_and_vcycle3_match_oracle(stmg, ctx, oracle, nx, r, k, N, nh, amp, tc, kmin):
    H, S = _pair(stmg, ctx, nx, r, k, N, nh, amp, tc, kmin)
    c0 = H.level[0]
    n0 = N >> H.levels[0]["tshift"]
    bc = o3.make_consistent3(np.random.default_rng(6).uniform(-1, 1, n0 * c0.size), c0, n0)
    xc = torch.zeros(n0 * c0.size, dtype=torch.float64, device="cuda")
    S.coarse_forward(_cuda(bc), xc, n0)
    assert _rel(xc.cpu().numpy(), H.coarse_forward(bc, n0)) <= 1e-10
    f = H.level[-1]
    b = o3.make_consistent3(np.random.default_rng(8).uniform(-1, 1, N * f.size), f, N)
    x = torch.zeros(N * f.size, dtype=torch.float64, device="cuda")
    S.vcycle_all_at_once(_cuda(b), x, N)
    assert _rel(x.cpu().numpy(), H.vcycle(b, N)) <= 1e-10


@pytest.mark.parametrize("nx,r,k,N,nh,amp,tc,kmin", HIER)
def test_fgmres3_solve_matches_time_marched(stmg, ctx, oracle, nx, r, k, N, nh, amp, tc, kmin):
    """All-at-once solve = time-marched solution of the same system (<= 1e-8),
    iterations within +-1 of the oracle's FGMRES."""
    H, S = _pair(stmg, ctx, nx, r, k, N, nh, amp, tc, kmin, rtol=1e-10)
    f = H.level[-1]
    b = o3.make_consistent3(np.random.default_rng(9).uniform(-1, 1, N * f.size), f, N)
    X = torch.zeros(N * f.size, dtype=torch.float64, device="cuda")
    it, hist = S.solve_all_at_once(_cuda(b), X, N)
    xr, itr = H.fgmres(b, N, rtol=1e-10)
    assert abs(it - itr) <= 1, (it, itr)
    xd = f.direct_time_march(b, N)
    assert np.linalg.norm(X.cpu().numpy() - xd) / np.linalg.norm(xd) <= 1e-8


def test_time_slab_partition3_loopback(stmg, ctx, oracle):
    """Two time slabs (threads, host-synchronised loopback exchanges) reproduce
    the unpartitioned 3D all-at-once solve, time coarsening included."""
    from paper_2502_09159_b200 import timeslab

    nx, r, k, n_local, world = 2, 1, 1, 2, 2
    N = n_local * world
    S1 = stmg.Solver3(ctx, nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, n_hcoarse=1, rtol=1e-11)
    f = S1.finest
    ref = o3.OracleLevel3(nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, smoother=False)
    F = _cuda(o3.make_consistent3(np.random.default_rng(10).uniform(-1, 1, N * f.size), ref, N))
    X1 = torch.zeros_like(F)
    it1, _ = S1.solve_all_at_once(F, X1, N)
    torch.cuda.synchronize()
    hub = timeslab.LoopbackHub(world, timeout=120.0)
    Xp = torch.zeros_like(F)
    results, errors = {}, []
    m = n_local * f.size

    def run(rank):
        try:
            stream = torch.cuda.Stream()
            with torch.cuda.stream(stream):
                ctx_r = stmg.Context(0, stream=stream)
                sol = stmg.Solver3(ctx_r, nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, n_hcoarse=1, rtol=1e-11)
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
    assert len(set(results.values())) == 1
    assert abs(results[0] - it1) <= 1
    torch.cuda.synchronize()
    assert float((Xp - X1).norm() / X1.norm()) <= 1e-9


def test_affine_patch_smoother_solve_on_deformed_mesh(stmg, ctx, oracle):
    """affine_patches: the undeformed patch inverses as an approximate local
    solve on a deformed mesh (the C5-scale setting). The smoother differs from
    the reference's exact one, the converged all-at-once solution does not:
    it equals the oracle's direct time-marched solution (<= 1e-8)."""
    nx, r, k, N = 2, 2, 2, 2
    verts = o3.vertices(nx, nx, nx, 0.1, seed=4)
    S = stmg.Solver3(ctx, nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, n_hcoarse=1, time_coarsen=False, k_min=1,
                     vertices=verts, affine_patches=True, rtol=1e-10)
    ref = o3.OracleLevel3(nx, nx, nx, r, k, 1.0 / 8, 1.0, 1.0, vertices=verts, smoother=False)
    b = o3.make_consistent3(np.random.default_rng(12).uniform(-1, 1, N * ref.size), ref, N)
    X = torch.zeros(N * ref.size, dtype=torch.float64, device="cuda")
    it, _ = S.solve_all_at_once(_cuda(b), X, N)
    xd = ref.direct_time_march(b, N)
    assert np.linalg.norm(X.cpu().numpy() - xd) / np.linalg.norm(xd) <= 1e-8
    assert it <= 40


def test_vmult3_gemm_kernel_matches_oracle(stmg, ctx, oracle, monkeypatch):
    """The opt-in DMMA GEMM vmult (Cartesian r = 1, dense element operator) on
    the same parity bar as the default kernel: plain, raw, coupled, residual."""
    monkeypatch.setenv("STMG_V3_GEMM", "1")
    for nx, ny, nz, k, gamma in [(2, 2, 2, 1, 1.0), (3, 2, 4, 0, 0.0), (2, 3, 2, 2, 0.7)]:
        tau = 1.0 / 8
        ref = o3.OracleLevel3(nx, ny, nz, 1, k, tau, 1.0, gamma, smoother=False)
        lvl = stmg.Level3(ctx, nx, ny, nz, 1, k, tau, 1.0, gamma, stmg.SMOOTHER_NONE)
        rng = np.random.default_rng(3)
        n = 3
        x = rng.uniform(-1, 1, n * ref.size)
        halo = rng.uniform(-1, 1, ref.mv)
        b = rng.uniform(-1, 1, n * ref.size)
        for raw in (False, True):
            y = torch.zeros(ref.size, dtype=torch.float64, device="cuda")
            lvl.apply_block(_cuda(x[:ref.size]), y, 1, raw=raw)
            assert _rel(y.cpu().numpy(), ref.apply_block(x[:ref.size], raw=raw)) <= 1e-12
        y = torch.zeros(n * ref.size, dtype=torch.float64, device="cuda")
        lvl.vmult(_cuda(x), y, n, _cuda(halo))
        yr = ref.vmult_all(x, n, halo)
        assert _rel(y.cpu().numpy(), yr) <= 1e-12
        r_ = torch.zeros_like(y)
        lvl.residual(_cuda(b), _cuda(x), r_, n, _cuda(halo), coupled=True)
        assert _rel(r_.cpu().numpy(), b - yr) <= 1e-12


def test_3d_status_codes(stmg, ctx):
    """invalid_argument cases of the 3D entry points map to STMG_EINVAL (1),
    like the reference's exceptions (vanka.cpp:223-224, transfer.cpp:155-158)."""
    with pytest.raises(stmg.StmgError) as e:
        stmg.Level3(ctx, 2, 2, 2, 3, 1, 0.1, 1.0, 1.0, stmg.SMOOTHER_CELL)  # r = 3 not instantiated in 3D
    assert e.value.code == 1
    with pytest.raises(stmg.StmgError) as e:
        stmg.Level3(ctx, 2, 2, 2, 1, 1, -0.1, 1.0, 1.0, stmg.SMOOTHER_CELL)  # tau <= 0
    assert e.value.code == 1
    with pytest.raises(stmg.StmgError) as e:
        stmg.Level3(ctx, 2, 2, 2, 1, 1, 0.1, 1.0, 1.0, stmg.SMOOTHER_VERTEX_STAR)  # cell Vanka only in 3D
    assert e.value.code == 1
    lvl = stmg.Level3(ctx, 2, 2, 2, 1, 1, 0.1, 1.0, 1.0, stmg.SMOOTHER_CELL)
    b = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    with pytest.raises(stmg.StmgError) as e:
        lvl.smooth_step(b, b.clone(), 1.5, 1)  # omega outside (0, 1]
    assert e.value.code == 1
    with pytest.raises(stmg.StmgError) as e:
        stmg.Solver3(ctx, 3, 3, 3, 1, 1, 0.1, n_hcoarse=1)  # mesh not divisible
    assert e.value.code == 1
    S = stmg.Solver3(ctx, 2, 2, 2, 1, 1, 0.1, n_hcoarse=1, time_coarsen=True)
    F = torch.zeros(3 * S.finest.size, dtype=torch.float64, device="cuda")
    with pytest.raises(stmg.StmgError) as e:
        S.solve_all_at_once(F, F.clone(), 3)  # 3 intervals cannot halve in time
    assert e.value.code == 1


@pytest.mark.parametrize("nx,ny,nz,r,k", [(2, 2, 2, 1, 1), (3, 2, 2, 2, 2), (2, 3, 2, 1, 2), (2, 2, 3, 2, 1)])
def test_gpu_patch_setup_matches_host_and_oracle(stmg, ctx, oracle, nx, ny, nz, r, k):
    """Deformed levels build their exact per-cell patch inverses on the GPU
    (element matrices, R_T S R_T^T, batched Gauss-Jordan; patch3_gpu.cu):
    the smoother step equals the host-built one (LU with partial pivoting,
    STMG_PATCH3_HOST) and the oracle's (vanka.cpp:30-233) to <= 1e-10."""
    import os

    verts = o3.vertices(nx, ny, nz, 0.1, seed=21)
    tau = 1.0 / 8
    gpu = stmg.Level3(ctx, nx, ny, nz, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=verts)
    assert gpu.patch_setup["on_gpu"] and gpu.patch_setup["classes"] == nx * ny * nz
    os.environ["STMG_PATCH3_HOST"] = "1"
    try:
        hst = stmg.Level3(ctx, nx, ny, nz, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=verts)
    finally:
        del os.environ["STMG_PATCH3_HOST"]
    assert not hst.patch_setup["on_gpu"]
    ref = o3.OracleLevel3(nx, ny, nz, r, k, tau, 1.0, 1.0, vertices=verts)
    rng = np.random.default_rng(22)
    n = 3
    u = rng.uniform(-1, 1, n * ref.size)
    b = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.mv)
    ur = ref.smooth_step_all(b, u, 0.8, n, halo)
    outs = []
    for lvl in (gpu, hst):
        ug = _cuda(u)
        lvl.smooth_step(_cuda(b), ug, 0.8, n, _cuda(halo), coupled=True)
        outs.append(ug.cpu().numpy())
        assert _rel(outs[-1], ur) <= 1e-10
    assert _rel(outs[0], outs[1]) <= 1e-10


@pytest.mark.parametrize("nx,ny,nz,r,n", [(4, 4, 4, 2, 20), (3, 4, 2, 1, 5)])
def test_time_diagonalised_patches_match_dense(stmg, ctx, nx, ny, nz, r, n):
    """DG(2) deformed levels apply their exact patch inverses in the
    time-diagonalised form (one real and one pair block per cell,
    vanka_big_fac_kernel): the smoother step equals the dense-inverse one
    (STMG_VANKA3_DENSE) to <= 1e-10, with a ragged 16-interval group."""
    import os

    verts = o3.vertices(nx, ny, nz, 0.1, seed=23)
    tau = 1.0 / 8
    fac = stmg.Level3(ctx, nx, ny, nz, r, 2, tau, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=verts)
    assert fac.patch_setup["factored"]
    os.environ["STMG_VANKA3_DENSE"] = "1"
    try:
        den = stmg.Level3(ctx, nx, ny, nz, r, 2, tau, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=verts)
    finally:
        del os.environ["STMG_VANKA3_DENSE"]
    assert den.patch_setup["on_gpu"] and not den.patch_setup["factored"]
    # the roofline bookkeeping of the bench: per patch of n_T = 3 n_s rows the factored form stores
    # 5 n_s^2 doubles (+ alignment), streams 3 n_s^2 per sweep and does 5 n_s^2 multiply-adds per column
    # (dense: n_T^2 = 9 n_s^2 of each); summed over the patches sum(n_T^2) = den.total_matrix_elements
    sum_nt2 = den.total_matrix_elements
    ps = fac.patch_setup
    assert ps["streamed_elements"] * 3 == sum_nt2 and ps["macs_per_column"] * 9 == sum_nt2 * 5
    assert sum_nt2 * 5 // 9 <= fac.total_matrix_elements <= sum_nt2 * 5 // 9 + 20 * nx * ny * nz
    assert den.patch_setup["streamed_elements"] == 0
    rng = np.random.default_rng(24)
    u = rng.uniform(-1, 1, n * fac.size)
    b = rng.uniform(-1, 1, n * fac.size)
    halo = rng.uniform(-1, 1, fac.n_velocity)
    outs = []
    for lvl in (fac, den):
        ug = _cuda(u)
        lvl.smooth_step(_cuda(b), ug, 0.8, n, _cuda(halo), coupled=True)
        outs.append(ug.cpu().numpy())
    assert _rel(outs[0], outs[1]) <= 1e-10
