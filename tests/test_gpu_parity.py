"""GPU tier: the sm_100a kernels through the C ABI against the oracle on the
same seeded inputs. Tolerances are the north star's: vmult relative
max-norm <= 1e-12, smoother step <= 1e-10, solve iterations within +-1 and
solution relative L2 <= 1e-8."""
import numpy as np
import pytest
import torch

import oracle_ctypes as oc

pytestmark = pytest.mark.gpu

VMULT_TOL = 1e-12
SMOOTH_TOL = 1e-10


def rel_max(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


LEVEL_CASES = [
    # nc, r, k, tau, nu, gamma
    (1, 1, 1, 0.25, 0.1, 1.0),
    (2, 1, 1, 0.25, 0.1, 0.0),
    (4, 2, 2, 0.25, 0.1, 1.0),
    (4, 3, 1, 0.5, 0.1, 0.7),
    (8, 1, 0, 0.125, 1.0, 1.0),
    (16, 1, 1, 0.125, 1.0, 1.0),   # C1 discretisation
    (32, 2, 2, 1 / 64, 1.0, 1.0),  # C2 discretisation, 2 strips
    (64, 1, 1, 1 / 64, 1.0, 1.0),  # 3 strips, row segments
    (4, 4, 4, 0.25, 0.1, 1.0),
    (8, 2, 3, 0.3, 0.5, 0.0),
]


@pytest.mark.parametrize("nc,r,k,tau,nu,gamma", LEVEL_CASES)
def test_apply_block_matches_oracle(ctx, stmg, nc, r, k, tau, nu, gamma):
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, nu, gamma, stmg.SMOOTHER_NONE)
    ref = oc.OracleLevel(nc, r, k, tau, nu, gamma, build_smoother=False)
    assert lvl.size == ref.size
    for seed, raw in ((1, False), (2, True)):
        x = oc.seeded(ref.size, seed)
        y = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
        lvl.apply_block(dev(x), y, raw=raw)
        err = rel_max(host(y), ref.apply_block(x, raw=raw))
        assert err <= VMULT_TOL, err


@pytest.mark.parametrize("nc,r,k,tau,nu,gamma", [c for c in LEVEL_CASES if c[0] >= 2])
def test_all_at_once_vmult_with_coupling(ctx, stmg, nc, r, k, tau, nu, gamma):
    """y_n = D x_n - Z C x_{n-1}[slot k] over N intervals plus the halo slot."""
    N = 5
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, nu, gamma, stmg.SMOOTHER_NONE)
    ref = oc.OracleLevel(nc, r, k, tau, nu, gamma, build_smoother=False)
    x = oc.seeded(N * ref.size, 11)
    halo = oc.seeded(ref.n_velocity, 12)
    y = torch.zeros(N * lvl.size, dtype=torch.float64, device="cuda")
    lvl.vmult(dev(x), y, N, dev(halo))
    err = rel_max(host(y), ref.vmult_all(x, N, halo))
    assert err <= VMULT_TOL, err
    # residual form b - A x
    b = oc.seeded(N * ref.size, 13)
    r_ = torch.zeros_like(y)
    lvl.residual(dev(b), dev(x), r_, N, dev(halo), coupled=True)
    err = rel_max(host(r_), b - ref.vmult_all(x, N, halo))
    assert err <= VMULT_TOL, err


def test_coupling_rhs_matches_oracle(ctx, stmg):
    lvl = stmg.Level(ctx, 8, 8, 2, 2, 0.25, 0.1, 1.0, stmg.SMOOTHER_NONE)
    ref = oc.OracleLevel(8, 2, 2, 0.25, 0.1, 1.0, build_smoother=False)
    v = oc.seeded(ref.n_velocity, 5)
    out = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    lvl.coupling_rhs(dev(v), out)
    assert rel_max(host(out), ref.coupling_rhs(v)) <= VMULT_TOL


SMOOTH_CASES = [
    (4, 1, 1, 0),
    (4, 2, 2, 0),
    (8, 1, 1, 1),
    (4, 2, 1, 1),
    (16, 1, 1, 0),
    (32, 2, 2, 0),
    (1, 2, 1, 0),   # whole-domain patch: pseudo-inverse (min-norm, vanka.cpp:167-176)
    (2, 3, 2, 0),
]


@pytest.mark.parametrize("nc,r,k,kind", SMOOTH_CASES)
def test_apply_additive_matches_oracle(ctx, stmg, nc, r, k, kind):
    tau, nu, gamma = 0.25, 0.1, 1.0
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, nu, gamma, kind)
    ref = oc.OracleLevel(nc, r, k, tau, nu, gamma, kind)
    res = oc.seeded(ref.size, 21)
    out = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    lvl.apply_additive(dev(res), out)
    err = rel_max(host(out), ref.apply_additive(res))
    assert err <= SMOOTH_TOL, err


@pytest.mark.parametrize("nc,r,k,kind", [c for c in SMOOTH_CASES if c[0] >= 2])
def test_smooth_step_all_at_once_matches_oracle(ctx, stmg, nc, r, k, kind):
    N, tau, nu, gamma, omega = 3, 0.25, 0.1, 1.0, 0.8
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, nu, gamma, kind)
    ref = oc.OracleLevel(nc, r, k, tau, nu, gamma, kind)
    b = oc.seeded(N * ref.size, 31)
    u = oc.seeded(N * ref.size, 32)
    halo = oc.seeded(ref.n_velocity, 33)
    ud = dev(u)
    lvl.smooth_step(dev(b), ud, omega, N, dev(halo), coupled=True)
    err = rel_max(host(ud), ref.smooth_step_all(b, u, omega, N, halo))
    assert err <= SMOOTH_TOL, err


def test_smooth_step_rejects_bad_omega(ctx, stmg):
    lvl = stmg.Level(ctx, 4, 4, 1, 1, 0.25, 0.1, 1.0, stmg.SMOOTHER_CELL)
    v = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    for omega in (0.0, 1.5):
        with pytest.raises(stmg.StmgError) as e:
            lvl.smooth_step(v, v.clone(), omega)
        assert e.value.code == 1


SOLVER_CASES = [
    # refinements, r, k, nu, gamma, smoother, nu1, nu2, h_only
    (2, 1, 1, 0.1, 1.0, 0, 1, 1, False),
    (2, 2, 2, 0.1, 1.0, 0, 1, 1, False),
    (3, 2, 2, 1.0, 1.0, 0, 2, 2, False),
    (2, 2, -1, 0.1, 1.0, 0, 1, 1, True),
    (2, 1, 1, 0.1, 1.0, 1, 1, 1, False),
    (4, 1, 1, 1.0, 1.0, 0, 2, 2, False),   # C1: 16x16, Q2/P1, DG(1), V(2,2)
]


def _consistent(sol, ref, seed, n_intervals=1):
    lv = sol.finest
    ncell = lv.n_pressure // ((ref.levels[-1]["r"] + 1) * (ref.levels[-1]["r"] + 2) // 2)
    npc = lv.n_pressure // ncell
    v = oc.seeded(n_intervals * lv.size, seed)
    return oc.make_consistent(v, lv.n_slots, lv.n_scalar, lv.grid_x, lv.n_pressure, ncell, npc, n_intervals)


@pytest.mark.parametrize("c,r,k,nu,gamma,kind,nu1,nu2,h_only", SOLVER_CASES)
def test_transfers_and_coarse_solve_match_oracle(ctx, stmg, c, r, k, nu, gamma, kind, nu1, nu2, h_only):
    sol = stmg.Solver(ctx, c, r, k, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2, h_only=h_only)
    ref = oc.OracleSolver(c, r, k, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2, h_only=h_only)
    assert sol.n_levels == ref.n_levels
    for l in range(1, sol.n_levels):
        fine = oc.seeded(ref.levels[l]["size"], 40 + l)
        coarse = oc.seeded(ref.levels[l - 1]["size"], 60 + l)
        cd = torch.zeros(ref.levels[l - 1]["size"], dtype=torch.float64, device="cuda")
        sol.restrict_residual(l, dev(fine), cd, True)
        assert rel_max(host(cd), ref.restrict_residual(l, fine)) <= 1e-12
        fd = torch.zeros(ref.levels[l]["size"], dtype=torch.float64, device="cuda")
        sol.prolongate_correction(l, dev(coarse), fd, True)
        assert rel_max(host(fd), ref.prolongate_correction(l, coarse)) <= 1e-12


@pytest.mark.parametrize("c,r,k,nu,gamma,kind,nu1,nu2,h_only", SOLVER_CASES)
def test_vcycle_and_gmres_match_oracle(ctx, stmg, c, r, k, nu, gamma, kind, nu1, nu2, h_only):
    sol = stmg.Solver(ctx, c, r, k, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2, h_only=h_only)
    ref = oc.OracleSolver(c, r, k, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2, h_only=h_only)
    b = _consistent(sol, ref, 77)
    x = torch.zeros(sol.finest.size, dtype=torch.float64, device="cuda")
    sol.vcycle(dev(b), x)
    assert rel_max(host(x), ref.vcycle(b)) <= SMOOTH_TOL
    it, hist = sol.gmres(dev(b), x)
    xr, itr, histr = ref.gmres(b)
    assert abs(it - itr) <= 1, (it, itr)
    xs = host(x)
    assert np.linalg.norm(xs - xr) <= 1e-8 * np.linalg.norm(xr)


@pytest.mark.parametrize("c,r,k,nu,gamma,kind,nu1,nu2,h_only", [SOLVER_CASES[0], SOLVER_CASES[5]])
def test_time_march_matches_oracle(ctx, stmg, c, r, k, nu, gamma, kind, nu1, nu2, h_only):
    """Seeded time marching (C1 = last case): per-step iterations within +-1,
    trajectory relative L2 <= 1e-8 after the per-slot mean-zero projection."""
    n_steps = 8
    sol = stmg.Solver(ctx, c, r, k, n_steps=n_steps, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2,
                      h_only=h_only)
    ref = oc.OracleSolver(c, r, k, n_steps=n_steps, nu=nu, gamma=gamma, smoother=kind, nu1=nu1, nu2=nu2,
                          h_only=h_only)
    F = _consistent(sol, ref, 99, n_steps)
    X = torch.zeros(n_steps * sol.finest.size, dtype=torch.float64, device="cuda")
    iters = sol.time_march(dev(F), X)
    Xr, itr, _ = ref.time_march(F)
    assert all(abs(a - b) <= 1 for a, b in zip(iters, itr)), (iters, itr)
    Xs = host(X)
    assert np.linalg.norm(Xs - Xr) <= 1e-8 * np.linalg.norm(Xr)
    # host-buffer entry point gives the same trajectory
    Xh = np.zeros_like(F)
    iters_h = sol.time_march_host(F, Xh)
    assert iters_h == iters
    assert np.linalg.norm(Xh - Xs) <= 1e-12 * np.linalg.norm(Xs)


def test_kernels_really_launch(ctx, stmg):
    before = ctx.launch_count()
    lvl = stmg.Level(ctx, 16, 16, 1, 1, 0.125, 1.0, 1.0, stmg.SMOOTHER_CELL)
    x = torch.rand(lvl.size, dtype=torch.float64, device="cuda")
    y = torch.zeros_like(x)
    lvl.vmult(x, y)
    lvl.smooth_step(x, y, 0.8)
    assert ctx.launch_count() - before >= 1 + 1 + 4


@pytest.mark.parametrize("nc,r,k,kind,n", [(32, 2, 2, 0, 16), (24, 1, 1, 1, 16), (20, 1, 1, 0, 8), (18, 1, 1, 1, 1),
                                          (33, 2, 2, 0, 20)])
def test_vanka_update_is_bitwise_deterministic(ctx, stmg, nc, r, k, kind, n):
    """Colour-separated stages: no two concurrently running tiles add into the
    same dof, so repeated smoother updates are bitwise identical."""
    lvl = stmg.Level(ctx, nc, nc, r, k, 1.0 / 64, 1.0, 1.0, kind)
    g = torch.Generator(device="cuda")
    g.manual_seed(5)
    res = torch.rand(n * lvl.size, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    u0 = torch.rand(n * lvl.size, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    outs = []
    for _ in range(3):
        u = u0.clone()
        lvl.vanka_update(res, u, 0.8, n)
        outs.append(u)
    torch.cuda.synchronize()
    assert torch.equal(outs[0], outs[1]) and torch.equal(outs[0], outs[2])


@pytest.mark.parametrize("nc,r,k,kind,n", [(16, 2, 2, 0, 20), (32, 1, 1, 1, 17), (8, 1, 1, 0, 3)])
@pytest.mark.parametrize("with_prev", [False, True])
def test_host_buffer_entry_points_match_device_path(ctx, stmg, oracle, nc, r, k, kind, n, with_prev):
    """stmg_vmult_host / stmg_smooth_step_host (pipelined over 8-interval
    chunks) equal the device-resident calls and the oracle."""
    tau = 1.0 / 64
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, 1.0, 1.0, kind)
    ref = oc.OracleLevel(nc, r, k, tau, 1.0, 1.0, kind)
    x = oc.seeded(n * lvl.size, 71)
    bb = oc.seeded(n * lvl.size, 72)
    prev = oc.seeded(lvl.n_velocity, 73) if with_prev else None
    # vmult through host buffers vs oracle
    y = np.zeros_like(x)
    lvl.vmult_host(np.ascontiguousarray(x), y, n, prev)
    y_ref = ref.vmult_all(x, n, prev)
    assert rel_max(y, y_ref) <= VMULT_TOL
    # smoother step through host buffers vs the device path (bitwise up to
    # the patch grouping of the chunked launch) and vs the oracle
    u = x.copy()
    lvl.smooth_step_host(bb, u, 0.8, n, prev, True)
    ud = dev(x)
    lvl.smooth_step(dev(bb), ud, 0.8, n, None if prev is None else dev(prev), coupled=True)
    assert rel_max(u, host(ud)) <= 1e-13
    u_ref = ref.smooth_step_all(bb, x.copy(), 0.8, n, prev)
    assert rel_max(u, u_ref) <= SMOOTH_TOL


def test_error_codes_mirror_reference_exceptions(ctx, stmg):
    """Status codes at the C ABI follow the reference's exceptions:
    invalid_argument -> STMG_EINVAL (1), runtime_error -> STMG_ERUNTIME (2)."""
    lvl = stmg.Level(ctx, 4, 4, 1, 1, 0.25, 0.1, 1.0, stmg.SMOOTHER_CELL)
    x = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    for bad in (0.0, -0.5, 1.5):  # vanka.cpp:223-224
        with pytest.raises(stmg.StmgError) as ei:
            lvl.smooth_step(x, x.clone(), bad)
        assert ei.value.code == 1
    for r, k in [(0, 1), (5, 1), (1, 5), (1, -1)]:  # degree range
        with pytest.raises(stmg.StmgError) as ei:
            stmg.Level(ctx, 4, 4, r, k, 0.25, 0.1, 1.0, stmg.SMOOTHER_CELL)
        assert ei.value.code == 1
    with pytest.raises(stmg.StmgError) as ei:
        lvl.assemble_rhs(x, 0.0, 1, problem=7)
    assert ei.value.code == 1
    # zero intervals: a no-op, not an error
    y = torch.full_like(x, 3.0)
    lvl.vmult(x, y, 0)
    lvl.vanka_update(x, y, 0.8, 0)
    torch.cuda.synchronize()
    assert bool((y == 3.0).all())
    # GMRES non-convergence -> runtime_error (solver.cpp:275)
    sol = stmg.Solver(ctx, 2, 1, 1, nu=0.1, rtol=1e-14, atol=0.0, max_iterations=1)
    b = torch.from_numpy(oc.make_consistent(oc.seeded(sol.finest.size, 3), sol.finest.n_slots, sol.finest.n_scalar,
                                            sol.finest.grid_x, sol.finest.n_pressure, 16, 3)).cuda()
    with pytest.raises(stmg.StmgError) as ei:
        sol.gmres(b, torch.zeros_like(b))
    assert ei.value.code == 2


@pytest.mark.parametrize("nc,k,n", [(8, 2, 3), (16, 2, 17), (2, 2, 2), (8, 3, 2), (4, 4, 2)])
def test_factored_vanka_matches_oracle(ctx, stmg, oracle, nc, k, n, monkeypatch):
    """Time-diagonalised patch inverses (opt-in, STMG_VANKA_FACTORED=1):
    A_T^{-1} = (V x I) blockdiag(B^{-1}) (W x I), parity with the oracle's
    dense LU patch solves, and bitwise determinism."""
    monkeypatch.setenv("STMG_VANKA_FACTORED", "1")
    r = 2 if k == 2 else 1
    tau = 1.0 / 16
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL)
    info = stmg.patch_info(nc, nc, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL)
    assert lvl.factored == info["factored"]
    ref = oc.OracleLevel(nc, r, k, tau, 1.0, 1.0, 0)
    b = oc.seeded(n * lvl.size, 81)
    u = oc.seeded(n * lvl.size, 82)
    prev = oc.seeded(lvl.n_velocity, 83)
    outs = []
    for _ in range(2):
        ud = dev(u)
        lvl.smooth_step(dev(b), ud, 0.8, n, dev(prev), coupled=True)
        outs.append(host(ud))
    assert np.array_equal(outs[0], outs[1])
    want = ref.smooth_step_all(b, u, 0.8, n, prev)
    assert rel_max(outs[0], want) <= SMOOTH_TOL


@pytest.mark.parametrize("nc,r,k", [(4, 1, 1), (8, 2, 2), (2, 3, 1)])
def test_step_health_matches_oracle(ctx, stmg, nc, r, k):
    """time_march's saddle-point health record (solver.cpp:286-299): max over
    slots of ||B v|| / sqrt(v^T M v) and |<mean, p>| / ||p||, per interval, on
    seeded vectors and on a converged time-march trajectory."""
    lvl = stmg.Level(ctx, nc, nc, r, k, 1.0 / 8, 1.0, 1.0, stmg.SMOOTHER_NONE)
    ref = oc.OracleLevel(nc, r, k, 1.0 / 8, 1.0, 1.0, 0, build_smoother=False)
    n = 3
    X = oc.seeded(n * ref.size, 21)
    got = lvl.step_health(torch.from_numpy(X).cuda(), n)
    for t in range(n):
        want = ref.step_health(np.ascontiguousarray(X[t * ref.size:(t + 1) * ref.size]))
        assert abs(got[t][0] - want[0]) <= 1e-12 * max(1.0, want[0])
        assert abs(got[t][1] - want[1]) <= 1e-12 * max(1.0, want[1])
    sol = stmg.Solver(ctx, 2, 1, 1, n_steps=4, nu=1.0, gamma=1.0, nu1=2, nu2=2)
    lv = sol.finest
    F = oc.make_consistent(oc.seeded(4 * lv.size, 5), lv.n_slots, lv.n_scalar, lv.grid_x, lv.n_pressure,
                           lv.n_pressure // 3, 3, 4)
    Xs = torch.zeros(4 * lv.size, dtype=torch.float64, device="cuda")
    sol.time_march(torch.from_numpy(F).cuda(), Xs)
    health = lv.step_health(Xs, 4)
    assert all(m <= 1e-10 for _, m in health)  # pressure projected mean-zero every step


def test_host_async_entry_points_queue_back_to_back(ctx, stmg, oracle):
    """stmg_vmult_host_async / stmg_smooth_step_host_async: several calls
    enqueued without synchronising (different inputs, multi-chunk) give the
    blocking results once the context is synchronised."""
    nc, r, k, n = 16, 2, 2, 9  # 3 chunks of <= 4 intervals
    lvl = stmg.Level(ctx, nc, nc, r, k, 0.125, 1.0, 1.0, stmg.SMOOTHER_CELL)
    pin = lambda a: torch.from_numpy(a).pin_memory().numpy()  # noqa: E731
    xs = [pin(oc.seeded(n * lvl.size, 91 + i)) for i in range(2)]
    bs = [pin(oc.seeded(n * lvl.size, 95 + i)) for i in range(2)]
    us = [pin(oc.seeded(n * lvl.size, 97 + i)) for i in range(2)]
    halo = pin(oc.seeded(lvl.n_velocity, 99))
    want_y = [lvl.vmult_host(x, np.empty_like(x), n, halo) for x in xs]
    want_u = [lvl.smooth_step_host(b, u.copy(), 0.8, n, halo, True) for b, u in zip(bs, us)]
    ys = [pin(np.zeros_like(x)) for x in xs]
    ua = [pin(u.copy()) for u in us]
    for i in range(2):
        lvl.vmult_host(xs[i], ys[i], n, halo, blocking=False)
        lvl.smooth_step_host(bs[i], ua[i], 0.8, n, halo, True, blocking=False)
    ctx.synchronize()
    for i in range(2):
        assert np.array_equal(ys[i], want_y[i])
        assert np.array_equal(ua[i], want_u[i])
