"""GPU tier: the built-in manufactured problem (problems.cpp:13-62) on the
device -- assemble_rhs (st_operator.cpp:423-467) and compute_errors
(harness.cpp:72-183) against the oracle, and acceptance Table 1
(tests/acceptance.cpp:383-420) end to end on the GPU:
assemble -> time_march -> errors."""
import math

import numpy as np
import pytest
import torch

import oracle_ctypes as oc

pytestmark = pytest.mark.gpu


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


@pytest.mark.parametrize("c,r,k", [(2, 1, 1), (2, 2, 2), (1, 4, 4), (3, 3, 1)])
def test_assemble_rhs_matches_oracle(ctx, stmg, c, r, k):
    sol = stmg.Solver(ctx, c, r, k, nu=0.1)
    ref = oc.OracleSolver(c, r, k, nu=0.1)
    lv = sol.finest
    tau = 1.0 / sol.n_steps
    n = 3
    F = torch.zeros(n * lv.size, dtype=torch.float64, device="cuda")
    lv.assemble_rhs(F, 0.25, n)
    Fh = host(F)
    for i in range(n):
        Fr = ref.assemble_rhs_manufactured(0.25 + i * tau)
        got = Fh[i * lv.size:(i + 1) * lv.size]
        assert np.abs(got - Fr).max() <= 1e-12 * np.abs(Fr).max(), i


@pytest.mark.parametrize("c,r,k", [(2, 1, 1), (2, 2, 2), (1, 4, 4)])
def test_compute_errors_match_oracle(ctx, stmg, c, r, k):
    sol = stmg.Solver(ctx, c, r, k, nu=0.1)
    ref = oc.OracleSolver(c, r, k, nu=0.1)
    lv = sol.finest
    X = oc.seeded(sol.n_steps * lv.size, 5) * 0.1
    got = lv.compute_errors(dev(X), 0.0, sol.n_steps)
    want = ref.manufactured_errors(X)
    for key, w in zip(["e_v_l2", "e_p_l2", "e_v_h1", "e_div", "e_v_linf"], want):
        assert abs(got[key] - w) <= 1e-11 * abs(w), (key, got[key], w)


def _gpu_manufactured_run(stmg, ctx, c, r):
    sol = stmg.Solver(ctx, c, r, -1, nu=0.1, gamma=1.0, rtol=1e-10, max_iterations=400)
    lv = sol.finest
    n = sol.n_steps
    F = torch.zeros(n * lv.size, dtype=torch.float64, device="cuda")
    lv.assemble_rhs(F, 0.0, n)
    X = torch.zeros_like(F)
    iters = sol.time_march(F, X)
    return sol, X, iters, lv.compute_errors(X, 0.0, n)


@pytest.mark.parametrize("c", [1, 2])
def test_manufactured_solve_matches_oracle(ctx, stmg, c):
    """Seeded-free end-to-end check: the GPU trajectory and its error norms
    equal the oracle's time_march of the manufactured problem (r = 2)."""
    sol, X, iters, err = _gpu_manufactured_run(stmg, ctx, c, 2)
    ref = oc.OracleSolver(c, 2, -1, nu=0.1, gamma=1.0, rtol=1e-10, maxit=400)
    Xr, itr = ref.time_march_manufactured()
    assert all(abs(a - b) <= 1 for a, b in zip(iters, itr)), (iters, itr)
    assert np.linalg.norm(host(X) - Xr) <= 1e-8 * np.linalg.norm(Xr)
    er = ref.manufactured_errors(Xr)
    assert abs(err["e_v_l2"] - er[0]) <= 1e-6 * er[0]
    assert abs(err["e_p_l2"] - er[1]) <= 1e-6 * er[1]


def test_table1_r4_on_gpu(ctx, stmg):
    """PAPER.md Table 1 (r = 4, c = 1..3): velocity and pressure L2(L2)
    errors within a factor 2 of the published values and velocity EOC within
    +-0.3 (acceptance.cpp:383-420), computed entirely on the GPU."""
    ref_v = [1.00279e-04, 2.32706e-06, 3.98114e-08]
    ref_p = [1.14907e-03, 1.11534e-04, 3.58645e-06]
    ref_eoc = [5.43, 5.87]
    ev, ep = [], []
    for c in (1, 2, 3):
        _, _, iters, err = _gpu_manufactured_run(stmg, ctx, c, 4)
        ev.append(err["e_v_l2"])
        ep.append(err["e_p_l2"])
        print(f"Table 1 GPU c={c}: e_v={err['e_v_l2']:.4e} e_p={err['e_p_l2']:.4e} "
              f"avg iters={sum(iters) / len(iters):.2f}")
        assert 0.5 < ev[-1] / ref_v[c - 1] < 2.0
        assert 0.5 < ep[-1] / ref_p[c - 1] < 2.0
    for i in (1, 2):
        assert abs(math.log2(ev[i - 1] / ev[i]) - ref_eoc[i - 1]) <= 0.3


@pytest.mark.parametrize("c,r,k", [(2, 1, 1), (2, 2, 2), (1, 4, 4)])
def test_interpolate_exact_matches_oracle(ctx, stmg, c, r, k):
    """interpolate_exact (harness.cpp:185-239) on the GPU equals the oracle's,
    and its error norms are the interpolation errors the oracle reports."""
    sol = stmg.Solver(ctx, c, r, k, nu=0.1)
    ref = oc.OracleSolver(c, r, k, nu=0.1)
    lv = sol.finest
    n = sol.n_steps
    X = torch.zeros(n * lv.size, dtype=torch.float64, device="cuda")
    lv.interpolate_exact(X, 0.0, n)
    Xr = ref.interpolate_manufactured()
    Xh = host(X)
    assert np.abs(Xh - Xr).max() <= 1e-13 * np.abs(Xr).max()
    got = lv.compute_errors(X, 0.0, n)
    want = ref.manufactured_errors(Xr)
    assert abs(got["e_v_l2"] - want[0]) <= 1e-9 * want[0]
    assert abs(got["e_p_l2"] - want[1]) <= 1e-9 * want[1]


@pytest.mark.parametrize("c,r,k,nu", [(2, 2, 2, 0.1), (3, 1, 1, 0.05)])
def test_cavity_time_march_with_lift_matches_oracle(ctx, stmg, c, r, k, nu):
    """time_march with inhomogeneous Dirichlet data (solver.cpp:251-283): the
    lid-driven cavity (problems.cpp:64-78) lifted on the GPU reproduces the
    oracle's trajectory; iterations within +-1."""
    n_steps = 4
    sol = stmg.Solver(ctx, c, r, k, n_steps=n_steps, t_end=8.0 * n_steps / 32, nu=nu, rtol=1e-10)
    ref = oc.OracleSolver(c, r, k, n_steps=n_steps, t_end=8.0 * n_steps / 32, nu=nu, rtol=1e-10)
    X = torch.zeros(n_steps * sol.finest.size, dtype=torch.float64, device="cuda")
    iters = sol.time_march_problem(stmg.PROBLEM_CAVITY, X)
    Xr, itr = ref.time_march_cavity()
    assert all(abs(a - b) <= 1 for a, b in zip(iters, itr)), (iters, itr)
    assert np.linalg.norm(Xr) > 0
    assert np.linalg.norm(host(X) - Xr) <= 1e-8 * np.linalg.norm(Xr)


def test_time_march_problem_manufactured_equals_assembled_path(ctx, stmg):
    sol = stmg.Solver(ctx, 2, 2, 2, nu=0.1, rtol=1e-10)
    lv = sol.finest
    n = sol.n_steps
    F = torch.zeros(n * lv.size, dtype=torch.float64, device="cuda")
    lv.assemble_rhs(F, 0.0, n)
    X1 = torch.zeros_like(F)
    it1 = sol.time_march(F, X1)
    X2 = torch.zeros_like(F)
    it2 = sol.time_march_problem(stmg.PROBLEM_MANUFACTURED, X2)
    assert it1 == it2
    assert float((X1 - X2).abs().max()) <= 1e-12 * float(X1.abs().max())


def _radau_right(n):
    """Right Gauss-Radau points on [-1, 1] (n points, +1 included): the
    mirror of the left rule, whose points are the roots of P_{n-1} + P_n."""
    c = np.zeros(n + 1)
    c[n - 1] = 1.0
    c[n] = 1.0
    return np.sort(-np.real(np.polynomial.legendre.legroots(c)))


def test_time_march_lifted_general_boundary_data(ctx, stmg):
    """General Dirichlet data through per-step lift vectors: the cavity lid
    written by the caller (set_boundary_values semantics, dof_space.cpp:71-81)
    reproduces the built-in cavity time march."""
    n_steps, k = 3, 2
    sol = stmg.Solver(ctx, 2, 2, k, n_steps=n_steps, t_end=0.75, nu=0.1, rtol=1e-10)
    lv = sol.finest
    X_ref = torch.zeros(n_steps * lv.size, dtype=torch.float64, device="cuda")
    it_ref = sol.time_march_problem(stmg.PROBLEM_CAVITY, X_ref)
    gx, gy, mv = lv.grid_x, lv.n_scalar // lv.grid_x, lv.n_velocity
    tau = 0.75 / n_steps
    lifts = np.zeros(n_steps * lv.size)
    for n in range(n_steps):
        for a, xi in enumerate(_radau_right(k + 1)):
            t = n * tau + 0.5 * tau * (xi + 1.0)
            base = n * lv.size + a * mv + (gy - 1) * gx  # top grid row, component 0
            lifts[base + 1: base + gx - 1] = math.sin(0.25 * math.pi * t)
    X = torch.zeros_like(X_ref)
    it = sol.time_march_ex(X, lifts=dev(lifts))
    assert it == it_ref
    assert float((X - X_ref).abs().max()) <= 1e-12 * float(X_ref.abs().max())


def test_time_march_initial_velocity_is_the_first_coupling(ctx, stmg):
    """An initial velocity v0 (solver.cpp:229-236) enters step 1 through the
    coupling: time_march_ex(v_init = v0) equals time_march with the load
    F_1 += coupling_rhs(v0) and zero initial data."""
    n_steps = 3
    sol = stmg.Solver(ctx, 3, 1, 1, n_steps=n_steps, nu=0.5, rtol=1e-11)
    lv = sol.finest
    g = torch.Generator(device="cuda")
    g.manual_seed(3)
    v0 = torch.rand(lv.n_velocity, dtype=torch.float64, device="cuda", generator=g)
    X1 = torch.zeros(n_steps * lv.size, dtype=torch.float64, device="cuda")
    it1 = sol.time_march_ex(X1, v_init=v0)
    F = torch.zeros_like(X1)
    lv.coupling_rhs(v0, F[:lv.size])
    X2 = torch.zeros_like(X1)
    it2 = sol.time_march(F, X2)
    assert it1 == it2
    assert float((X1 - X2).abs().max()) <= 1e-12 * float(X2.abs().max())
