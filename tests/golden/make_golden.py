#!/usr/bin/env python
"""Generates the committed golden vectors of the hot path (tests/golden/*.npz).

The reference (/root/reference/proj) needs Eigen, which this image does not
have, so it cannot be run here; the vectors come from oracle/ (its C++
restatement, pinned to the reference's known-answer tests and PAPER Table 1,
oracle/tests/oracle_tests.cpp). They freeze today's oracle outputs: the CPU
tier checks that the oracle still reproduces them (tests/test_cpu_golden.py),
the GPU tier checks the CUDA path against them through the C ABI
(tests/test_gpu_golden.py). Inputs are stored next to the outputs, so the
files do not depend on a random-number stream.

    python tests/golden/make_golden.py        # rewrites tests/golden/*.npz
"""
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parent))

import oracle3_ctypes as o3  # noqa: E402
import oracle_ctypes as oc  # noqa: E402

# name: (nc, r, k, tau, nu, gamma, smoother kind, intervals)
CASES_2D = {
    "c1_q2p1_dg1_cell": (8, 1, 1, 0.125, 1.0, 1.0, 0, 2),        # C1 discretisation
    "c2_q3p2_dg2_cell": (4, 2, 2, 1.0 / 64, 1.0, 1.0, 0, 2),     # C2 discretisation
    "c4_q2p1_dg1_vertex_star": (8, 1, 1, 1.0 / 64, 1.0, 1.0, 1, 2),  # C4 discretisation
    "q4p3_dg3_gamma0": (2, 3, 3, 0.25, 0.1, 0.0, 0, 1),
}
# name: (nx, ny, nz, r, k, tau, gamma, amp, intervals)
CASES_3D = {
    "c3_q2p1_dg1_cartesian": (3, 2, 2, 1, 1, 0.125, 1.0, 0.0, 2),  # C3 discretisation
    "c5_q3p2_dg2_deformed": (2, 2, 2, 2, 2, 0.125, 1.0, 0.1, 1),   # C5 discretisation
}
# FGMRES + hp-STMG V(2,2) solve of the C1 discretisation on 8 x 8 cells
SOLVE = dict(refinements=3, r=1, k=1, n_steps=8, nu=1.0, gamma=1.0, nu1=2, nu2=2)
OMEGA = 0.8


def make_2d(name, case):
    nc, r, k, tau, nu, gamma, kind, n = case
    ref = oc.OracleLevel(nc, r, k, tau, nu, gamma, kind)
    rng = np.random.default_rng(sum(map(ord, name)))
    x = rng.uniform(-1, 1, n * ref.size)
    b = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.n_velocity)
    y = ref.vmult_all(x, n, halo)
    u = ref.smooth_step_all(b, x, OMEGA, n, halo)
    z = ref.apply_additive(b[:ref.size])
    np.savez(HERE / f"{name}.npz", case=np.array(case, dtype=np.float64), x=x, b=b, halo=halo, vmult=y,
             smooth_step=u, apply_additive=z)


def make_3d(name, case):
    nx, ny, nz, r, k, tau, gamma, amp, n = case
    verts = o3.vertices(nx, ny, nz, amp, seed=11) if amp else None
    ref = o3.OracleLevel3(nx, ny, nz, r, k, tau, 1.0, gamma, vertices=verts)
    rng = np.random.default_rng(sum(map(ord, name)))
    x = rng.uniform(-1, 1, n * ref.size)
    b = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.mv)
    y = ref.vmult_all(x, n, halo)
    u = ref.smooth_step_all(b, x, OMEGA, n, halo)
    np.savez(HERE / f"{name}.npz", case=np.array(case, dtype=np.float64),
             vertices=verts if verts is not None else np.zeros(0), x=x, b=b, halo=halo, vmult=y, smooth_step=u)


def make_solve():
    rs = oc.OracleSolver(SOLVE["refinements"], SOLVE["r"], SOLVE["k"], n_steps=SOLVE["n_steps"], nu=SOLVE["nu"],
                         gamma=SOLVE["gamma"], nu1=SOLVE["nu1"], nu2=SOLVE["nu2"])
    nc = 2 ** SOLVE["refinements"]
    lv = oc.OracleLevel(nc, SOLVE["r"], SOLVE["k"], 1.0 / SOLVE["n_steps"], SOLVE["nu"], SOLVE["gamma"], 0,
                        build_smoother=False)
    S, npc = SOLVE["k"] + 1, (SOLVE["r"] + 1) * (SOLVE["r"] + 2) // 2
    gx = nc * (SOLVE["r"] + 1) + 1
    rhs = oc.make_consistent(np.random.default_rng(77).uniform(-1, 1, lv.size), S, gx * gx, gx, nc * nc * npc, nc * nc,
                             npc)
    x, its, _ = rs.gmres(rhs)
    np.savez(HERE / "c1_fgmres_stmg_v22.npz", rhs=rhs, solution=x, iterations=np.array([its]))


if __name__ == "__main__":
    oc.build_oracle()
    for nm, cs in CASES_2D.items():
        make_2d(nm, cs)
    for nm, cs in CASES_3D.items():
        make_3d(nm, cs)
    make_solve()
    for f in sorted(HERE.glob("*.npz")):
        print(f.name, f.stat().st_size)
