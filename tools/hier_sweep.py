"""FGMRES iterations of the 3D all-at-once solve for hierarchy / smoother
variants (C3 discretisation: Q2/P1disc, DG(1); Cartesian), to study the
BASELINE C3 plan (k 1 -> 0, then h in space AND time).
Usage: python tools/hier_sweep.py"""
import itertools
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench3d  # noqa: E402
import paper_2502_09159_b200 as stmg  # noqa: E402

ctx = stmg.Context(0)
out = []
for n, omega, (tc, kmin, nh), nu12 in itertools.product(
        [8, 16], [0.8, 0.6, 0.5, 0.4], [(True, 0, None), (False, 1, None)], [2, 3]):
    N = 2 * n  # tau = 1/(2n): lambda = tau/h^2 = n/2
    nh_ = nh if nh is not None else (2 if n == 8 else 3)  # coarse 2^3 x N/4 (8^3) / 2^3 x N/8 (16^3)
    try:
        sol = stmg.Solver3(ctx, n, n, n, 1, 1, 1.0 / N, 1.0, 1.0, n_hcoarse=nh_, time_coarsen=tc, k_min=kmin,
                           nu1=nu12, nu2=nu12, omega=omega, rtol=1e-8, max_iterations=150)
        f = sol.finest
        F = bench3d.consistent(torch, f, bench3d.seeded(torch, N * f.size, 5), N)
        X = torch.zeros_like(F)
        it, hist = sol.solve_all_at_once(F, X, N)
        rec = dict(n=n, N=N, omega=omega, time_coarsen=tc, k_min=kmin, n_hcoarse=nh_, nu=nu12, iterations=it)
    except Exception as exc:  # noqa: BLE001
        rec = dict(n=n, N=N, omega=omega, time_coarsen=tc, k_min=kmin, n_hcoarse=nh_, nu=nu12,
                   error=str(exc)[:120])
    out.append(rec)
    print(json.dumps(rec), flush=True)
    del sol
    torch.cuda.empty_cache()
