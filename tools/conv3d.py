#!/usr/bin/env python
"""FGMRES iteration counts of the 3D all-at-once hp-STMG for several
hierarchy / smoother settings (one B200). Prints one line per case.

Each argument: nx,r,k,N,n_hcoarse,amp,k_min,affine_patches,omega
"""
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

import bench3d  # noqa: E402
import paper_2502_09159_b200 as stmg  # noqa: E402

ctx = stmg.Context(0)
for arg in sys.argv[1:]:
    f_ = arg.split(",")
    nx, r, k, N, nh = (int(v) for v in f_[:5])
    amp, kmin, aff, omega = float(f_[5]), int(f_[6]), int(f_[7]), float(f_[8])
    verts = bench3d.c5_vertices(nx) if amp > 0 else None
    t0 = time.time()
    sol = stmg.Solver3(ctx, nx, nx, nx, r, k, 1.0 / 64, 1.0, 1.0, n_hcoarse=nh, time_coarsen=False, k_min=kmin,
                       vertices=verts, affine_patches=bool(aff), omega=omega, rtol=1e-8, max_iterations=300)
    f = sol.finest
    F = bench3d.consistent(torch, f, bench3d.seeded(torch, N * f.size, 7), N)
    X = torch.zeros_like(F)
    t1 = time.time()
    try:
        it, hist = sol.solve_all_at_once(F, X, N)
    except Exception as exc:
        it = str(exc)[:60]
    torch.cuda.synchronize()
    print(f"nx={nx} r={r} k={k} N={N} nh={nh} amp={amp} kmin={kmin} affine={aff} omega={omega} "
          f"levels={[(l['nx'], l['r'], l['k']) for l in sol.level_info]} its={it} setup={t1 - t0:.1f}s "
          f"solve={time.time() - t1:.1f}s", flush=True)
    del sol, F, X
