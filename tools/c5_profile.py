#!/usr/bin/env python
"""Driver for ncu launch lists of the C5 solve: the 32^3 deformed Q3/P2disc
DG(2) hierarchy of the bench (exact GPU-built patches, k kept, h in space to
2^3) and ONE all-at-once FGMRES solve of a slab of N intervals.
Usage: python tools/c5_profile.py [N=16] [n=32]"""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import torch  # noqa: E402

import bench3d  # noqa: E402
import paper_2502_09159_b200 as stmg  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 16
n = int(sys.argv[2]) if len(sys.argv) > 2 else 32
ctx = stmg.Context(0)
sol = stmg.Solver3(ctx, n, n, n, 2, 2, 1.0 / 128, 1.0, 1.0, n_hcoarse=4, time_coarsen=False, k_min=2,
                   vertices=bench3d.c5_vertices(n), nu1=2, nu2=2, rtol=1e-8)
f = sol.finest
F = bench3d.consistent(torch, f, bench3d.seeded(torch, N * f.size, 500), N)
X = torch.zeros_like(F)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
it, hist = sol.solve_all_at_once(F, X, N)
e.record()
torch.cuda.synchronize()
print(f"C5 slab of {N} intervals: {it} iterations, {s.elapsed_time(e):.1f} ms, launches {ctx.launch_count()}")
