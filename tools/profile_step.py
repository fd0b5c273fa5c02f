"""One C2 step (vmult + residual + Vanka update) for ncu captures.
Usage: python tools/profile_step.py [--nx 256] [--intervals 64] [--reps 2]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2502_09159_b200 as stmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=256)
ap.add_argument("--intervals", type=int, default=64)
ap.add_argument("--r", type=int, default=2)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--reps", type=int, default=2)
ap.add_argument("--kind", type=int, default=0, help="0 cell Vanka, 1 vertex-star Vanka")
a = ap.parse_args()
ctx = stmg.Context(0)
lvl = stmg.Level(ctx, a.nx, a.nx, a.r, a.k, 1.0 / 64, 1.0, 1.0, a.kind)
n = a.intervals * lvl.size
x = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.rand_like(x)
u = torch.rand_like(x)
y = torch.empty_like(x)
res = torch.empty_like(x)
halo = torch.zeros(lvl.n_velocity, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    lvl.vmult(x, y, a.intervals, halo)
    lvl.residual(b, u, res, a.intervals, halo, coupled=True)
    lvl.vanka_update(res, u, 0.8, a.intervals)
torch.cuda.synchronize()
print("ok", ctx.launch_count())
