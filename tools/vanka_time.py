"""Time the C2 Vanka update alone (CUDA events), for kernel experiments.
Usage: [STMG_LIB=...] python tools/vanka_time.py [--reps 10] [--kind 0] [--nx 256] [--r 2] [--k 2] [--intervals 64]"""
import argparse
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2502_09159_b200 as stmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--nx", type=int, default=256)
ap.add_argument("--r", type=int, default=2)
ap.add_argument("--k", type=int, default=2)
ap.add_argument("--intervals", type=int, default=64)
ap.add_argument("--kind", type=int, default=0)
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tag", default="")
a = ap.parse_args()
ctx = stmg.Context(0)
lvl = stmg.Level(ctx, a.nx, a.nx, a.r, a.k, 1.0 / 64, 1.0, 1.0, a.kind)
n = a.intervals * lvl.size
res = torch.rand(n, dtype=torch.float64, device="cuda")
u = torch.rand(n, dtype=torch.float64, device="cuda")
for _ in range(3):
    lvl.vanka_update(res, u, 0.8, a.intervals)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(a.reps):
    lvl.vanka_update(res, u, 0.8, a.intervals)
e.record()
torch.cuda.synchronize()
ms = s.elapsed_time(e) / a.reps
flops = 2.0 * lvl.total_matrix_elements * a.intervals
print(f"{a.tag} vanka_update {ms:.3f} ms  {flops / ms / 1e9:.2f} TF/s")
