"""Time the all-at-once vmult and residual alone (CUDA events), for kernel
experiments. Usage: [STMG_LIB=...] python tools/vmult_time.py [--nx 256] [--r 2] [--k 2] [--intervals 64]"""
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
ap.add_argument("--reps", type=int, default=10)
ap.add_argument("--tag", default="")
a = ap.parse_args()
ctx = stmg.Context(0)
lvl = stmg.Level(ctx, a.nx, a.nx, a.r, a.k, 1.0 / 64, 1.0, 1.0, stmg.SMOOTHER_NONE)
n = a.intervals * lvl.size
x = torch.rand(n, dtype=torch.float64, device="cuda")
b = torch.rand(n, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
halo = torch.rand(lvl.n_velocity, dtype=torch.float64, device="cuda")
out = []
for name, fn in (("vmult", lambda: lvl.vmult(x, y, a.intervals, halo)),
                 ("residual", lambda: lvl.residual(b, x, y, a.intervals, halo))):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    out.append(f"{name} {s.elapsed_time(e) / a.reps:.3f} ms")
print(a.tag, " ".join(out), f"checksum {float(y.double().sum()):.12e}")
