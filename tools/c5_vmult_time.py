"""Time the C5 vmult (32^3 deformed Q3/P2disc DG(2), 128 intervals) alone.
Usage: [STMG_LIB=...] python tools/c5_vmult_time.py [n=32] [N=128] [reps=5]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench3d  # noqa: E402
import paper_2502_09159_b200 as stmg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 128
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
ctx = stmg.Context(0)
lvl = stmg.Level3(ctx, n, n, n, 2, 2, 1.0 / N, 1.0, 1.0, stmg.SMOOTHER_NONE, vertices=bench3d.c5_vertices(n))
x = bench3d.seeded(torch, N * lvl.size, 1)
y = torch.empty_like(x)
halo = bench3d.seeded(torch, lvl.n_velocity, 3)
ms = bench3d.timed(torch, lambda: lvl.vmult(x, y, N, halo), reps)
print(f"C5 vmult {ms:.2f} ms  {N * lvl.size / ms / 1e6:.3e} DoF/s  checksum {float(y.sum()):.10e}")
