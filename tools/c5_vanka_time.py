"""Time one C5 fine-level Vanka sweep (8 colours) on 16 intervals: 32^3
deformed Q3/P2disc DG(2) with the exact GPU-built patches.
Usage: [STMG_LIB=...] [STMG_VANKA3_DENSE=1] python tools/c5_vanka_time.py [n=32] [N=16]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench3d  # noqa: E402
import paper_2502_09159_b200 as stmg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 16
ctx = stmg.Context(0)
lvl = stmg.Level3(ctx, n, n, n, 2, 2, 1.0 / 128, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=bench3d.c5_vertices(n))
r = bench3d.seeded(torch, N * lvl.size, 1)
u = torch.zeros_like(r)
ms = bench3d.timed(torch, lambda: lvl.vanka_update(r, u, 0.8, N), 3)
ps = lvl.patch_setup
print(f"C5 Vanka sweep {N} intervals: {ms:.2f} ms (factored={ps['factored']}, setup {ps['seconds']:.2f} s)")
