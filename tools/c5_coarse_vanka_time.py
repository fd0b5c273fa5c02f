"""Time one Vanka sweep (8 colours, 16 intervals) on the deformed r = 1, k = 2 levels of the C5
hierarchy (n_T = 255: time-diagonalised blocks of 85 / 170 rows). Usage: python tools/c5_coarse_vanka_time.py"""
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import bench3d  # noqa: E402
import paper_2502_09159_b200 as stmg  # noqa: E402

ctx = stmg.Context(0)
N = 16
for n in (32, 16, 8):
    verts = np.ascontiguousarray(np.asarray(bench3d.c5_vertices(32)).reshape(33, 33, 33, 3)[::32 // n, ::32 // n, ::32 // n].reshape(-1))
    lvl = stmg.Level3(ctx, n, n, n, 1, 2, 1.0 / 128, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=verts)
    r = bench3d.seeded(torch, N * lvl.size, 1)
    u = torch.zeros_like(r)
    ms = bench3d.timed(torch, lambda: lvl.vanka_update(r, u, 0.8, N), 5)
    ps = lvl.patch_setup
    print(f"{n}^3 r=1 k=2: sweep {ms:.3f} ms, max n_T {lvl.max_patch}, factored={ps['factored']}, "
          f"streamed {8 * ps['streamed_elements'] / 1e9:.2f} GB")
