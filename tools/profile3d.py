#!/usr/bin/env python
"""Driver for ncu captures of the 3D kernels (C3 discretisation): a few vmult
and smoother-step launches on 32^3 cells, Q2/P1disc, DG(1), N intervals."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2502_09159_b200 as stmg  # noqa: E402

n = int(sys.argv[1]) if len(sys.argv) > 1 else 32
N = int(sys.argv[2]) if len(sys.argv) > 2 else 8
r = int(sys.argv[3]) if len(sys.argv) > 3 else 1
k = int(sys.argv[4]) if len(sys.argv) > 4 else 1
ctx = stmg.Context(0)
lvl = stmg.Level3(ctx, n, n, n, r, k, 1.0 / 64, 1.0, 1.0, stmg.SMOOTHER_CELL)
dofs = N * lvl.size
x = torch.rand(dofs, dtype=torch.float64, device="cuda")
b = torch.rand(dofs, dtype=torch.float64, device="cuda")
y = torch.empty_like(x)
halo = torch.rand(lvl.n_velocity, dtype=torch.float64, device="cuda")
for _ in range(2):
    lvl.vmult(x, y, N, halo)
    lvl.smooth_step(b, x, 0.8, N, halo, coupled=True, work=y)
torch.cuda.synchronize()
print("done", dofs)
