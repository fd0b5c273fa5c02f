"""Time-marching FGMRES + hp-STMG solve throughput on the GPU.

python tools/solve_bench.py --refinements 10 --r 1 --k 1 --steps 4 --smoother 1
Prints one JSON line: dofs, seconds, DoF/s, iterations per step.
"""
import argparse
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2502_09159_b200 as stmg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--refinements", type=int, default=4)
ap.add_argument("--r", type=int, default=1)
ap.add_argument("--k", type=int, default=1)
ap.add_argument("--steps", type=int, default=8, help="time steps solved (n_steps of the hierarchy)")
ap.add_argument("--total-steps", type=int, default=0, help="tau = 1/total_steps (default: steps)")
ap.add_argument("--smoother", type=int, default=0)
ap.add_argument("--nu", type=float, default=1.0)
ap.add_argument("--nu1", type=int, default=2)
ap.add_argument("--nu2", type=int, default=2)
ap.add_argument("--rtol", type=float, default=1e-8)
a = ap.parse_args()
total = a.total_steps or a.steps
t0 = time.perf_counter()
ctx = stmg.Context(0)
sol = stmg.Solver(ctx, a.refinements, a.r, a.k, n_steps=a.steps, t_end=a.steps / total, nu=a.nu, gamma=1.0,
                  smoother=a.smoother, nu1=a.nu1, nu2=a.nu2, rtol=a.rtol)
torch.cuda.synchronize()
setup_s = time.perf_counter() - t0
lv = sol.finest
n = sol.n_steps * lv.size
gen = torch.Generator(device="cuda")
gen.manual_seed(7)
F = torch.rand(n, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
# consistent RHS: zero constrained velocity, mean-zero pressure per slot
gx, gy = lv.grid_x, lv.n_scalar // lv.grid_x
Fv = F.view(sol.n_steps, lv.size)
for a_ in range(lv.n_slots):
    for c in range(2):
        base = a_ * lv.n_velocity + c * lv.n_scalar
        g = Fv[:, base: base + lv.n_scalar].view(sol.n_steps, gy, gx)
        g[:, 0, :] = 0
        g[:, -1, :] = 0
        g[:, :, 0] = 0
        g[:, :, -1] = 0
    npc = (sol.level_info[-1]["r"] + 1) * (sol.level_info[-1]["r"] + 2) // 2
    pb = lv.n_slots * lv.n_velocity + a_ * lv.n_pressure
    p = Fv[:, pb: pb + lv.n_pressure].view(sol.n_steps, -1, npc)
    p[:, :, 0] -= p[:, :, 0].mean(dim=1, keepdim=True)
X = torch.zeros_like(F)
iters = sol.time_march(F, X)  # warm-up (also builds Krylov workspace)
torch.cuda.synchronize()
launches0 = ctx.launch_count()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
iters = sol.time_march(F, X)
e.record()
torch.cuda.synchronize()
sec = s.elapsed_time(e) / 1e3
print(json.dumps({"levels": sol.level_info, "n_steps": sol.n_steps, "dofs": n, "seconds": sec,
                  "dofs_per_s": n / sec, "iterations": iters, "avg_iterations": sum(iters) / len(iters),
                  "setup_s": setup_s, "kernels": ctx.launch_count() - launches0}))
