"""Kernel-time breakdown of one all-at-once C4 slab solve (torch.profiler / CUPTI,
no replay). Usage: python tools/solve_profile.py [--refinements 10] [--slab 8]"""
import argparse
import collections
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2502_09159_b200 as stmg  # noqa: E402
import bench  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--refinements", type=int, default=10)
ap.add_argument("--slab", type=int, default=8)
a = ap.parse_args()
ctx = stmg.Context(0)
sol = stmg.Solver(ctx, a.refinements, 1, 1, n_steps=a.slab, t_end=a.slab / 64.0, nu=1.0, gamma=1.0,
                  smoother=stmg.SMOOTHER_VERTEX_STAR, nu1=2, nu2=2, omega=0.8, rtol=1e-8)
F = bench._consistent_rhs(torch, sol, a.slab, 101)
X = torch.zeros_like(F)
sol.solve_all_at_once(F, X, a.slab)
torch.cuda.synchronize()
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    it, _ = sol.solve_all_at_once(F, X, a.slab)
    torch.cuda.synchronize()
agg = collections.defaultdict(lambda: [0, 0.0])
for e in prof.events():
    if e.device_type == torch.autograd.DeviceType.CUDA:
        name = e.name.replace("(anonymous namespace)::", "").split("(")[0].replace("void ", "")[:70]
        agg[name][0] += 1
        agg[name][1] += e.device_time_total / 1e3 if hasattr(e, "device_time_total") else e.cuda_time_total / 1e3
tot = sum(v[1] for v in agg.values())
print(f"iterations {it}, kernels {sum(v[0] for v in agg.values())}, kernel ms {tot:.1f}")
for k, (n, ms) in sorted(agg.items(), key=lambda kv: -kv[1][1])[:16]:
    print(f"{k:72s} {n:6d} {ms:9.2f} ms {100 * ms / tot:5.1f}%")
