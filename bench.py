#!/usr/bin/env python
"""Benchmark of the B200 hp-STMG hot path (BASELINE.json configs[1], "C2").

Workload (one step): the all-at-once space-time operator vmult plus one cell
Vanka smoother step, over the full C2 system: 2D Stokes, Q3/P2disc (r=2),
DG(2), Cartesian 256x256 mesh, 64 intervals on [0,1], nu=1, gamma=1, FP64,
3.03e8 space-time dofs per GPU, seeded uniform[-1,1] inputs resident in HBM.
Local Vanka inverses are precomputed once and shared by all intervals.

  value   = space-time dofs processed per second by the whole job
            (n_gpus * dofs_per_gpu / ms_per_step), step = vmult + smoother step
  e2e     = the same step through the host-buffer C-ABI entry points
            (stmg_vmult_host + stmg_smooth_step_host), H2D/D2H inside
  --gpus N: one process per GPU (torchrun), time slabs of 64 intervals per
            rank (weak scaling); the DG jump couples rank p to p-1 through the
            slot-k velocity halo, exchanged with NCCL send/recv every vmult
            and smoother residual.
  --impl reference: the CPU restatement of the reference (oracle/, OpenMP over
            intervals on all host cores) on a bounded sample of the same
            discretisation; rank 0 only.

Extra fields of the JSON line (not the headline; skipped with --no-solve):
  solve.C1             FGMRES + V(2,2) time marching of C1 (16^2, Q2/P1, DG(1))
  solve.C4_first2      time marching of the C4 discretisation, first 2 intervals
  solve.C4_all_at_once all-at-once slab solve of C4, 8 intervals per rank,
                       partitioned over all ranks (NCCL time slabs)
  solve.C4_full        (1 GPU) the whole 64-interval C4 system as 8 macro steps
  solve.C3_all_at_once the 64-interval C3 system (32^3, Q2/P1disc, DG(1))
                       split into time slabs over all ranks (NCCL)
  solve.C5_hybrid      (N >= 4, even) the whole 128-interval C5 system as one
                       all-at-once solve, hybrid 2 z parts x N/2 time slabs
  C4_step              C4 vmult + vertex-star smoother step over 8 intervals
  3D.C3                (1 GPU) C3: 32^3 Q2/P1disc, DG(1), 64 intervals: vmult,
                       cell-Vanka step, full all-at-once solve (tools/bench3d.py)
  3D.C5                (1 GPU) C5: 32^3 deformed Q3/P2disc, DG(2), 128 intervals: vmult
                       and the full solve as 8 macro steps of 16 intervals
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIG = dict(workload="C2: all-at-once vmult + cell-Vanka smoother step", mesh="256x256", r=2, k=2,
              intervals_per_gpu=64, nu=1.0, gamma=1.0, omega=0.8, domain="unit square x (0,1]")
METRIC = "space-time DoF/s: matrix-free vmult, Vanka step, full hp-STMG solve"
UNIT = "DoF/s"


def peaks():
    """HBM GB/s (MEASURED_PEAKS.json) and the measured FP64 peaks of this pool's
    B200: DFMA (CUDA-core pipe) and DMMA (FP64 tensor path), TF/s."""
    hbm, fp64, dmma, src = 6443.2, 36.77, 37.13, []
    try:
        mp = json.loads((ROOT / "MEASURED_PEAKS.json").read_text())
        hbm = float(mp["hbm_gbs"])
        src.append("MEASURED_PEAKS.json hbm_gbs")
    except Exception:
        src.append("fallback hbm 6443")
    for f in sorted((ROOT / "profiles").glob("fp64_peaks_r*.json")):
        try:
            rec = json.loads(f.read_text().strip().splitlines()[0])
            fp64, dmma = float(rec["dfma_tflops"]), float(rec["dmma_tflops"])
            src.append(f"{f.name} dfma_tflops/dmma_tflops")
        except Exception:
            pass
    return hbm, fp64, dmma, ", ".join(src)


def vmult_fma_per_cell(r, k, coupled=True):
    """FMAs of the fused vmult kernel per cell and interval (all output slots),
    excluding the 1/31 + 1/rows halo recompute (see vmult_impl.cuh)."""
    N1, NP, PL, S = r + 2, (r + 1) * (r + 2) // 2, r + 1, k + 1
    per_slot = S * NP + 2 * N1 * NP + 2 * PL * N1 * N1 + N1 * (
        4 * S * N1 + (2 * N1 if coupled else 0) + 8 * N1 * N1 + 6 * N1 * N1 + 2 * PL * N1 + 2 * NP)
    return per_slot * S


class ClockSampler:
    """nvidia-smi clocks / throttle reasons during the timed region."""

    def __init__(self, index=0):
        self.index, self.samples, self.proc = index, [], None

    def __enter__(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", "-i", str(self.index), f"--query-gpu={q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.thread = threading.Thread(target=self._read, daemon=True)
            self.thread.start()
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.samples.append(parts)

    def __exit__(self, *a):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except Exception:
                self.proc.kill()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        sm = [float(s[0]) for s in self.samples if s[0].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for s in self.samples for i in range(4) if s[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": float(self.samples[0][1]) if self.samples[0][1].replace(".", "").isdigit() else None,
                "power_w_max": max(float(s[2]) for s in self.samples if s[2].replace(".", "").isdigit()),
                "reasons": reasons, "samples": len(self.samples)}


# ---------------------------------------------------------------- reference arm
def host_cpu():
    """Host core count as the box reports it (lscpu), for the baselines."""
    info = {"logical_cpus": os.cpu_count()}
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        for line in out.splitlines():
            k, _, v = line.partition(":")
            k, v = k.strip(), v.strip()
            if k in ("Model name", "Socket(s)", "Core(s) per socket", "Thread(s) per core"):
                info[k] = v
        if "Socket(s)" in info and "Core(s) per socket" in info:
            info["physical_cores"] = int(info["Socket(s)"]) * int(info["Core(s) per socket"])
    except Exception:
        pass
    return info


def cpu_sample():
    """The one bounded CPU sample both arms time: the C2 discretisation (Q3/P2disc,
    DG(2), nu = gamma = 1, tau = 1/64) on 64^2 cells, one interval per host
    thread (the oracle parallelises over intervals with OpenMP, so every
    thread has an interval), vmult + cell-Vanka step per step."""
    threads = os.cpu_count() or 1
    return {"nc": 64, "n_int": max(threads, 1), "threads": threads}


def time_oracle(threads, n_int, steps, warmup, nc=64):
    """DoF/s of the oracle (C++ restatement of the reference, -O3) on one step
    = all-at-once vmult + one Vanka smoother step over n_int intervals."""
    sys.path.insert(0, str(ROOT / "tests"))
    import oracle_ctypes as oc

    lvl = oc.OracleLevel(nc, CONFIG["r"], CONFIG["k"], 1.0 / 64, CONFIG["nu"], CONFIG["gamma"], 0)
    dofs = n_int * lvl.size
    x = oc.seeded(dofs, 1)
    b = oc.seeded(dofs, 2)
    halo = oc.seeded(lvl.n_velocity, 3)
    u = x.copy()
    for _ in range(warmup):
        lvl.vmult_all(x, n_int, halo, threads)
        u = lvl.smooth_step_all(b, u, CONFIG["omega"], n_int, halo, threads)
    t0 = time.perf_counter()
    for _ in range(steps):
        lvl.vmult_all(x, n_int, halo, threads)
        u = lvl.smooth_step_all(b, u, CONFIG["omega"], n_int, halo, threads)
    dt = (time.perf_counter() - t0) / steps
    return dofs / dt, dt, dofs


def _sample_text(smp, threads, n_int, steps):
    return (f"oracle port of the reference (C++ restatement, -O3, OpenMP over intervals) on {smp['nc']}x{smp['nc']} "
            f"cells, r=2, k=2, tau=1/64, {n_int} intervals, {threads} thread(s) busy, vmult + Vanka step, "
            f"{steps} timed steps; per-dof rate of the C2 workload (intervals are independent work)")


def arm_config(world, dofs_per_gpu=None, nx=256, N=64):
    """The workload config, identical in both arms."""
    return dict(CONFIG, mesh=f"{nx}x{nx}", intervals_per_gpu=N,
                dofs_per_gpu=dofs_per_gpu if dofs_per_gpu is not None else N * c2_interval_size(nx),
                parallelism=f"time-slab dp{world}" if world > 1 else "single GPU",
                l2="inputs 2.4 GB per vector >> 126 MB L2 (no flush needed)")


def c2_interval_size(nx, r=2, k=2):
    g = nx * (r + 1) + 1
    return (k + 1) * (2 * g * g + nx * nx * (r + 1) * (r + 2) // 2)


def run_reference(args):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    smp = cpu_sample()
    threads, n_int = smp["threads"], smp["n_int"]
    value, dt, dofs = time_oracle(threads, n_int, args.steps, args.warmup, smp["nc"])
    one, _, _ = time_oracle(1, 1, 2, 1, smp["nc"])
    line = {"impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1])",
            "config": arm_config(args.gpus, nx=args.nx, N=args.intervals),
            "cpu_baseline": {"value": value, "unit": UNIT, "cores": min(threads, n_int), "kind": "port",
                             "sample": _sample_text(smp, min(threads, n_int), n_int, args.steps)},
            "cpu_baseline_1core": {"value": one, "unit": UNIT, "cores": 1, "kind": "port",
                                   "sample": _sample_text(smp, 1, 1, 2)},
            "host": host_cpu(),
            "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def cpu_baseline_quick():
    """The reference arm's sample (same mesh, intervals and threads), fewer
    steps, for the cpu_baseline field of our own line; plus the 1-core rate."""
    smp = cpu_sample()
    threads, n_int = smp["threads"], smp["n_int"]
    value, _, _ = time_oracle(threads, n_int, 2, 1, smp["nc"])
    one, _, _ = time_oracle(1, 1, 2, 1, smp["nc"])
    return ({"value": value, "unit": UNIT, "cores": min(threads, n_int), "kind": "port",
             "sample": _sample_text(smp, min(threads, n_int), n_int, 2)},
            {"value": one, "unit": UNIT, "cores": 1, "kind": "port", "sample": _sample_text(smp, 1, 1, 2)})


def _consistent_rhs(torch, sol, n_steps, seed):
    """Seeded uniform[-1,1] load vectors made consistent: constrained velocity
    rows zero, per-slot pressure mean zero."""
    lv = sol.finest
    gen = torch.Generator(device="cuda")
    gen.manual_seed(seed)
    F = torch.rand(n_steps * lv.size, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    gx, gy = lv.grid_x, lv.n_scalar // lv.grid_x
    Fv = F.view(n_steps, lv.size)
    npc = (sol.level_info[-1]["r"] + 1) * (sol.level_info[-1]["r"] + 2) // 2
    for a in range(lv.n_slots):
        for c in range(2):
            base = a * lv.n_velocity + c * lv.n_scalar
            g = Fv[:, base: base + lv.n_scalar].view(n_steps, gy, gx)
            g[:, 0, :] = 0
            g[:, -1, :] = 0
            g[:, :, 0] = 0
            g[:, :, -1] = 0
        pb = lv.n_slots * lv.n_velocity + a * lv.n_pressure
        p = Fv[:, pb: pb + lv.n_pressure].view(n_steps, -1, npc)
        p[:, :, 0] -= p[:, :, 0].mean(dim=1, keepdim=True)
    return F


def solve_legs(stmg, ctx, torch):
    """Full FGMRES + hp-STMG V(2,2) time-marching solves to rtol 1e-8 on
    seeded consistent load vectors: C1 exactly (16^2, Q2/P1, DG(1), 8
    intervals, cell Vanka) and the C4 discretisation (1024^2, Q2/P1, DG(1),
    tau = 1/64, vertex-star Vanka) over its first 2 intervals."""
    out = {}
    for name, kw in [("C1", dict(refinements=4, r=1, k=1, n_steps=8, t_end=1.0, smoother=stmg.SMOOTHER_CELL)),
                     ("C4_first2", dict(refinements=10, r=1, k=1, n_steps=2, t_end=2.0 / 64,
                                        smoother=stmg.SMOOTHER_VERTEX_STAR))]:
        sol = stmg.Solver(ctx, nu=1.0, gamma=1.0, nu1=2, nu2=2, omega=0.8, rtol=1e-8, **kw)
        F = _consistent_rhs(torch, sol, sol.n_steps, 11)
        X = torch.zeros_like(F)
        sol.time_march(F, X)  # warm-up: Krylov workspace
        torch.cuda.synchronize()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s.record()
        iters = sol.time_march(F, X)
        e.record()
        torch.cuda.synchronize()
        sec = s.elapsed_time(e) / 1e3
        out[name] = {"dofs": F.numel(), "seconds": sec, "dofs_per_s": F.numel() / sec,
                     "avg_gmres_iterations": sum(iters) / len(iters), "levels": sol.n_levels,
                     "smoother": "cell" if kw["smoother"] == stmg.SMOOTHER_CELL else "vertex_star"}
        del sol, F, X
    return out


def c4_step_leg(stmg, ctx, torch, n_int=8, reps=5):
    """C4 discretisation (1024^2, Q2/P1, DG(1), tau = 1/64, vertex-star Vanka)
    over one 8-interval slab (1.85e8 space-time dofs): all-at-once vmult and
    one smoother step (residual + Vanka update), CUDA-event timed."""
    lvl = stmg.Level(ctx, 1024, 1024, 1, 1, 1.0 / 64, 1.0, 1.0, stmg.SMOOTHER_VERTEX_STAR)
    n = n_int * lvl.size
    g = torch.Generator(device="cuda")
    g.manual_seed(77)
    x = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    b = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    u = torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1
    y, res = torch.empty_like(x), torch.empty_like(x)
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    tv, tr, tk = [], [], []
    for it in range(reps + 2):
        ev[0].record()
        lvl.vmult(x, y, n_int)
        ev[1].record()
        lvl.residual(b, u, res, n_int, None, coupled=True)
        ev[2].record()
        lvl.vanka_update(res, u, 0.8, n_int)
        ev[3].record()
        torch.cuda.synchronize()
        if it >= 2:
            tv.append(ev[0].elapsed_time(ev[1]))
            tr.append(ev[1].elapsed_time(ev[2]))
            tk.append(ev[2].elapsed_time(ev[3]))
    vm, rs, vk = (statistics.mean(t) for t in (tv, tr, tk))
    flops_vk = 2.0 * lvl.total_matrix_elements * n_int
    out = {"dofs": n, "vmult_ms": vm, "residual_ms": rs, "vanka_update_ms": vk,
           "vmult_dofs_per_s": n / (vm * 1e-3), "smoother_step_dofs_per_s": n / ((rs + vk) * 1e-3),
           "vanka_TFLOP/s": flops_vk / vk / 1e9, "smoother": "vertex_star (n_T = 124)"}
    del lvl, x, b, u, y, res
    return out


def vmult3c_fma_per_cell_slot(S, coupled=True):
    """FMAs of vmult3c_kernel (st3d.cu) per cell and output slot, counted from
    the kernel: x pass (temporal combination 3*3*(2S+1), x contraction 3*3*12,
    pressure partials 4*3*4), y pass (3*3*18), z pass (3*3*(9+4)), per line
    thread x 9 lines, plus the cell's pressure moments (4*S)."""
    per_line = 3 * 3 * (2 * S + (1 if coupled else 0)) + 108 + 48 + 162 + 117
    return 9 * per_line + 4 * S


def three_d_leg(torch, stmg):
    """BASELINE configs[2] (C3: 32^3 Q2/P1disc, DG(1), 64 intervals: vmult,
    cell-Vanka step, full all-at-once FGMRES + hp-STMG solve) and configs[4]
    (C5: 32^3 deformed Q3/P2disc, DG(2), 128 intervals: vmult) on this GPU."""
    sys.path.insert(0, str(ROOT / "tools"))
    import bench3d

    a = argparse.Namespace(reps=5, c3_cells=32, c3_intervals=64, c3_hcoarse=3, c3_variant="robust", maxit=200,
                           no_solve=False, c5_cells=32, c5_intervals=128, c5_slab=16, c5_variant="robust")
    out = {"C3": bench3d.run_c3(torch, stmg, a)}
    c3 = out["C3"]
    hbm, fp64, dmma, src = peaks()
    cells, S, nI = a.c3_cells ** 3, 2, a.c3_intervals
    flops = 2.0 * vmult3c_fma_per_cell_slot(S) * cells * S * nI
    byts = 16.0 * c3["dofs"]
    c3["vmult_roofline"] = {
        "kernel": "vmult3c_kernel (C3 vmult, 1D-factor form)", "bound": "fp64",
        "flops_per_launch": flops, "algorithmic_bytes": byts,
        "achieved_TFLOPs": flops / (c3["vmult_ms"] * 1e-3) / 1e12,
        "fp64_frac": flops / (c3["vmult_ms"] * 1e-3) / 1e12 / fp64,
        "hbm_frac": byts / (c3["vmult_ms"] * 1e-3) / 1e9 / hbm, "peak_source": src}
    c3["vanka_dmma_frac"] = c3["vanka_update_TFLOPs"] / dmma
    torch.cuda.empty_cache()
    out["C5"] = bench3d.run_c5(torch, stmg, a)
    torch.cuda.empty_cache()
    out["C5"]["solve"] = bench3d.run_c5_solve(torch, stmg, a)
    torch.cuda.empty_cache()
    return out


def c3_slab_leg(stmg, torch, dist, world, rank, n_total=64):
    """BASELINE configs[2] (C3) partitioned by time slabs: the 64-interval
    32^3 Q2/P1disc DG(1) all-at-once system split over the ranks (strong
    scaling), FGMRES + hp-STMG V(2,2) (h in space down to 2^3, k kept at 1,
    exact coarse forward substitution in time over all intervals), halo /
    Krylov dots / coarse right-hand sides over NCCL. Time = max over ranks."""
    from paper_2502_09159_b200 import timeslab

    sys.path.insert(0, str(ROOT / "tools"))
    import bench3d

    n_local = n_total // world
    ctx = stmg.Context(torch.cuda.current_device())
    sol = stmg.Solver3(ctx, 32, 32, 32, 1, 1, 1.0 / n_total, 1.0, 1.0, n_hcoarse=4, time_coarsen=False, k_min=1,
                       nu1=2, nu2=2, rtol=1e-8)
    if world > 1:  # the library's C++ NCCL communicator; CGS2: two all-reduces per iteration
        sol.set_comm(timeslab.nccl_comm())
        sol.set_krylov(stmg.ORTHO_CGS2)
    f = sol.finest
    F = bench3d.consistent(torch, f, bench3d.seeded(torch, n_local * f.size, 301 + rank), n_local)
    X = torch.zeros_like(F)
    sol.solve_all_at_once(F, X, n_local)  # warm-up: Krylov workspace
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    it, hist = sol.solve_all_at_once(F, X, n_local)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3
    if world > 1:
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    total = world * F.numel()
    out = {"dofs": total, "intervals": n_total, "seconds": sec, "dofs_per_s": total / sec, "fgmres_iterations": it,
           "relative_residual": hist[-1] / hist[0], "levels": sol.n_levels, "smoother": "cell (n_T = 170)",
           "partition": f"{world} time slabs x {n_local} intervals (strong scaling)"}
    del sol, F, X
    torch.cuda.empty_cache()
    return out


def c5_hybrid_leg(stmg, torch, dist, world, rank, n=32, n_total=128, parts=2):
    """BASELINE configs[4] (C5) as specified: ONE all-at-once FGMRES solve of
    the whole 128-interval 32^3 deformed Q3/P2disc DG(2) system, hybrid
    partition of `world` = parts (z) x slabs (time) GPUs (2 x 4 on 8 GPUs;
    stmg3_solver_create_split). Both communicators are the library's NCCL
    ones: time slabs among the ranks of one z part, interface planes / part
    sums among the ranks of one slab. RHS: a hash of the global dof index
    (so the parts agree on their shared planes), made consistent with the
    global pressure mean. Hierarchy as the 1-GPU C5 leg (r 2 -> 1, h in space
    to 2^3, k kept at 2, exact patch inverses built on the GPU). Time = max
    over ranks."""
    from paper_2502_09159_b200 import timeslab

    sys.path.insert(0, str(ROOT / "tools"))
    import bench3d

    slabs = world // parts
    part, slab = rank % parts, rank // parts
    n_local = n_total // slabs
    # every rank creates every group, in the same order
    tgroups = [dist.new_group([s * parts + p for s in range(slabs)]) for p in range(parts)]
    sgroups = [dist.new_group([s * parts + p for p in range(parts)]) for s in range(slabs)]
    ctx = stmg.Context(torch.cuda.current_device())
    t0 = time.perf_counter()
    sol = stmg.Solver3(ctx, n, n, n, 2, 2, 1.0 / n_total, 1.0, 1.0, n_hcoarse=4, time_coarsen=False, k_min=2,
                       vertices=bench3d.c5_vertices(n), nu1=2, nu2=2, rtol=1e-8, z_parts=parts, z_part=part)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    if slabs > 1:
        sol.set_comm(timeslab.nccl_comm(group=tgroups[part]))
    sol.set_space_comm(timeslab.nccl_comm(group=sgroups[slab]))
    sol.set_krylov(stmg.ORTHO_CGS2)
    f = sol.finest
    idx = torch.from_numpy(timeslab.z_part_dofs(n, n, n, 2, 2, parts, part)).cuda()
    gn = torch.arange(slab * n_local, (slab + 1) * n_local, device="cuda", dtype=torch.int64)[:, None]
    h = (idx[None, :] * 2654435761 + gn * 2246822519 + 12345) % 4294967296
    h = (h ^ (h >> 13)) * 1274126177 % 4294967296
    F = (h.double() / 4294967296.0 * 2 - 1).reshape(-1).contiguous()
    del h
    V = F.view(n_local, f.size)
    bnd = torch.zeros((f.gz, f.gy, f.gx), dtype=torch.bool, device="cuda")
    bnd[:, 0] = bnd[:, -1] = True
    bnd[:, :, 0] = bnd[:, :, -1] = True
    if part == 0:
        bnd[0] = True
    if part == parts - 1:
        bnd[-1] = True
    bnd = bnd.reshape(-1)
    for a in range(f.n_slots):
        for c in range(3):
            base = a * f.n_velocity + c * f.n_scalar
            V[:, base:base + f.n_scalar][:, bnd] = 0.0
        p0 = f.n_slots * f.n_velocity + a * f.n_pressure
        P = V[:, p0:p0 + f.n_pressure].view(n_local, -1, f.n_p)
        m = P[:, :, 0].sum(dim=1).contiguous()
        dist.all_reduce(m, group=sgroups[slab])
        P[:, :, 0] -= (m / (n ** 3))[:, None]
    X = torch.zeros_like(F)
    torch.cuda.synchronize()
    dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    it, hist = sol.solve_all_at_once(F, X, n_local)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3
    t = torch.tensor([sec], device="cuda")
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    sec = float(t.item())
    # whole-system dofs: the parts' interface planes are stored twice
    total = n_total * (f.size * parts - (parts - 1) * f.n_slots * 3 * f.gx * f.gy)
    out = {"dofs": int(total), "intervals": n_total, "seconds": sec, "dofs_per_s": total / sec,
           "fgmres_iterations": it, "relative_residual": hist[-1] / hist[0], "setup_s": setup,
           "levels": sol.n_levels, "smoother": "cell Vanka, exact per-cell patch inverses (built on the GPU)",
           "partition": f"hybrid {parts} z parts x {slabs} time slabs of {n_local} intervals (one all-at-once solve)",
           "deviation_from_baseline": "hierarchy substituted: k kept at 2 (BASELINE configs[4]: k 2->1->0), h in "
                                      "space only, exact coarse forward substitution over all 128 intervals"}
    del sol, F, X
    torch.cuda.empty_cache()
    return out


def slab_solve_leg(stmg, ctx, torch, dist, world, rank, n_local=8):
    """All-at-once FGMRES + hp-STMG V(2,2) solve of the C4 discretisation
    (1024^2, Q2/P1, DG(1), tau = 1/64, vertex-star Vanka) partitioned by time
    slabs: every rank owns n_local intervals of a world*n_local system
    (weak scaling; 8 GPUs x 8 intervals = the full 64-interval C4 system).
    Halo, Krylov dots and coarse right-hand sides go over NCCL. Time = max
    over ranks of CUDA-event time of the solve."""
    from paper_2502_09159_b200 import timeslab

    sol = stmg.Solver(ctx, 10, 1, 1, n_steps=n_local, t_end=n_local / 64.0, nu=1.0, gamma=1.0,
                      smoother=stmg.SMOOTHER_VERTEX_STAR, nu1=2, nu2=2, omega=0.8, rtol=1e-8)
    if world > 1:  # the library's C++ NCCL communicator; CGS2: two all-reduces per iteration
        sol.set_comm(timeslab.nccl_comm())
        sol.set_krylov(stmg.ORTHO_CGS2)
    F = _consistent_rhs(torch, sol, n_local, 101 + rank)
    X = torch.zeros_like(F)
    sol.solve_all_at_once(F, X, n_local)  # warm-up: Krylov workspace, coarse tables
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    it, hist = sol.solve_all_at_once(F, X, n_local)
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3
    if world > 1:
        t = torch.tensor([sec], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        sec = float(t.item())
    total = world * F.numel()
    out = {"dofs": total, "intervals": world * n_local, "seconds": sec, "dofs_per_s": total / sec,
           "fgmres_iterations": it, "relative_residual": hist[-1] / hist[0], "levels": sol.n_levels,
           "smoother": "vertex_star", "partition": f"{world} time slabs x {n_local} intervals"}
    del sol, F, X
    return out


def c4_full_leg(stmg, ctx, torch, n_total=64, slab=8):
    """The whole C4 system on one GPU: 1024^2, Q2/P1, DG(1), 64 intervals on
    [0, 1] (1.48e9 space-time dofs), vertex-star Vanka V(2,2), FGMRES to
    1e-8 per slab. One all-at-once slab would need a ~350 GB Krylov basis, so
    the 64 intervals are solved as 8 macro steps of 8,
    each slab continuing from the previous slab's last velocity (v_init).
    Time = CUDA events around all 8 slab solves."""
    sol = stmg.Solver(ctx, 10, 1, 1, n_steps=slab, t_end=slab / float(n_total), nu=1.0, gamma=1.0,
                      smoother=stmg.SMOOTHER_VERTEX_STAR, nu1=2, nu2=2, omega=0.8, rtol=1e-8)
    lv = sol.finest
    F = _consistent_rhs(torch, sol, slab, 303)  # one slab of load vectors, reused per macro step
    X = torch.zeros_like(F)
    v = torch.zeros(lv.n_velocity, dtype=torch.float64, device="cuda")
    last = (slab - 1) * lv.size + (lv.n_slots - 1) * lv.n_velocity
    sol.solve_all_at_once(F, X, slab)  # warm-up
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    iters = []
    s.record()
    for m in range(n_total // slab):
        it, _ = sol.solve_all_at_once(F, X, slab, v_init=None if m == 0 else v)
        iters.append(it)
        v.copy_(X[last:last + lv.n_velocity])
    e.record()
    torch.cuda.synchronize()
    sec = s.elapsed_time(e) / 1e3
    dofs = n_total * lv.size
    out = {"dofs": dofs, "intervals": n_total, "seconds": sec, "dofs_per_s": dofs / sec,
           "fgmres_iterations_per_slab": iters, "smoother": "vertex_star",
           "partition": f"1 GPU, {n_total // slab} macro steps x {slab} intervals"}
    del sol, F, X
    return out


# ---------------------------------------------------------------- our arm
def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--nx", type=int, default=256)
    ap.add_argument("--intervals", type=int, default=64)
    ap.add_argument("--e2e-steps", type=int, default=5)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-solve", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
        return

    import torch
    import torch.distributed as dist

    import paper_2502_09159_b200 as stmg
    from paper_2502_09159_b200 import timeslab

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
    ctx = stmg.Context(local)
    nx, N, r, k = args.nx, args.intervals, CONFIG["r"], CONFIG["k"]
    tau = 1.0 / (N * world)
    lvl = stmg.Level(ctx, nx, nx, r, k, tau, CONFIG["nu"], CONFIG["gamma"], stmg.SMOOTHER_CELL)
    isz, mv, S = lvl.size, lvl.n_velocity, lvl.n_slots
    dofs = N * isz
    gen = torch.Generator(device="cuda")
    gen.manual_seed(1234 + rank)
    x = torch.rand(dofs, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    b = torch.rand(dofs, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    u = torch.rand(dofs, dtype=torch.float64, device="cuda", generator=gen) * 2 - 1
    y = torch.empty_like(x)
    res = torch.empty_like(x)
    halo_x = torch.zeros(mv, dtype=torch.float64, device="cuda")
    halo_u = torch.zeros(mv, dtype=torch.float64, device="cuda")

    comm_stream = torch.cuda.Stream() if world > 1 else None
    if world > 1:  # halo send/recv through the library's NCCL communicator (stmg_comm_nccl_ops)
        step_comm = timeslab.nccl_comm()
        step_ops = step_comm.ops()

    def coupled(apply, src, halo, dst, *extra):
        """Time-slab application with the halo exchange overlapped: the NCCL
        send/recv of the slot-k velocity runs on a side stream while
        intervals 1..N-1 (local predecessor) are computed; interval 0 then
        waits for the halo."""
        if world == 1:
            apply(src, dst, N, None, *extra)
            return
        main = torch.cuda.current_stream()
        comm_stream.wait_stream(main)
        send = src[(N - 1) * isz + (S - 1) * mv:(N - 1) * isz + S * mv]
        if step_ops.exchange_halo(step_ops.user, send.data_ptr(), halo.data_ptr(), mv, comm_stream.cuda_stream) != 0:
            raise RuntimeError("halo exchange failed")
        h = halo if rank > 0 else None
        if N > 1:
            apply(src[isz:], dst[isz:], N - 1, src[(S - 1) * mv:S * mv], *[e[isz:] for e in extra])
        main.wait_stream(comm_stream)
        apply(src[:isz], dst[:isz], 1, h, *[e[:isz] for e in extra])

    def vmult(src, dst, n, prev):
        lvl.vmult(src, dst, n, prev)

    def residual(src, dst, n, prev, bb):
        lvl.residual(bb, src, dst, n, prev, coupled=True)

    ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    t_vmult, t_resid, t_vanka = [], [], []

    def step(record):
        if record:
            ev[0].record()
        coupled(vmult, x, halo_x, y)
        if record:
            ev[1].record()
        coupled(residual, u, halo_u, res, b)
        if record:
            ev[2].record()
        lvl.vanka_update(res, u, CONFIG["omega"], N)
        if record:
            ev[3].record()

    for _ in range(args.warmup):
        step(False)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    torch.cuda.synchronize()
    launches0 = ctx.launch_count()
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with ClockSampler(local) as clk:
        start.record()
        for _ in range(args.steps):
            step(True)
            torch.cuda.synchronize()  # per-step event readout (kernel shares below)
            t_vmult.append(ev[0].elapsed_time(ev[1]))
            t_resid.append(ev[1].elapsed_time(ev[2]))
            t_vanka.append(ev[2].elapsed_time(ev[3]))
        stop.record()
        torch.cuda.synchronize()
    gpu_launches = ctx.launch_count() - launches0
    ms = start.elapsed_time(stop) / args.steps
    if world > 1:
        t = torch.tensor([ms], device="cuda")
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        dist.barrier()
    value = world * dofs / (ms * 1e-3)

    # ---- end to end through the host-buffer C ABI (pinned host memory)
    e2e = None
    if args.e2e_steps > 0:
        hx = torch.empty(dofs, dtype=torch.float64, pin_memory=True)
        hb = torch.empty(dofs, dtype=torch.float64, pin_memory=True)
        hu = torch.empty(dofs, dtype=torch.float64, pin_memory=True)
        hy = torch.empty(dofs, dtype=torch.float64, pin_memory=True)
        hh = torch.empty(mv, dtype=torch.float64, pin_memory=True)
        hx.copy_(x)
        hb.copy_(b)
        hu.copy_(u)
        hh.zero_()
        nx_, nb_, nu_, ny_, nh_ = hx.numpy(), hb.numpy(), hu.numpy(), hy.numpy(), hh.numpy()
        halo_arg = nh_ if rank > 0 else None
        # the step's two calls are the non-blocking host entry points: the
        # smoother's H2D copies overlap the vmult's kernels and D2H copies;
        # every step ends with a synchronisation (its results are on the host)
        lvl.vmult_host(nx_, ny_, N, halo_arg, blocking=False)  # warm-up of both entry points
        lvl.smooth_step_host(nb_, nu_, CONFIG["omega"], N, halo_arg, True, blocking=False)
        ctx.synchronize()
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        t0 = time.perf_counter()
        for _ in range(args.e2e_steps):
            lvl.vmult_host(nx_, ny_, N, halo_arg, blocking=False)
            lvl.smooth_step_host(nb_, nu_, CONFIG["omega"], N, halo_arg, True, blocking=False)
            ctx.synchronize()
        e2e_s = (time.perf_counter() - t0) / args.e2e_steps
        if world > 1:
            t = torch.tensor([e2e_s], device="cuda")
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            e2e_s = float(t.item())
        e2e = {"value": world * dofs / e2e_s, "unit": UNIT, "h2d_bytes_per_step": 8 * (3 * dofs + 2 * mv),
               "d2h_bytes_per_step": 8 * 2 * dofs}

    line = None
    hbm, fp64, dmma, peak_src = peaks()
    ncell = nx * nx
    vm_ms = statistics.mean(t_vmult)
    rs_ms = statistics.mean(t_resid)
    vk_ms = statistics.mean(t_vanka)
    vm_flops = 2.0 * vmult_fma_per_cell(r, k) * ncell * N
    vm_bytes = 16.0 * dofs
    sum_nt2 = lvl.total_matrix_elements
    vk_flops = 2.0 * sum_nt2 * N
    vk_bytes = 24.0 * dofs
    kernels = {
        "vmult": {"ms": vm_ms, "GB/s": vm_bytes / vm_ms / 1e6, "TFLOP/s": vm_flops / vm_ms / 1e9,
                  "algorithmic_bytes": vm_bytes, "algorithmic_flops": vm_flops},
        "residual": {"ms": rs_ms, "GB/s": 24.0 * dofs / rs_ms / 1e6, "TFLOP/s": vm_flops / rs_ms / 1e9},
        "vanka_update": {"ms": vk_ms, "GB/s": vk_bytes / vk_ms / 1e6, "TFLOP/s": vk_flops / vk_ms / 1e9,
                         "algorithmic_bytes": vk_bytes, "algorithmic_flops": vk_flops, "launches": 4},
    }
    dom = "vanka_update" if vk_ms >= vm_ms else "vmult"
    kd = kernels[dom]
    # both candidate roofs; the binding one is the larger time bound. The Vanka
    # update runs on the FP64 tensor path (DMMA), the vmult on the DFMA pipe
    # (they share one FP64 datapath: profiles/fp64_peaks_r01.json).
    pk = dmma if dom == "vanka_update" else fp64
    t_hbm = kd["algorithmic_bytes"] / (hbm * 1e9)
    t_fp = kd["algorithmic_flops"] / (pk * 1e12)
    if t_fp >= t_hbm:
        roof = {"bound": "tensor", "achieved": kd["TFLOP/s"], "peak": pk, "unit": "TFLOP/s",
                "frac": kd["TFLOP/s"] / pk,
                "pipe": "FP64 mma.sync m8n8k4 (DMMA)" if dom == "vanka_update" else "FP64 DFMA"}
    else:
        roof = {"bound": "hbm", "achieved": kd["GB/s"], "peak": hbm, "unit": "GB/s", "frac": kd["GB/s"] / hbm}
    traffic = None
    try:  # dram__bytes_read+write per launch of this kernel from the committed ncu capture
        tr = json.loads(sorted((ROOT / "profiles").glob("r*_traffic.json"))[-1].read_text())  # latest round
        per = tr["per_launch_dram_bytes"]
        traffic = per["vmult"] if dom == "vmult" else per["vanka_update_pass"] * tr["launches_per_step"]["vanka_update_pass"]
    except Exception:
        pass
    roof.update({"kernel": dom, "traffic": traffic, "algorithmic_bytes": kd["algorithmic_bytes"],
                 "traffic_basis": ("bytes per Vanka update = 4 launches (one per strip colour); achieved TF/s is the "
                                   "same per launch" if dom == "vanka_update" else "bytes per launch"),
                 "peak_source": peak_src, "hbm_frac": kd["GB/s"] / hbm, "fp64_frac": kd["TFLOP/s"] / pk})
    line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded uniform[-1,1], torch Philox on device)",
            "config": arm_config(world, dofs, nx, N),
            "components": {"vmult_dofs_per_s": world * dofs / (vm_ms * 1e-3),
                           "vanka_step_dofs_per_s": world * dofs / ((rs_ms + vk_ms) * 1e-3)},
            "kernels": kernels, "roofline": roof, "gpu_launches": gpu_launches,
            "clocks": clk.summary(), "e2e": e2e}
    # ---- collective side legs (every rank takes part). With several ranks they
    # run under a deadline: a rank that raised while its peers wait in a
    # collective would otherwise hang the job and lose the headline line.
    watchdog = None
    if world > 1 and not args.no_solve:
        deadline = float(os.environ.get("STMG_BENCH_SIDE_TIMEOUT", "900"))

        def give_up():
            if rank == 0:
                line["solve"] = {"error": f"multi-rank side legs exceeded {deadline:.0f} s; headline only"}
                print(json.dumps(line), flush=True)
            os._exit(0)

        watchdog = threading.Timer(deadline, give_up)
        watchdog.daemon = True
        watchdog.start()
    slab = c3slab = c5hyb = None
    if not args.no_solve:
        try:  # a side leg: a failure is reported in the line, never fatal for the headline
            slab = slab_solve_leg(stmg, ctx, torch, dist, world, rank)
        except Exception as exc:
            slab = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        try:
            c3slab = c3_slab_leg(stmg, torch, dist, world, rank)
        except Exception as exc:
            c3slab = {"error": f"{type(exc).__name__}: {exc}"[:300]}
        if world >= 4 and world % 2 == 0:  # >= 2 time slabs: <= 64 intervals (~100 GB) per rank
            try:
                c5hyb = c5_hybrid_leg(stmg, torch, dist, world, rank)
            except Exception as exc:
                c5hyb = {"error": f"{type(exc).__name__}: {exc}"[:300]}

    if watchdog is not None:
        watchdog.cancel()
    if rank != 0:
        if world > 1:
            dist.destroy_process_group()
        return
    if not args.no_solve:
        def side(fn):
            try:
                return fn()
            except Exception as exc:  # reported, never fatal for the headline
                return {"error": f"{type(exc).__name__}: {exc}"[:300]}
        line["solve"] = side(lambda: solve_legs(stmg, ctx, torch))
        line["solve"]["C4_all_at_once"] = slab
        line["solve"]["C3_all_at_once"] = c3slab
        if c5hyb is not None:
            line["solve"]["C5_hybrid"] = c5hyb
        line["C4_step"] = side(lambda: c4_step_leg(stmg, ctx, torch))
        if world == 1:
            line["solve"]["C4_full"] = side(lambda: c4_full_leg(stmg, ctx, torch))
            line["3D"] = side(lambda: three_d_leg(torch, stmg))
    if not args.no_cpu_baseline:
        try:
            line["cpu_baseline"], line["cpu_baseline_1core"] = cpu_baseline_quick()
            line["host"] = host_cpu()
        except Exception as exc:  # the baseline is reported, never required
            line["cpu_baseline"] = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "port",
                                    "sample": f"failed: {exc}"}
    print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
