#!/usr/bin/env python
"""3D workloads of BASELINE.json on one B200 (configs[2] "C3", configs[4] "C5").

  C3: 3D Stokes, Q2/P1disc (r=1), DG(1), 32^3 Cartesian cells, 64 intervals,
      ~1.2e8 space-time dofs. vmult, cell-Vanka smoother step and the full
      all-at-once FGMRES + hp-STMG solve (p: k 1 -> 0, then h in space AND time
      down to 4^3 x 8, exact coarse forward substitution on the GPU).
  C5: 3D Stokes, Q3/P2disc (r=2), DG(2), 32^3 cells with interior vertices
      perturbed by <= 0.1 h (seeded), 128 intervals, ~1.2e9 dofs: vmult.

Prints one JSON object. Inputs are seeded uniform[-1,1] on the device;
timings are CUDA events on the library's stream after warm-up.
"""
from __future__ import annotations

import argparse
import json
import sys
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))


def seeded(torch, n, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.rand(n, dtype=torch.float64, device="cuda", generator=g) * 2 - 1


def consistent(torch, lvl, F, n):
    """Constrained velocity rows zero, per-slot pressure component along the
    constant mode removed."""
    gx, gy, gz = lvl.gx, lvl.gy, lvl.gz
    bnd = torch.zeros((gz, gy, gx), dtype=torch.bool, device="cuda")
    bnd[0] = bnd[-1] = True
    bnd[:, 0] = bnd[:, -1] = True
    bnd[:, :, 0] = bnd[:, :, -1] = True
    bnd = bnd.reshape(-1)
    V = F.view(n, lvl.size)
    for a in range(lvl.n_slots):
        for c in range(3):
            base = a * lvl.n_velocity + c * lvl.n_scalar
            V[:, base:base + lvl.n_scalar][:, bnd] = 0.0
        p0 = lvl.n_slots * lvl.n_velocity + a * lvl.n_pressure
        P = V[:, p0:p0 + lvl.n_pressure].view(n, -1, lvl.n_p)
        P[:, :, 0] -= P[:, :, 0].mean(dim=1, keepdim=True)
    return F


def timed(torch, fn, reps, warm=2):
    for _ in range(warm):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def run_c3(torch, stmg, args):
    ctx = stmg.Context(0)
    n, N = args.c3_cells, args.c3_intervals
    out = {"config": f"C3: {n}^3 Q2/P1disc, DG(1), {N} intervals, nu=1, gamma=1, V(2,2) cell Vanka"}
    t0 = time.perf_counter()
    spec = args.c3_variant == "spec"
    # "spec": BASELINE's plan, k 1 -> 0 (temporal p-step on the coarsest
    # level, as combine_hierarchies) and h in space AND time down to 4^3 x 8;
    # "robust": k kept at 1, h in space only down to 2^3, exact coarse
    # forward substitution over all intervals (time
    # coarsening and k -> 0 cost iterations with the time-block-diagonal Vanka)
    sol = stmg.Solver3(ctx, n, n, n, 1, 1, 1.0 / N, 1.0, 1.0, n_hcoarse=args.c3_hcoarse if spec else args.c3_hcoarse + 1,
                       time_coarsen=spec, k_min=0 if spec else 1, nu1=2, nu2=2, rtol=1e-8, max_iterations=args.maxit)
    out["variant"] = args.c3_variant
    if not spec:
        out["deviation_from_baseline"] = (
            "hierarchy substituted: k kept at 1 and h-coarsening in space only (to 2^3), exact coarse forward "
            "substitution in time over all intervals. BASELINE configs[2] asks for k 1->0 then h in space AND time "
            "down to 4^3x8; with the reference's cell Vanka that plan is not h-robust: its time h-coarsening costs "
            "42 / 94 FGMRES iterations at 8^3 / 16^3 (k->0 alone: 15 / 15; damping 0.4-0.8 and a forward "
            "Gauss-Seidel sweep in time do not help), DESIGN.md 3.4; at 32^3 x 64 its Krylov space does not fit, "
            "so the full BASELINE plan is unmeasured; solve_k_to_0 measures its k->0 part")
    torch.cuda.synchronize()
    out["setup_s"] = time.perf_counter() - t0
    out["levels"] = sol.level_info
    f = sol.finest
    dofs = N * f.size
    out["dofs"] = dofs
    x = seeded(torch, dofs, 1)
    y = torch.empty_like(x)
    b = seeded(torch, dofs, 2)
    halo = seeded(torch, f.n_velocity, 3)
    ms = timed(torch, lambda: f.vmult(x, y, N, halo), args.reps)
    out["vmult_ms"] = ms
    out["vmult_dofs_per_s"] = dofs / (ms * 1e-3)
    ms = timed(torch, lambda: f.residual(b, x, y, N, halo), args.reps)
    out["residual_ms"] = ms
    fl = sol.levels[-1]
    # smoother step on the finest level of the hierarchy (has cell Vanka only
    # below the finest? the finest carries the smoother too)
    u = x.clone()
    work = torch.empty_like(x)
    ms = timed(torch, lambda: fl.smooth_step(b, u, 0.8, N, halo, coupled=True, work=work), args.reps)
    out["smooth_step_ms"] = ms
    out["smooth_step_dofs_per_s"] = dofs / (ms * 1e-3)
    out["max_patch"] = fl.max_patch
    out["vanka_flops"] = 2.0 * fl.total_matrix_elements * N
    out["vanka_update_TFLOPs"] = out["vanka_flops"] / ((ms - out["residual_ms"]) * 1e-3) / 1e12
    del u, work
    if not args.no_solve:
        F = consistent(torch, f, seeded(torch, dofs, 4), N)
        X = torch.zeros_like(F)
        sol.solve_all_at_once(F, X, N)  # warm (workspaces)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        it, hist = sol.solve_all_at_once(F, X, N)
        e1.record()
        torch.cuda.synchronize()
        s = e0.elapsed_time(e1) * 1e-3
        out["solve"] = {"seconds": s, "fgmres_iterations": it, "dofs_per_s": dofs / s,
                        "relative_residual": hist[-1] / hist[0]}
        if not spec:
            # the part of BASELINE's plan that is h-robust with this smoother:
            # k 1 -> 0 (temporal p-coarsening) + h in space only; the time
            # h-coarsening is what breaks robustness
            del sol
            torch.cuda.empty_cache()
            sk = stmg.Solver3(ctx, n, n, n, 1, 1, 1.0 / N, 1.0, 1.0, n_hcoarse=args.c3_hcoarse + 1, time_coarsen=False,
                              k_min=0, nu1=2, nu2=2, rtol=1e-8, max_iterations=args.maxit)
            X = torch.zeros_like(F)
            sk.solve_all_at_once(F, X, N)
            torch.cuda.synchronize()
            e0.record()
            it, hist = sk.solve_all_at_once(F, X, N)
            e1.record()
            torch.cuda.synchronize()
            s = e0.elapsed_time(e1) * 1e-3
            out["solve_k_to_0"] = {"seconds": s, "fgmres_iterations": it, "dofs_per_s": dofs / s,
                                   "relative_residual": hist[-1] / hist[0],
                                   "hierarchy": "k 1 -> 0 on the coarsest level, h in space only to 2^3 "
                                                "(BASELINE's plan without the time h-coarsening)"}
    return out


def c5_vertices(n, seed=2025):
    """Unit-cube vertices, interior ones displaced by a seeded uniform
    perturbation of at most 0.1 h per coordinate (BASELINE C5)."""
    import numpy as np

    rng = np.random.default_rng(seed)
    z, yy, xx = np.meshgrid(np.arange(n + 1) / n, np.arange(n + 1) / n, np.arange(n + 1) / n, indexing="ij")
    v = np.stack([xx, yy, z], axis=-1)
    inner = np.zeros(v.shape[:3], dtype=bool)
    inner[1:-1, 1:-1, 1:-1] = True
    v[inner] += rng.uniform(-1, 1, v.shape)[inner] * 0.1 / n
    return np.ascontiguousarray(v.reshape(-1))


def run_c5_solve(torch, stmg, args):
    """C5 full solve on one GPU: the 128-interval system as macro steps of
    args.c5_slab intervals (v_init hand-off), FGMRES +
    hp-STMG V(2,2): p in r 2 -> 1, h in space down to 2^3 ("robust": k kept
    at 2; "spec": k 2 -> 1 -> 0 on the coarsest levels), cell Vanka with the
    exact per-cell patch inverses (default) or the undeformed ones
    (--c5-patches affine)."""
    n, N, slab = args.c5_cells, args.c5_intervals, args.c5_slab
    verts = c5_vertices(n)
    ctx = stmg.Context(0)
    t0 = time.perf_counter()
    sol = stmg.Solver3(ctx, n, n, n, 2, 2, 1.0 / N, 1.0, 1.0, n_hcoarse=4, time_coarsen=False,
                       k_min=2 if args.c5_variant == "robust" else 0, vertices=verts,
                       affine_patches=getattr(args, "c5_patches", "exact") == "affine", nu1=2, nu2=2, rtol=1e-8,
                       max_iterations=args.maxit)
    torch.cuda.synchronize()
    setup = time.perf_counter() - t0
    free, total = torch.cuda.mem_get_info()
    f = sol.finest
    nsl = N // slab
    Fs = [consistent(torch, f, seeded(torch, slab * f.size, 500 + m), slab) for m in range(nsl)]
    X = torch.zeros(slab * f.size, dtype=torch.float64, device="cuda")
    sol.solve_all_at_once(Fs[0], X, slab)  # warm-up (workspaces)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    its = []
    v = None
    e0.record()
    for m in range(nsl):
        it, hist = sol.solve_all_at_once(Fs[m], X, slab, v_init=v)
        its.append(it)
        v = X[(slab - 1) * f.size + (f.n_slots - 1) * f.n_velocity:(slab - 1) * f.size + f.n_slots * f.n_velocity].clone()
    e1.record()
    torch.cuda.synchronize()
    s = e0.elapsed_time(e1) * 1e-3
    # one fine-level Vanka sweep (8 colour launches) over the slab: the
    # smoother kernel's own roofline (it streams the patch blocks from HBM)
    rr = seeded(torch, slab * f.size, 777)
    uu = torch.zeros_like(rr)
    sweep_ms = timed(torch, lambda: f.vanka_update(rr, uu, 0.8, slab), 3)
    # Roofline of the sweep. Bytes: what the kernel streams from HBM per sweep
    # (time-diagonalised form: the real block and the u-columns [P; Q] of the
    # pair block of every patch, 3 n_s^2 of the 5 n_s^2 stored doubles; dense
    # form: the whole inverse) plus 24 B per dof (read r, read-modify-write u).
    # Flops: 2 x multiply-adds per (patch, interval) column x intervals.
    ps = f.patch_setup
    stored_bytes = 8.0 * f.total_matrix_elements
    streamed_bytes = 8.0 * ps["streamed_elements"] if ps["factored"] else stored_bytes
    macs = ps["macs_per_column"] if ps["factored"] else f.total_matrix_elements
    groups = (slab + 15) // 16  # the blocks are streamed once per group of <= 16 intervals
    alg_bytes = streamed_bytes * groups + 24.0 * slab * f.size
    flops = 2.0 * macs * slab
    hbm = dmma = None
    try:
        import json
        from pathlib import Path
        root = Path(__file__).resolve().parents[1]
        hbm = float(json.loads((root / "MEASURED_PEAKS.json").read_text())["hbm_gbs"])
    except Exception:
        pass
    try:
        import json
        from pathlib import Path
        root = Path(__file__).resolve().parents[1]
        dmma = float(json.loads((root / "profiles" / "fp64_peaks_r01.json").read_text())["dmma_tflops"])
    except Exception:
        pass
    gbs, tfs = alg_bytes / sweep_ms / 1e6, flops / sweep_ms / 1e9
    sweep = {"ms": sweep_ms, "intervals": slab, "stored_patch_block_bytes": stored_bytes,
             "streamed_patch_block_bytes": streamed_bytes * groups, "algorithmic_bytes": alg_bytes,
             "algorithmic_flops": flops, "achieved_GBs": gbs, "achieved_TFLOPs": tfs,
             "hbm_frac": gbs / hbm if hbm else None, "dmma_frac": tfs / dmma if dmma else None,
             "kernel": "vanka_big_fac_kernel (time-diagonalised blocks, cp.async.bulk chunk ring)"
             if ps["factored"] else "vanka_big_kernel (dense inverses)"}
    if hbm and dmma:
        t_hbm, t_mma = alg_bytes / (hbm * 1e9), flops / (dmma * 1e12)
        sweep["bound"] = "tensor" if t_mma >= t_hbm else "hbm"
        sweep["frac"] = max(t_hbm, t_mma) / (sweep_ms * 1e-3)
    del rr, uu
    return {"dofs": N * f.size, "seconds": s, "dofs_per_s": N * f.size / s, "setup_s": setup,
            "fine_vanka_sweep": sweep,
            "device_memory_after_setup_gb": (total - free) / 1e9,
            "fgmres_iterations_per_slab": its, "levels": sol.level_info,
            "partition": f"1 GPU, {nsl} macro steps x {slab} intervals",
            "smoother": ("cell Vanka, undeformed patch inverses (affine_patches)"
                         if getattr(args, "c5_patches", "exact") == "affine" else
                         "cell Vanka, exact per-cell patch inverses built on the GPU, applied in the "
                         "time-diagonalised form (one real + one complex-pair block per cell)"),
            "patch_setup": [l.patch_setup for l in sol.levels[1:]], "variant": args.c5_variant,
            "deviation_from_baseline": (
                ("hierarchy substituted: k kept at 2 (BASELINE configs[4]: k 2->1->0), h in space only; BASELINE's plan "
                 "(--c5-variant spec: k 2->1->0 on the three coarsest levels) measured 42-43 FGMRES iterations per "
                 "slab and 69.9 s for the 128 intervals (8-interval slabs), DESIGN.md 3.4; " if
                 args.c5_variant == "robust" else "") +
                f"one GPU as {nsl} macro steps of {slab} intervals (BASELINE: one all-at-once solve on 8 GPUs, "
                "2 spatial x 4 temporal)")}


def run_c5(torch, stmg, args):
    ctx = stmg.Context(0)
    n, N = args.c5_cells, args.c5_intervals
    verts = c5_vertices(n)
    lvl = stmg.Level3(ctx, n, n, n, 2, 2, 1.0 / N, 1.0, 1.0, stmg.SMOOTHER_NONE, vertices=verts)
    dofs = N * lvl.size
    out = {"config": f"C5: {n}^3 deformed (<= 0.1 h), Q3/P2disc, DG(2), {N} intervals", "dofs": dofs}
    x = seeded(torch, dofs, 1)
    y = torch.empty_like(x)
    halo = seeded(torch, lvl.n_velocity, 3)
    ms = timed(torch, lambda: lvl.vmult(x, y, N, halo), args.reps)
    out["vmult_ms"] = ms
    out["vmult_dofs_per_s"] = dofs / (ms * 1e-3)
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--case", default="C3,C5")
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--c3-cells", type=int, default=32)
    ap.add_argument("--c3-intervals", type=int, default=64)
    ap.add_argument("--c3-hcoarse", type=int, default=3)
    ap.add_argument("--c5-cells", type=int, default=32)
    ap.add_argument("--c5-intervals", type=int, default=128)
    ap.add_argument("--no-solve", action="store_true")
    ap.add_argument("--c3-variant", default="robust", choices=["robust", "spec"])
    ap.add_argument("--maxit", type=int, default=200)
    ap.add_argument("--c5-slab", type=int, default=16)
    ap.add_argument("--c5-variant", default="robust", choices=["robust", "spec"])
    ap.add_argument("--c5-patches", default="exact", choices=["exact", "affine"])
    args = ap.parse_args()
    import torch
    import paper_2502_09159_b200 as stmg

    res = {}
    if "C3" in args.case:
        res["C3"] = run_c3(torch, stmg, args)
    if "C5" in args.case:
        res["C5"] = run_c5(torch, stmg, args)
        if not args.no_solve:
            torch.cuda.empty_cache()
            res["C5"]["solve"] = run_c5_solve(torch, stmg, args)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
