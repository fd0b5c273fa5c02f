"""Debug helper: product apply_additive vs oracle, error map by dof kind."""
import sys
from pathlib import Path
import numpy as np
import torch
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parents[1] / "tests"))
import paper_2502_09159_b200 as stmg
import oracle_ctypes as oc
ctx = stmg.Context(0)
for (nc, r, k, kind) in [(8, 1, 1, 1), (4, 1, 1, 1), (2, 1, 1, 1), (8, 1, 1, 0), (4, 2, 1, 1)]:
    lvl = stmg.Level(ctx, nc, nc, r, k, 0.25, 0.1, 1.0, kind)
    ref = oc.OracleLevel(nc, r, k, 0.25, 0.1, 1.0, kind)
    res = oc.seeded(ref.size, 21)
    out = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    lvl.apply_additive(torch.from_numpy(res).cuda(), out)
    torch.cuda.synchronize()
    o = out.cpu().numpy()
    e = ref.apply_additive(res)
    d = np.abs(o - e)
    S, mv = ref.n_slots, ref.n_velocity
    nsc = ref.n_scalar
    gx = ref.grid_x
    print(nc, r, k, kind, "max rel", d.max() / np.abs(e).max(), "classes", lvl.n_patch_classes)
    bad = np.where(d > 1e-9 * np.abs(e).max())[0]
    for idx in bad[:12]:
        if idx < S * mv:
            a, rem = divmod(idx, mv); c, s = divmod(rem, nsc); print("  vel slot", a, "comp", c, "node", s % gx, s // gx, o[idx], e[idx])
        else:
            q = idx - S * mv; a, cm = divmod(q, ref.n_pressure); print("  pre slot", a, "cellmode", cm, o[idx], e[idx])
    print("  n bad", len(bad), "of", ref.size)
