"""GPU tier at the BASELINE meshes: parity with the oracle where the size
dependent launch shapes actually occur (strip / row-segment vmult split,
8-super-cell strips and the 48-tile staging of the Vanka tile tables, the
16- and 8-interval tile sets with a ragged last interval group, the 3D block
and tile paths).

* vmult / residual over the whole vector: relative max-norm <= 1e-12
  (st_operator.cpp:321-421 + Eq. GloSys coupling).
* One all-at-once smoother step (vanka.cpp:196-233), <= 1e-10. In 2D the full
  set of patch factorizations at 256^2 / 1024^2 is 6.8 GB / 129 GB in the
  oracle, so the oracle factors only the patches that contain a sample of
  rows (oracle_smooth_step_rows: the requested rows receive exactly the full
  sweep's additions in the full sweep's order; CPU-tested to be bitwise equal
  to the full sweep). The sample: 4000 seeded random rows plus the first and
  last rows of every velocity component and pressure block of every slot,
  compared in every interval. In 3D the oracle runs the full sweep.
"""
import numpy as np
import pytest
import torch

import oracle3_ctypes as o3
import oracle_ctypes as oc

pytestmark = pytest.mark.gpu

VMULT_TOL = 1e-12
SMOOTH_TOL = 1e-10


def rel_max(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def dev(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    torch.cuda.synchronize()
    return t.cpu().numpy()


def sample_rows(ref, count=4000, seed=17):
    rows = set(np.random.default_rng(seed).integers(0, ref.size, count).tolist())
    S, mv, mp, nsc = ref.n_slots, ref.n_velocity, ref.n_pressure, ref.n_scalar
    for a in range(S):
        for c in range(2):
            base = a * mv + c * nsc
            rows.update([base, base + 1, base + ref.grid_x + 1, base + nsc // 2, base + nsc - 2, base + nsc - 1])
        pb = S * mv + a * mp
        rows.update([pb, pb + 1, pb + mp // 2, pb + mp - 1])
    return np.array(sorted(rows), dtype=np.int64)


C2D = [  # name, nc, r, k, tau, smoother, intervals
    # BASELINE configs[1] (C2): 256^2, Q3/P2disc, DG(2); 17 intervals = the
    # 16-interval tile set plus a ragged group of 1
    ("C2", 256, 2, 2, 1 / 64, 0, 17),
    # BASELINE configs[3] (C4): 1024^2, Q2/P1disc, DG(1), vertex-star patches;
    # 9 intervals = the 8-interval slab set plus a ragged group of 1
    ("C4", 1024, 1, 1, 1 / 64, 1, 9),
    # C4 mesh through the time-marching tile set (one interval per block)
    ("C4-march", 1024, 1, 1, 1 / 64, 1, 2),
]


@pytest.fixture(scope="module")
def threads():
    import os

    return os.cpu_count() or 1


@pytest.mark.parametrize("name,nc,r,k,tau,smoother,n", C2D, ids=[c[0] for c in C2D])
def test_baseline_mesh_vmult_and_smoother_2d(ctx, stmg, threads, name, nc, r, k, tau, smoother, n):
    ref = oc.OracleLevel(nc, r, k, tau, 1.0, 1.0, smoother, build_smoother=2)
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, 1.0, 1.0, smoother)
    assert lvl.size == ref.size
    x = oc.seeded(n * ref.size, 31)
    halo = oc.seeded(ref.n_velocity, 32)
    yr = ref.vmult_all(x, n, halo, threads)
    y = torch.zeros(n * lvl.size, dtype=torch.float64, device="cuda")
    xd, hd = dev(x), dev(halo)
    lvl.vmult(xd, y, n, hd)
    err = rel_max(host(y), yr)
    assert err <= VMULT_TOL, (name, "vmult", err)
    b = oc.seeded(n * ref.size, 33)
    bd = dev(b)
    res = torch.zeros_like(y)
    lvl.residual(bd, xd, res, n, hd, coupled=True)
    err = rel_max(host(res), b - yr)
    assert err <= VMULT_TOL, (name, "residual", err)
    del y, res
    rows = sample_rows(ref)
    ur = ref.smooth_step_rows(b, x, 0.8, n, rows, halo, threads)
    lvl.smooth_step(bd, xd, 0.8, n, hd, coupled=True)
    ug = host(xd).reshape(n, lvl.size)[:, rows]
    err = rel_max(ug, ur)
    assert err <= SMOOTH_TOL, (name, "smooth_step", err)


C3D = [  # name, n, r, k, tau, amp, intervals, smoother
    # BASELINE configs[2] (C3) discretisation at 16^3: Q2/P1disc, DG(1), 176-row Vanka split
    ("C3-16", 16, 1, 1, 1 / 64, 0.0, 5, True),
    # the C3 mesh itself, 32^3 (the oracle's assembled operator alone is ~15 GB)
    ("C3-32", 32, 1, 1, 1 / 64, 0.0, 2, False),
    # BASELINE configs[4] (C5) discretisation at 8^3: deformed (<= 0.1 h), Q3/P2disc, DG(2),
    # exact per-cell 606 x 606 patch inverses on the big-patch kernel
    ("C5-8", 8, 2, 2, 1 / 128, 0.1, 2, True),
]


@pytest.mark.parametrize("name,nc,r,k,tau,amp,n,smooth", C3D, ids=[c[0] for c in C3D])
def test_baseline_mesh_vmult_and_smoother_3d(ctx, stmg, name, nc, r, k, tau, amp, n, smooth):
    verts = o3.vertices(nc, nc, nc, amp, seed=3) if amp else None
    ref = o3.OracleLevel3(nc, nc, nc, r, k, tau, 1.0, 1.0, vertices=verts, smoother=smooth)
    lvl = stmg.Level3(ctx, nc, nc, nc, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL if smooth else stmg.SMOOTHER_NONE,
                      vertices=verts)
    assert lvl.size == ref.size
    rng = np.random.default_rng(41)
    x = rng.uniform(-1, 1, n * ref.size)
    b = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.mv)
    yr = ref.vmult_all(x, n, halo)
    y = torch.zeros(n * lvl.size, dtype=torch.float64, device="cuda")
    xd, hd = dev(x), dev(halo)
    lvl.vmult(xd, y, n, hd)
    err = rel_max(host(y), yr)
    assert err <= VMULT_TOL, (name, "vmult", err)
    if not smooth:
        return
    ur = ref.smooth_step_all(b, x, 0.8, n, halo)
    lvl.smooth_step(dev(b), xd, 0.8, n, hd, coupled=True)
    err = rel_max(host(xd), ur)
    assert err <= SMOOTH_TOL, (name, "smooth_step", err)
