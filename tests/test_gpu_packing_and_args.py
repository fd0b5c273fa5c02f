"""GPU tier: launch packings the size heuristics never pick on small meshes,
and the binding's argument checks.

* Intervals per block of the item Vanka kernels (vanka.cu): several intervals
  packed into one tile column set (patch = j / ng, n = n0 + j - patch * ng)
  and a ragged last interval group (6 intervals in groups of 4). Forced with
  the stmg_set_tuning hook, for the 128-row DMMA kernel (3D k = 0, n_T <= 85),
  the 176-row split (3D r = 1, k = 1, n_T = 170; 2D r = 2, k = 3, n_T = 152)
  and the L2-streamed big-patch kernel (3D r = 1, k = 2, n_T = 255; 2D r = 3,
  k = 2, n_T = 180). Smoother step against the oracle, <= 1e-10
  (vanka.cpp:196-233).
* Short, mistyped or foreign-device tensors raise ValueError before the C ABI
  sees them.
"""
import numpy as np
import pytest
import torch

import oracle3_ctypes as o3
import oracle_ctypes as oc

pytestmark = pytest.mark.gpu


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.fixture
def tuning(stmg):
    lib = stmg.load_library()

    def set_groups(dmma, big):
        assert lib.stmg_set_tuning(b"vanka_group", dmma) == 0
        assert lib.stmg_set_tuning(b"vanka_big_group", big) == 0

    yield set_groups
    set_groups(0, 0)


CASES3 = [  # nx, ny, nz, r, k, amp  (kernel)
    (3, 2, 2, 1, 0, 0.0),  # 128-row DMMA item kernel
    (3, 2, 2, 1, 1, 0.0),  # 176-row split
    (2, 2, 3, 1, 1, 0.1),  # 176-row split, deformed (one class per cell)
    (2, 2, 2, 1, 2, 0.0),  # big-patch kernel
]


@pytest.mark.parametrize("group", [2, 3, 4])
@pytest.mark.parametrize("nx,ny,nz,r,k,amp", CASES3)
def test_smooth_step3_interval_groups(stmg, ctx, oracle, tuning, group, nx, ny, nz, r, k, amp):
    verts = o3.vertices(nx, ny, nz, amp, seed=5) if amp else None
    tau = 1.0 / 8
    ref = o3.OracleLevel3(nx, ny, nz, r, k, tau, 1.0, 1.0, vertices=verts)
    lvl = stmg.Level3(ctx, nx, ny, nz, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL, vertices=verts)
    rng = np.random.default_rng(40 + group)
    n = 6  # not a multiple of 4: ragged last group
    u = rng.uniform(-1, 1, n * ref.size)
    b = rng.uniform(-1, 1, n * ref.size)
    halo = rng.uniform(-1, 1, ref.mv)
    tuning(group, group)
    ug = _cuda(u)
    lvl.smooth_step(_cuda(b), ug, 0.8, n, _cuda(halo), coupled=True)
    assert _rel(ug.cpu().numpy(), ref.smooth_step_all(b, u, 0.8, n, halo)) <= 1e-10


@pytest.mark.parametrize("group", [2, 4])
@pytest.mark.parametrize("nc,r,k", [(4, 2, 3), (4, 3, 2)])
def test_smooth_step2_interval_groups(stmg, ctx, oracle, tuning, group, nc, r, k):
    """2D patches beyond 128 rows run on the item kernels too."""
    tau = 0.125
    ref = oc.OracleLevel(nc, r, k, tau, 1.0, 1.0, 0)
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, 1.0, 1.0, stmg.SMOOTHER_CELL)
    n = 6
    u = oc.seeded(n * ref.size, 7)
    b = oc.seeded(n * ref.size, 8)
    halo = oc.seeded(ref.n_velocity, 9)
    tuning(group, group)
    ug = _cuda(u)
    lvl.smooth_step(_cuda(b), ug, 0.8, n, _cuda(halo), coupled=True)
    assert _rel(ug.cpu().numpy(), ref.smooth_step_all(b, u, 0.8, n, halo)) <= 1e-10


def test_tuning_rejects_bad_keys(stmg):
    lib = stmg.load_library()
    assert lib.stmg_set_tuning(b"no_such_key", 1) == 1
    assert lib.stmg_set_tuning(b"vanka_group", -1) == 1
    assert lib.stmg_set_tuning(b"vanka_group", 0) == 0


def test_binding_rejects_bad_tensors(stmg, ctx):
    lvl = stmg.Level(ctx, 4, 4, 1, 1, 0.25, 1.0, 1.0, stmg.SMOOTHER_CELL)
    x = torch.zeros(2 * lvl.size, dtype=torch.float64, device="cuda")
    y = torch.zeros(2 * lvl.size, dtype=torch.float64, device="cuda")
    lvl.vmult(x, y, 2)  # fits
    with pytest.raises(ValueError, match="elements"):
        lvl.vmult(x, y, 3)  # too short for 3 intervals
    with pytest.raises(ValueError, match="float64"):
        lvl.vmult(x.to(torch.int64), y, 1)
    with pytest.raises(ValueError, match="float64"):
        lvl.vmult(x.to(torch.complex64), y, 1)
    with pytest.raises(ValueError, match="elements"):
        lvl.vmult(x, y, 1, torch.zeros(lvl.n_velocity - 1, dtype=torch.float64, device="cuda"))
    with pytest.raises(ValueError, match="CUDA"):
        lvl.vmult(x.cpu(), y, 1)
    with pytest.raises(ValueError, match="elements"):
        lvl.smooth_step(x, y, 0.8, 2, work=torch.zeros(lvl.size, dtype=torch.float64, device="cuda"))
    l3 = stmg.Level3(ctx, 2, 2, 2, 1, 1, 0.25, 1.0, 1.0, stmg.SMOOTHER_CELL)
    x3 = torch.zeros(l3.size, dtype=torch.float64, device="cuda")
    with pytest.raises(ValueError, match="elements"):
        l3.vmult(x3, x3.clone(), 2)
