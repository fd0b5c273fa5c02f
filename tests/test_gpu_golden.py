"""GPU tier: the CUDA path, called through the C ABI, against the committed
golden vectors (tests/golden/*.npz; generator tests/golden/make_golden.py).
Tolerances are BASELINE.json's: vmult relative max-norm <= 1e-12, one
smoother step <= 1e-10, FGMRES iterations +-1 and solution relative L2
<= 1e-8. Nothing here calls the oracle."""
from pathlib import Path

import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"


def _constants():
    # only the case tables: importing the generator would import the oracle
    src = (GOLD / "make_golden.py").read_text()
    ns = {}
    start = src.index("# name: (nc, r, k")
    stop = src.index("def make_2d")
    exec(src[start:stop], ns)
    return ns


C = _constants()


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _cuda(a):
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


@pytest.mark.parametrize("name", sorted(C["CASES_2D"]))
def test_gpu_matches_golden_2d(stmg, ctx, name):
    g = np.load(GOLD / f"{name}.npz")
    nc, r, k, tau, nu, gamma, kind, n = C["CASES_2D"][name]
    lvl = stmg.Level(ctx, nc, nc, r, k, tau, nu, gamma, stmg.SMOOTHER_CELL if kind == 0 else stmg.SMOOTHER_VERTEX_STAR)
    assert n * lvl.size == g["x"].size
    y = torch.zeros(n * lvl.size, dtype=torch.float64, device="cuda")
    lvl.vmult(_cuda(g["x"]), y, n, _cuda(g["halo"]))
    assert _rel(y.cpu().numpy(), g["vmult"]) <= 1e-12
    u = _cuda(g["x"])
    lvl.smooth_step(_cuda(g["b"]), u, C["OMEGA"], n, _cuda(g["halo"]), coupled=True)
    assert _rel(u.cpu().numpy(), g["smooth_step"]) <= 1e-10
    z = torch.zeros(lvl.size, dtype=torch.float64, device="cuda")
    lvl.apply_additive(_cuda(g["b"][:lvl.size]), z)
    assert _rel(z.cpu().numpy(), g["apply_additive"]) <= 1e-10


@pytest.mark.parametrize("name", sorted(C["CASES_3D"]))
def test_gpu_matches_golden_3d(stmg, ctx, name):
    g = np.load(GOLD / f"{name}.npz")
    nx, ny, nz, r, k, tau, gamma, amp, n = C["CASES_3D"][name]
    verts = np.ascontiguousarray(g["vertices"]) if amp else None
    lvl = stmg.Level3(ctx, nx, ny, nz, r, k, tau, 1.0, gamma, stmg.SMOOTHER_CELL, vertices=verts)
    assert n * lvl.size == g["x"].size
    y = torch.zeros(n * lvl.size, dtype=torch.float64, device="cuda")
    lvl.vmult(_cuda(g["x"]), y, n, _cuda(g["halo"]))
    assert _rel(y.cpu().numpy(), g["vmult"]) <= 1e-12
    u = _cuda(g["x"])
    lvl.smooth_step(_cuda(g["b"]), u, C["OMEGA"], n, _cuda(g["halo"]), coupled=True)
    assert _rel(u.cpu().numpy(), g["smooth_step"]) <= 1e-10


def test_gpu_matches_golden_solve(stmg, ctx):
    g = np.load(GOLD / "c1_fgmres_stmg_v22.npz")
    s = C["SOLVE"]
    sol = stmg.Solver(ctx, s["refinements"], s["r"], s["k"], n_steps=s["n_steps"], nu=s["nu"], gamma=s["gamma"],
                      nu1=s["nu1"], nu2=s["nu2"])
    x = torch.zeros(g["rhs"].size, dtype=torch.float64, device="cuda")
    its, _ = sol.gmres(_cuda(g["rhs"]), x)
    assert abs(its - int(g["iterations"][0])) <= 1
    xs = x.cpu().numpy()
    assert np.linalg.norm(xs - g["solution"]) <= 1e-8 * np.linalg.norm(g["solution"])
