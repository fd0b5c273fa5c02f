"""CPU tier: the oracle reproduces the committed golden vectors
(tests/golden/*.npz, written by tests/golden/make_golden.py), so a change of
the checker itself cannot silently move the target the GPU parity tests aim
at. Tolerance 1e-12 relative max-norm: the oracle is compiled -march=native,
so FMA contraction may differ between hosts."""
from pathlib import Path

import numpy as np
import pytest

import oracle3_ctypes as o3
import oracle_ctypes as oc

GOLD = Path(__file__).resolve().parent / "golden"


def _rel(a, b):
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def _cases(prefix_filter):
    import importlib.util

    spec = importlib.util.spec_from_file_location("make_golden", GOLD / "make_golden.py")
    mg = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(mg)
    return mg


MG = _cases(None)


def test_every_golden_file_is_committed():
    names = set(MG.CASES_2D) | set(MG.CASES_3D) | {"c1_fgmres_stmg_v22"}
    assert {f.stem for f in GOLD.glob("*.npz")} == names


@pytest.mark.parametrize("name", sorted(MG.CASES_2D))
def test_oracle_reproduces_golden_2d(oracle, name):
    g = np.load(GOLD / f"{name}.npz")
    nc, r, k, tau, nu, gamma, kind, n = MG.CASES_2D[name]
    assert np.array_equal(g["case"], np.array(MG.CASES_2D[name], dtype=np.float64))
    ref = oc.OracleLevel(nc, r, k, tau, nu, gamma, kind)
    assert g["x"].size == n * ref.size
    assert _rel(ref.vmult_all(g["x"], n, g["halo"]), g["vmult"]) <= 1e-12
    assert _rel(ref.smooth_step_all(g["b"], g["x"], MG.OMEGA, n, g["halo"]), g["smooth_step"]) <= 1e-12
    assert _rel(ref.apply_additive(g["b"][:ref.size]), g["apply_additive"]) <= 1e-12


@pytest.mark.parametrize("name", sorted(MG.CASES_3D))
def test_oracle_reproduces_golden_3d(oracle, name):
    g = np.load(GOLD / f"{name}.npz")
    nx, ny, nz, r, k, tau, gamma, amp, n = MG.CASES_3D[name]
    verts = g["vertices"] if amp else None
    ref = o3.OracleLevel3(nx, ny, nz, r, k, tau, 1.0, gamma, vertices=verts)
    assert _rel(ref.vmult_all(g["x"], n, g["halo"]), g["vmult"]) <= 1e-12
    assert _rel(ref.smooth_step_all(g["b"], g["x"], MG.OMEGA, n, g["halo"]), g["smooth_step"]) <= 1e-12


def test_oracle_reproduces_golden_solve(oracle):
    g = np.load(GOLD / "c1_fgmres_stmg_v22.npz")
    s = MG.SOLVE
    rs = oc.OracleSolver(s["refinements"], s["r"], s["k"], n_steps=s["n_steps"], nu=s["nu"], gamma=s["gamma"],
                         nu1=s["nu1"], nu2=s["nu2"])
    x, its, _ = rs.gmres(g["rhs"])
    assert its == int(g["iterations"][0])
    assert np.linalg.norm(x - g["solution"]) <= 1e-10 * np.linalg.norm(g["solution"])
