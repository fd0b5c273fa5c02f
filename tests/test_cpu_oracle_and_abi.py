"""CPU tier: the oracle against the reference's known-answer tests, the C ABI
surface, and the product's host-side setup (hierarchy plan, Vanka patch
classes and their inverses) against the oracle. No GPU needed."""
import ctypes
import subprocess

import numpy as np
import pytest

import oracle_ctypes as oc

SUITES = ["quadrature", "time_basis", "mesh", "dof_space", "st_operator", "vanka", "transfer", "hierarchy", "solver"]


@pytest.mark.parametrize("suite", SUITES)
def test_oracle_pinned_to_reference_known_answers(oracle, suite):
    """oracle/tests/oracle_tests.cpp ports the reference doctest suites
    (tests/test_*.cpp) with their tolerances."""
    res = subprocess.run([str(oc.TESTS_BIN), suite], capture_output=True, text=True, timeout=600)
    assert res.returncode == 0, res.stdout + res.stderr
    assert "[PASS]" in res.stdout and "[FAIL]" not in res.stdout


@pytest.mark.slow
def test_oracle_reproduces_paper_table1(oracle):
    """acceptance.cpp:383-420: r=4 velocity/pressure errors within a factor 2
    of PAPER.md Table 1 and EOC within 0.3 (full solve chain)."""
    res = subprocess.run([str(oc.TESTS_BIN), "acceptance_table1"], capture_output=True, text=True, timeout=900)
    assert res.returncode == 0, res.stdout


def test_library_exports_every_header_symbol(stmg):
    lib = stmg.load_library()
    syms = stmg.exported_symbols()
    assert len(syms) >= 30
    for s in syms:
        assert hasattr(lib, s), s
    assert b"sm_100a" in lib.stmg_version()


def test_library_is_sm100a_cubin(stmg):
    out = subprocess.run(["cuobjdump", "--list-elf", str(stmg.LIB_PATH)], capture_output=True, text=True)
    assert "sm_100a" in out.stdout


@pytest.mark.parametrize("refinements,r,k,h_only", [(4, 1, 1, False), (2, 2, 2, False), (3, 4, -1, False),
                                                     (2, 3, 1, False), (2, 2, -1, True), (0, 1, 1, False)])
def test_hierarchy_plan_matches_oracle(oracle, stmg, refinements, r, k, h_only):
    plan = stmg.plan_levels(refinements, r, k, h_only=h_only)
    ref = oc.OracleSolver(refinements, r, k, h_only=h_only)
    assert plan["n_steps"] == ref.n_steps
    assert len(plan["levels"]) == ref.n_levels
    for mine, theirs in zip(plan["levels"], ref.levels):
        assert (mine["nx"], mine["r"], mine["k"], mine["size"]) == (theirs["nx"], theirs["r"], theirs["k"],
                                                                    theirs["size"])
        assert stmg.TRANSFER_KINDS.index(mine["kind"]) == theirs["kind"]


def test_invalid_arguments_map_to_einval(stmg):
    lib = stmg.load_library()
    out = (ctypes.c_int64 * 64)()
    assert lib.stmg_plan_levels(2, 0, 1, 0, 1.0, 0, out) == 1  # r < 1 -> std::invalid_argument
    assert lib.stmg_patch_info(4, 4, 9, 1, 0.25, 0.1, 1.0, 0, out, None, 0) == 1


@pytest.mark.parametrize("nc,r,k,kind", [(4, 1, 1, 0), (4, 2, 2, 0), (8, 1, 1, 1), (4, 2, 1, 1), (1, 2, 1, 0)])
def test_patch_classes_invert_oracle_local_matrices(oracle, stmg, nc, r, k, kind):
    """Every oracle patch matrix R_T S R_T^T (vanka.cpp:92-165) is inverted by
    the product's class inverse (pseudo-inverse for the whole-domain patch)."""
    tau, nu, gamma = 0.25, 0.1, 1.0
    info = stmg.patch_info(nc, nc, r, k, tau, nu, gamma, kind)
    lvl = oc.OracleLevel(nc, r, k, tau, nu, gamma, kind)
    assert info["n_patches"] == lvl.n_patches
    sizes = sorted({lvl.patch(i)[0].size for i in range(lvl.n_patches)})
    assert sorted(set(info["class_sizes"][: info["n_classes"]])) == sizes
    assert info["sum_nt2"] == sum(lvl.patch(i)[0].size ** 2 for i in range(lvl.n_patches))
    lib = stmg.load_library()
    # match every oracle patch to a product class by its local matrix
    invs = []
    for c in range(info["n_classes"]):
        n = info["class_sizes"][c]
        buf = np.zeros(n * n)
        out = (ctypes.c_int64 * 64)()
        assert lib.stmg_patch_info(nc, nc, r, k, tau, nu, gamma, kind, out,
                                   buf.ctypes.data_as(ctypes.POINTER(ctypes.c_double)), c) == 0
        invs.append(buf.reshape(n, n))
    for i in range(lvl.n_patches):
        dofs, w, A = lvl.patch(i)
        best = min((np.abs(inv @ A - np.eye(A.shape[0])).max() for inv in invs if inv.shape == A.shape),
                   default=np.inf)
        if nc == 1:  # whole-domain patch: pseudo-inverse, A^+ A is a projector
            inv = [v for v in invs if v.shape == A.shape][0]
            assert np.abs(A @ inv @ A - A).max() < 1e-10 * np.abs(A).max()
        else:
            assert best < 1e-9, (i, best)


def test_binding_rejects_host_and_mistyped_tensors(stmg):
    """The binding checks every vector before it reaches the C ABI (no GPU:
    a CPU tensor is refused as such; sizes are checked on the GPU tier)."""
    import torch

    with pytest.raises(ValueError, match="CUDA"):
        stmg._ptr(torch.zeros(4, dtype=torch.float64))
    with pytest.raises(ValueError, match="float64"):
        stmg._hptr(np.zeros(4, dtype=np.int64))
    with pytest.raises(ValueError, match="elements"):
        stmg._hptr(np.zeros(4), 5)
    assert stmg._ptr(None) is None


def test_tuning_hook_validates_without_gpu(stmg):
    lib = stmg.load_library()
    assert lib.stmg_set_tuning(b"vanka_group", 4) == 0
    assert lib.stmg_set_tuning(b"vanka_group", 0) == 0
    assert lib.stmg_set_tuning(b"bogus", 1) == 1
    assert lib.stmg_set_tuning(b"vanka_big_group", 5000) == 1


@pytest.mark.parametrize("nc,r,k,kind", [(8, 2, 2, 0), (8, 1, 1, 1), (4, 1, 2, 1)])
def test_oracle_row_subset_smoother_equals_full_sweep(oracle, nc, r, k, kind):
    """oracle_smooth_step_rows (patches factored on demand, the checker of
    the BASELINE-size GPU parity tests) returns the full sweep's values,
    bitwise, at the requested rows."""
    tau = 1 / 16
    full = oc.OracleLevel(nc, r, k, tau, 1.0, 1.0, kind)
    lazy = oc.OracleLevel(nc, r, k, tau, 1.0, 1.0, kind, build_smoother=2)
    n = 3
    u = oc.seeded(n * full.size, 21)
    b = oc.seeded(n * full.size, 22)
    halo = oc.seeded(full.n_velocity, 23)
    ref = full.smooth_step_all(b, u, 0.8, n, halo).reshape(n, full.size)
    rows = np.unique(np.random.default_rng(5).integers(0, full.size, 97))
    got = lazy.smooth_step_rows(b, u, 0.8, n, rows, halo)
    assert np.array_equal(got, ref[:, rows])
