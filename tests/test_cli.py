"""The drop-in command line (tools/stmg_cli.cpp -> _build/stmg_gpu) against the
reference's `stmg` behaviour (tools/stmg.cpp): dotted flags, flat-INI config
with command-line precedence, exit code 3 for a bad config, the hierarchy
table, and (GPU) the convergence / robustness / cavity / selftest runs."""
import subprocess

import numpy as np
import pytest

import oracle_ctypes as oc
from paper_2502_09159_b200 import build

CLI = build.BUILD / "stmg_gpu"


def run(*args, timeout=600):
    return subprocess.run([str(CLI), *args], capture_output=True, text=True, timeout=timeout)


@pytest.fixture(scope="module", autouse=True)
def cli_built():
    if not CLI.exists():
        build.build()
    assert CLI.exists()


@pytest.mark.parametrize("c,r,mode", [(3, 2, "hp"), (2, 4, "hp"), (2, 2, "h_only")])
def test_hierarchy_table_matches_oracle_plan(oracle, c, r, mode):
    res = run("hierarchy", "--mesh.refinements", str(c), "--discretization.r", str(r), "--mg.mode", mode)
    assert res.returncode == 0, res.stderr
    rows = [ln for ln in res.stdout.splitlines()[2:] if ln.strip()]
    ref = oc.OracleSolver(c, r, -1, h_only=(mode == "h_only"))
    assert len(rows) == ref.n_levels
    for line, lvl in zip(rows, reversed(ref.levels)):
        cols = [p.split() for p in line.split("|")]
        assert int(cols[1][1]) == lvl["r"] and int(cols[2][1]) == lvl["k"]
        assert abs(float(cols[1][0]) - 1.0 / lvl["nx"]) < 1e-12


def test_config_file_precedence_and_errors(tmp_path):
    good = tmp_path / "run.ini"
    good.write_text("# study\n[mesh]\nrefinements = 1\n[discretization]\nr = 2\n")
    res = run("hierarchy", "--config", str(good))
    assert res.returncode == 0 and len([ln for ln in res.stdout.splitlines()[2:] if ln.strip()]) == 3
    # a command-line flag wins over the config value (stmg.cpp:160-170)
    res2 = run("hierarchy", "--config", str(good), "--mesh.refinements", "3")
    assert res2.returncode == 0 and len([ln for ln in res2.stdout.splitlines()[2:] if ln.strip()]) == 5
    bad = tmp_path / "bad.ini"
    bad.write_text("[mesh]\nrefinements = 1\nbogus = 2\n")
    assert run("hierarchy", "--config", str(bad)).returncode == 3
    assert run("hierarchy", "--config", str(tmp_path / "missing.ini")).returncode == 3
    assert run("hierarchy", "--no.such_flag", "1").returncode != 0


@pytest.mark.gpu
def test_convergence_subcommand_runs_on_gpu(tmp_path):
    csv = tmp_path / "conv.csv"
    res = run("convergence", "--r_list", "2", "--c_list", "1,2", "--output.csv_path", str(csv))
    assert res.returncode == 0, res.stderr
    rows = np.loadtxt(csv, delimiter=",", skiprows=1)
    assert rows.shape == (2, 11)
    assert rows[1, 3] < rows[0, 3]      # velocity L2 error decreases with h
    assert rows[1, 4] > 2.5             # EOC of the Q3 velocity


@pytest.mark.gpu
def test_cavity_robustness_selftest_on_gpu(tmp_path):
    res = run("cavity", "--mesh.refinements", "2", "--discretization.r", "1", "--problem.nu", "1.0")
    assert res.returncode == 0, res.stderr
    assert "avg GMRES iterations" in res.stdout
    res = run("robustness", "--r_list", "1", "--c_list", "2", "--n_sm_list", "1,2", "--mg.smoother", "vertex_star")
    assert res.returncode == 0, res.stderr
    assert len(res.stdout.strip().splitlines()) == 3
    res = run("selftest")
    assert res.returncode == 0, res.stdout + res.stderr
    assert "[FAIL]" not in res.stdout
