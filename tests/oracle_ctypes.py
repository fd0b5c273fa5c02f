"""ctypes binding of the ORACLE (oracle/_build/liboracle.so) for the tests.

Test infrastructure only: the oracle is the CPU restatement of the reference
path (see oracle/include/oracle/oracle.hpp). Only tests/, the smoke check and
bench.py's CPU-baseline leg use it, always as the checker.
"""
from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parents[1]
ORACLE_DIR = ROOT / "oracle"
LIB = ORACLE_DIR / "_build" / "liboracle.so"
TESTS_BIN = ORACLE_DIR / "_build" / "oracle_tests"

_lib = None
_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)


def build_oracle() -> None:
    if not LIB.exists() or not TESTS_BIN.exists():
        subprocess.run(["make", "-C", str(ORACLE_DIR), "-j8"], check=True, capture_output=True)


def lib():
    global _lib
    if _lib is None:
        build_oracle()
        _lib = ctypes.CDLL(str(LIB))
        L = _lib
        L.oracle_last_error.restype = ctypes.c_char_p
        L.oracle_level_create.argtypes = [ctypes.c_int] * 3 + [ctypes.c_double] * 3 + [ctypes.c_int, ctypes.c_int,
                                                                                       ctypes.POINTER(_P)]
        L.oracle_level_destroy.argtypes = [_P]
        L.oracle_level_sizes.argtypes = [_P, ctypes.POINTER(ctypes.c_long)]
        L.oracle_apply_block.argtypes = [_P, _D, _D, ctypes.c_int]
        L.oracle_coupling_rhs.argtypes = [_P, _D, _D]
        L.oracle_step_health.argtypes = [_P, _D, _D]
        L.oracle_vmult_all.argtypes = [_P, _D, _D, ctypes.c_int, _D, ctypes.c_int]
        L.oracle_apply_additive.argtypes = [_P, _D, _D]
        L.oracle_smooth_step_all.argtypes = [_P, _D, _D, ctypes.c_double, ctypes.c_int, _D, ctypes.c_int]
        L.oracle_smooth_step_rows.argtypes = [_P, _D, _D, ctypes.c_double, ctypes.c_int, _D,
                                              ctypes.POINTER(ctypes.c_long), ctypes.c_long, _D, ctypes.c_int]
        L.oracle_patch_count.argtypes = [_P]
        L.oracle_patch_count.restype = ctypes.c_long
        L.oracle_patch_size.argtypes = [_P, ctypes.c_long]
        L.oracle_patch_size.restype = ctypes.c_long
        L.oracle_patch.argtypes = [_P, ctypes.c_long, ctypes.POINTER(ctypes.c_long), _D, _D]
        L.oracle_solver_create.argtypes = ([ctypes.c_int] * 4 + [ctypes.c_double] * 3 + [ctypes.c_int] * 3 +
                                           [ctypes.c_double, ctypes.c_int, ctypes.c_double, ctypes.c_double,
                                            ctypes.c_int, ctypes.POINTER(_P)])
        L.oracle_solver_destroy.argtypes = [_P]
        L.oracle_solver_info.argtypes = [_P, ctypes.POINTER(ctypes.c_long)]
        L.oracle_solver_n_steps.argtypes = [_P]
        L.oracle_solver_tau.argtypes = [_P]
        L.oracle_solver_tau.restype = ctypes.c_double
        L.oracle_level_apply_block.argtypes = [_P, ctypes.c_int, _D, _D]
        L.oracle_level_smooth_step.argtypes = [_P, ctypes.c_int, _D, _D, ctypes.c_double]
        L.oracle_level_restrict_residual.argtypes = [_P, ctypes.c_int, _D, _D, ctypes.c_int]
        L.oracle_level_prolongate_correction.argtypes = [_P, ctypes.c_int, _D, _D, ctypes.c_int]
        L.oracle_vcycle.argtypes = [_P, _D, _D]
        L.oracle_gmres.argtypes = [_P, _D, _D, ctypes.POINTER(ctypes.c_int), _D, ctypes.c_int]
        L.oracle_time_march_seeded.argtypes = [_P, _D, _D, ctypes.POINTER(ctypes.c_int), _D]
        L.oracle_assemble_rhs_manufactured.argtypes = [_P, ctypes.c_double, _D]
        L.oracle_time_march_manufactured.argtypes = [_P, _D, ctypes.POINTER(ctypes.c_int)]
        L.oracle_manufactured_errors.argtypes = [_P, _D, _D]
        L.oracle_interpolate_manufactured.argtypes = [_P, _D]
        L.oracle_time_march_cavity.argtypes = [_P, _D, ctypes.POINTER(ctypes.c_int)]
    return _lib


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def _chk(code):
    if code != 0:
        raise RuntimeError(f"oracle error {code}: {lib().oracle_last_error().decode()}")


class OracleLevel:
    """One operator level (+ optional smoother) on an nc x nc unit-square mesh."""

    def __init__(self, nc, r, k, tau, nu, gamma, smoother=0, build_smoother=True):
        h = _P()
        _chk(lib().oracle_level_create(nc, r, k, tau, nu, gamma, smoother, int(build_smoother), ctypes.byref(h)))
        self.h = h
        s = (ctypes.c_long * 7)()
        lib().oracle_level_sizes(h, s)
        self.n_slots, self.n_velocity, self.n_pressure, self.size, self.n_scalar, self.grid_x, self.n_patches = map(int, s)

    def apply_block(self, x, raw=False):
        y = np.zeros(self.size)
        _chk(lib().oracle_apply_block(self.h, _d(x), _d(y), int(raw)))
        return y

    def step_health(self, x):
        out = np.zeros(2)
        _chk(lib().oracle_step_health(self.h, _d(x), _d(out)))
        return float(out[0]), float(out[1])

    def coupling_rhs(self, v_prev):
        y = np.zeros(self.size)
        _chk(lib().oracle_coupling_rhs(self.h, _d(v_prev), _d(y)))
        return y

    def vmult_all(self, x, n, x_prev=None, threads=1):
        y = np.zeros_like(x)
        _chk(lib().oracle_vmult_all(self.h, _d(x), _d(y), n, _d(x_prev), threads))
        return y

    def smooth_step_rows(self, b, u, omega, n, rows, x_prev=None, threads=0):
        """smooth_step_all evaluated at `rows` (indices within one interval) of
        every interval: shape (n, len(rows)). With build_smoother == 2 only the
        patches containing a requested row are factored."""
        rows = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.zeros(n * rows.size)
        _chk(lib().oracle_smooth_step_rows(self.h, _d(b), _d(u), omega, n, _d(x_prev),
                                           rows.ctypes.data_as(ctypes.POINTER(ctypes.c_long)), rows.size, _d(out),
                                           threads))
        return out.reshape(n, rows.size)

    def apply_additive(self, r):
        y = np.zeros(self.size)
        _chk(lib().oracle_apply_additive(self.h, _d(r), _d(y)))
        return y

    def smooth_step_all(self, b, u, omega, n, x_prev=None, threads=1):
        u = u.copy()
        _chk(lib().oracle_smooth_step_all(self.h, _d(b), _d(u), omega, n, _d(x_prev), threads))
        return u

    def patch(self, i):
        n = lib().oracle_patch_size(self.h, i)
        dofs = (ctypes.c_long * n)()
        w = np.zeros(n)
        a = np.zeros(n * n)
        _chk(lib().oracle_patch(self.h, i, dofs, _d(w), _d(a)))
        return np.array(list(dofs)), w, a.reshape(n, n, order="F")

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_level_destroy(self.h)
            self.h = None


class OracleSolver:
    def __init__(self, refinements, r, k=-1, n_steps=0, t_end=1.0, nu=0.1, gamma=1.0, smoother=0, nu1=1, nu2=1,
                 omega=0.8, h_only=False, rtol=1e-8, atol=1e-14, maxit=200):
        h = _P()
        _chk(lib().oracle_solver_create(refinements, r, k, n_steps, t_end, nu, gamma, smoother, nu1, nu2, omega,
                                        int(h_only), rtol, atol, maxit, ctypes.byref(h)))
        self.h = h
        info = (ctypes.c_long * 400)()
        lib().oracle_solver_info(h, info)
        self.n_levels = int(info[0])
        self.levels = [dict(nx=int(info[1 + 5 * l]), r=int(info[2 + 5 * l]), k=int(info[3 + 5 * l]),
                            kind=int(info[4 + 5 * l]), size=int(info[5 + 5 * l])) for l in range(self.n_levels)]
        self.n_steps = lib().oracle_solver_n_steps(h)
        self.size = self.levels[-1]["size"]

    def apply_block(self, l, x):
        y = np.zeros(self.levels[l]["size"])
        _chk(lib().oracle_level_apply_block(self.h, l, _d(x), _d(y)))
        return y

    def smooth_step(self, l, b, u, omega):
        u = u.copy()
        _chk(lib().oracle_level_smooth_step(self.h, l, _d(b), _d(u), omega))
        return u

    def restrict_residual(self, l, fine, project=True):
        c = np.zeros(self.levels[l - 1]["size"])
        _chk(lib().oracle_level_restrict_residual(self.h, l, _d(fine), _d(c), int(project)))
        return c

    def prolongate_correction(self, l, coarse, project=True):
        f = np.zeros(self.levels[l]["size"])
        _chk(lib().oracle_level_prolongate_correction(self.h, l, _d(coarse), _d(f), int(project)))
        return f

    def vcycle(self, b):
        x = np.zeros(self.size)
        _chk(lib().oracle_vcycle(self.h, _d(b), _d(x)))
        return x

    def gmres(self, b):
        x = np.zeros(self.size)
        it = ctypes.c_int(0)
        hist = np.zeros(512)
        _chk(lib().oracle_gmres(self.h, _d(b), _d(x), ctypes.byref(it), _d(hist), 512))
        return x, it.value, hist[: it.value + 1]

    def time_march(self, F):
        X = np.zeros(self.n_steps * self.size)
        it = (ctypes.c_int * self.n_steps)()
        thr = np.zeros(1)
        _chk(lib().oracle_time_march_seeded(self.h, _d(F), _d(X), it, _d(thr)))
        return X, list(it), float(thr[0])

    def assemble_rhs_manufactured(self, t_start):
        out = np.zeros(self.size)
        _chk(lib().oracle_assemble_rhs_manufactured(self.h, t_start, _d(out)))
        return out

    def time_march_manufactured(self):
        X = np.zeros(self.n_steps * self.size)
        it = (ctypes.c_int * self.n_steps)()
        _chk(lib().oracle_time_march_manufactured(self.h, _d(X), it))
        return X, list(it)

    def time_march_cavity(self):
        X = np.zeros(self.n_steps * self.size)
        it = (ctypes.c_int * self.n_steps)()
        _chk(lib().oracle_time_march_cavity(self.h, _d(X), it))
        return X, list(it)

    def interpolate_manufactured(self):
        X = np.zeros(self.n_steps * self.size)
        _chk(lib().oracle_interpolate_manufactured(self.h, _d(X)))
        return X

    def manufactured_errors(self, X):
        out = np.zeros(5)
        _chk(lib().oracle_manufactured_errors(self.h, _d(np.ascontiguousarray(X)), _d(out)))
        return out

    def __del__(self):
        if getattr(self, "h", None):
            lib().oracle_solver_destroy(self.h)
            self.h = None


def seeded(n, seed):
    """Seeded uniform[-1, 1] FP64 vector (numpy PCG64)."""
    return np.random.default_rng(seed).uniform(-1.0, 1.0, n)


def make_consistent(v, n_slots, nsc, gx, n_pressure, ncells, np_cell, n_intervals=1):
    """Zero constrained velocity entries and project each slot's pressure to
    mean zero (dof_space.cpp:62-68, 110-119): the consistent seeded RHS of
    SURVEY.md section 0.4."""
    gy = nsc // gx
    mv = 2 * nsc
    isz = n_slots * (mv + n_pressure)
    v = v.reshape(n_intervals, isz)
    bnd = np.zeros((gy, gx), dtype=bool)
    bnd[0, :] = bnd[-1, :] = bnd[:, 0] = bnd[:, -1] = True
    bnd = bnd.ravel()
    for n in range(n_intervals):
        for a in range(n_slots):
            for c in range(2):
                seg = v[n, a * mv + c * nsc: a * mv + (c + 1) * nsc]
                seg[bnd] = 0.0
            p = v[n, n_slots * mv + a * n_pressure: n_slots * mv + (a + 1) * n_pressure].reshape(ncells, np_cell)
            p[:, 0] -= p[:, 0].mean()
    return v.reshape(-1)
