"""ctypes binding of the ORACLE's 3D restatement (oracle/src/st3d.cpp) for the
tests. Test infrastructure only (see oracle_ctypes.py)."""
from __future__ import annotations

import ctypes

import numpy as np

import oracle_ctypes as oc

_P = ctypes.c_void_p
_D = ctypes.POINTER(ctypes.c_double)
_I = ctypes.c_int
_F = ctypes.c_double
_set = False


def lib():
    global _set
    L = oc.lib()
    if not _set:
        L.o3_last_error.restype = ctypes.c_char_p
        L.o3_level_create.argtypes = [_I] * 5 + [_F] * 3 + [_D, _I, ctypes.POINTER(_P)]
        L.o3_level_destroy.argtypes = [_P]
        L.o3_level_sizes.argtypes = [_P, ctypes.POINTER(ctypes.c_long)]
        L.o3_apply_block.argtypes = [_P, _D, _D, _I]
        L.o3_vmult_all.argtypes = [_P, _D, _D, _I, _D]
        L.o3_smooth_step_all.argtypes = [_P, _D, _D, _F, _I, _D]
        L.o3_patch_count.argtypes = [_P]
        L.o3_patch_count.restype = ctypes.c_long
        L.o3_project_mean_zero.argtypes = [_P, _D]
        L.o3_project_residual.argtypes = [_P, _D]
        L.o3_hier_create.argtypes = [_I] * 6 + [_F] * 3 + [_I, _I, _D, _I, _I, _F, ctypes.POINTER(_P)]
        L.o3_hier_destroy.argtypes = [_P]
        L.o3_hier_info.argtypes = [_P, ctypes.POINTER(ctypes.c_long)]
        L.o3_hier_level.argtypes = [_P, _I]
        L.o3_hier_level.restype = _P
        L.o3_hier_prolongate.argtypes = [_P, _I, _D, _D, _I]
        L.o3_hier_restrict.argtypes = [_P, _I, _D, _D, _I]
        L.o3_hier_coarse_forward.argtypes = [_P, _D, _D, _I]
        L.o3_hier_vcycle.argtypes = [_P, _D, _D, _I]
        L.o3_hier_fgmres.argtypes = [_P, _D, _D, _I, _F, _I, ctypes.POINTER(_I)]
        L.o3_direct_time_march.argtypes = [_P, _D, _D, _I]
        L.o3_set_kmin.argtypes = [_I]
        _set = True
    return L


def _d(a):
    if a is None:
        return None
    assert a.dtype == np.float64 and a.flags["C_CONTIGUOUS"]
    return a.ctypes.data_as(_D)


def _chk(code):
    if code != 0:
        raise RuntimeError(f"oracle3 error {code}: {lib().o3_last_error().decode()}")


class OracleLevel3:
    def __init__(self, nx, ny, nz, r, k, tau, nu, gamma, vertices=None, smoother=True, _borrowed=None):
        if _borrowed is not None:
            self.h, self.owned = _borrowed, False
        else:
            h = _P()
            _chk(lib().o3_level_create(nx, ny, nz, r, k, tau, nu, gamma, _d(vertices), 0 if smoother else -1,
                                       ctypes.byref(h)))
            self.h, self.owned = h, True
        out = (ctypes.c_long * 9)()
        lib().o3_level_sizes(self.h, out)
        (self.S, self.mv, self.mp, self.size, self.nsc, self.gx, self.gy, self.gz, self.np) = [int(v) for v in out]

    def apply_block(self, x, raw=False):
        y = np.zeros(self.size)
        _chk(lib().o3_apply_block(self.h, _d(x), _d(y), int(raw)))
        return y

    def vmult_all(self, x, n, x_prev=None):
        y = np.zeros(n * self.size)
        _chk(lib().o3_vmult_all(self.h, _d(x), _d(y), n, _d(x_prev)))
        return y

    def smooth_step_all(self, b, u, omega, n, x_prev=None):
        u = u.copy()
        _chk(lib().o3_smooth_step_all(self.h, _d(b), _d(u), omega, n, _d(x_prev)))
        return u

    def project_mean_zero(self, p):
        p = p.copy()
        _chk(lib().o3_project_mean_zero(self.h, _d(p)))
        return p

    def project_residual(self, p):
        p = p.copy()
        _chk(lib().o3_project_residual(self.h, _d(p)))
        return p

    def direct_time_march(self, b, n):
        x = np.zeros(n * self.size)
        _chk(lib().o3_direct_time_march(self.h, _d(b), _d(x), n))
        return x

    def __del__(self):
        if getattr(self, "owned", False) and self.h:
            lib().o3_level_destroy(self.h)
            self.h = None


class OracleHier3:
    def __init__(self, nx, ny, nz, r, k, N, t_end=1.0, nu=1.0, gamma=1.0, n_hcoarse=1, time_coarsen=True,
                 vertices=None, nu1=2, nu2=2, omega=0.8, k_min=0):
        lib().o3_set_kmin(k_min)
        h = _P()
        _chk(lib().o3_hier_create(nx, ny, nz, r, k, N, t_end, nu, gamma, n_hcoarse, int(time_coarsen), _d(vertices),
                                  nu1, nu2, omega, ctypes.byref(h)))
        self.h = h
        out = (ctypes.c_long * (1 + 7 * 32))()
        lib().o3_hier_info(h, out)
        self.n_levels = int(out[0])
        self.levels = [dict(nx=int(out[1 + 7 * l]), ny=int(out[2 + 7 * l]), nz=int(out[3 + 7 * l]),
                            r=int(out[4 + 7 * l]), k=int(out[5 + 7 * l]), tshift=int(out[6 + 7 * l]),
                            size=int(out[7 + 7 * l])) for l in range(self.n_levels)]
        self.level = [OracleLevel3(0, 0, 0, 0, 0, 0, 0, 0, _borrowed=lib().o3_hier_level(h, l))
                      for l in range(self.n_levels)]

    def prolongate(self, l, xc, nc):
        nf = 2 * nc if self.levels[l - 1]["tshift"] > self.levels[l]["tshift"] else nc
        xf = np.zeros(nf * self.levels[l]["size"])
        _chk(lib().o3_hier_prolongate(self.h, l, _d(xc), _d(xf), nc))
        return xf

    def restrict(self, l, xf, nc):
        xc = np.zeros(nc * self.levels[l - 1]["size"])
        _chk(lib().o3_hier_restrict(self.h, l, _d(xf), _d(xc), nc))
        return xc

    def coarse_forward(self, b, n):
        x = np.zeros(n * self.levels[0]["size"])
        _chk(lib().o3_hier_coarse_forward(self.h, _d(b), _d(x), n))
        return x

    def vcycle(self, b, n):
        x = np.zeros(n * self.levels[-1]["size"])
        _chk(lib().o3_hier_vcycle(self.h, _d(b), _d(x), n))
        return x

    def fgmres(self, b, n, rtol=1e-8, maxit=200):
        x = np.zeros(n * self.levels[-1]["size"])
        it = _I(0)
        _chk(lib().o3_hier_fgmres(self.h, _d(b), _d(x), n, rtol, maxit, ctypes.byref(it)))
        return x, int(it.value)

    def __del__(self):
        if getattr(self, "h", None):
            lib().o3_hier_destroy(self.h)
            self.h = None


def boundary_mask3(gx, gy, gz):
    m = np.zeros((gz, gy, gx), dtype=bool)
    m[0], m[-1], m[:, 0], m[:, -1], m[:, :, 0], m[:, :, -1] = True, True, True, True, True, True
    return m.ravel()


def make_consistent3(v, lvl, n_intervals=1, pmean=None):
    """Zero constrained velocity rows and remove each slot's pressure component
    along the left null vector (the constant-mode coefficients):
    the consistent seeded RHS, 3D (= mean zero on Cartesian meshes)."""
    v = v.reshape(n_intervals, lvl.size).copy()
    bnd = boundary_mask3(lvl.gx, lvl.gy, lvl.gz)
    for n in range(n_intervals):
        for a in range(lvl.S):
            for c in range(3):
                seg = v[n, a * lvl.mv + c * lvl.nsc: a * lvl.mv + (c + 1) * lvl.nsc]
                seg[bnd] = 0.0
            p0 = lvl.S * lvl.mv + a * lvl.mp
            v[n, p0: p0 + lvl.mp] = lvl.project_residual(np.ascontiguousarray(v[n, p0: p0 + lvl.mp]))
    return v.reshape(-1)


def vertices(nx, ny, nz, amp=0.0, seed=5):
    """Unit-cube vertex coordinates with interior vertices moved by a seeded
    uniform displacement of at most amp * h (BASELINE C5)."""
    rng = np.random.default_rng(seed)
    z, y, x = np.meshgrid(np.arange(nz + 1) / nz, np.arange(ny + 1) / ny, np.arange(nx + 1) / nx, indexing="ij")
    v = np.stack([x, y, z], axis=-1).astype(np.float64)
    if amp > 0:
        d = rng.uniform(-1, 1, v.shape) * amp * np.array([1 / nx, 1 / ny, 1 / nz])
        interior = np.zeros(v.shape[:3], dtype=bool)
        interior[1:-1, 1:-1, 1:-1] = True
        v[interior] += d[interior]
    return np.ascontiguousarray(v.reshape(-1))
