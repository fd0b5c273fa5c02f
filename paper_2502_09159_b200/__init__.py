"""stmg_b200 — B200-native hot path of the hp space-time multigrid Stokes
solver of arXiv 2502.09159 (matrix-free space-time operator, additive Vanka
smoothers, hp transfers, V-cycle, GMRES, time marching; FP64, sm_100a).

This module is a thin ctypes binding of the C ABI in ``include/stmg_b200.h``
(``_build/libstmg_b200.so``). The names mirror the reference interfaces
(/root/reference/proj/include/stmg/st_operator.hpp, vanka.hpp, transfer.hpp,
solver.hpp). Device vectors are torch float64 CUDA tensors (plumbing only);
every computation runs in the library's CUDA kernels. There is no CPU
fallback: if the library is missing or the device is not a CUDA GPU, calls
raise.
"""
from __future__ import annotations

import ctypes
import os
from pathlib import Path
from typing import Optional, Sequence

_PKG = Path(__file__).resolve().parent
LIB_PATH = _PKG / "_build" / "libstmg_b200.so"
HEADER_PATH = _PKG.parent / "include" / "stmg_b200.h"

PROBLEM_MANUFACTURED = 0
PROBLEM_CAVITY = 1

ORTHO_MGS = 0   # modified Gram-Schmidt (the reference's, solver.cpp:146-152)
ORTHO_CGS2 = 1  # classical Gram-Schmidt twice: two batched all-reduces per iteration

SMOOTHER_NONE = -1
SMOOTHER_CELL = 0
SMOOTHER_VERTEX_STAR = 1

TRANSFER_KINDS = ["identity", "h_space", "p_space", "p_time", "h_space+p_time", "p_space+p_time"]


class StmgError(RuntimeError):
    """Raised for non-zero status codes (1 invalid argument, 2 runtime, 3 CUDA)."""

    def __init__(self, code: int, msg: str):
        super().__init__(f"stmg_b200 error {code}: {msg}")
        self.code = code


_lib: Optional[ctypes.CDLL] = None

_c_int, _c_double, _c_void_p = ctypes.c_int, ctypes.c_double, ctypes.c_void_p
_c_i64p = ctypes.POINTER(ctypes.c_int64)
_SIGNATURES = {
    "stmg_last_error": ([], ctypes.c_char_p),
    "stmg_version": ([], ctypes.c_char_p),
    "stmg_set_tuning": ([ctypes.c_char_p, ctypes.c_int64], _c_int),
    "stmg_ctx_create": ([_c_int, ctypes.POINTER(_c_void_p)], _c_int),
    "stmg_ctx_destroy": ([_c_void_p], _c_int),
    "stmg_ctx_set_stream": ([_c_void_p, _c_void_p], _c_int),
    "stmg_ctx_synchronize": ([_c_void_p], _c_int),
    "stmg_ctx_launch_count": ([_c_void_p], ctypes.c_int64),
    "stmg_level_create": ([_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_double, _c_double, _c_double, _c_int,
                           ctypes.POINTER(_c_void_p)], _c_int),
    "stmg_level_destroy": ([_c_void_p], _c_int),
    "stmg_level_sizes": ([_c_void_p, _c_i64p], _c_int),
    "stmg_apply_block": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int], _c_int),
    "stmg_vmult": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p], _c_int),
    "stmg_residual": ([_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p, _c_int], _c_int),
    "stmg_coupling_rhs": ([_c_void_p, _c_void_p, _c_void_p], _c_int),
    "stmg_step_health": ([_c_void_p, _c_void_p, _c_int, ctypes.POINTER(_c_double)], _c_int),
    "stmg_apply_additive": ([_c_void_p, _c_void_p, _c_void_p, _c_int], _c_int),
    "stmg_smooth_step": ([_c_void_p, _c_void_p, _c_void_p, _c_double, _c_int, _c_void_p, _c_int, _c_void_p], _c_int),
    "stmg_vanka_update": ([_c_void_p, _c_void_p, _c_void_p, _c_double, _c_int], _c_int),
    "stmg_vmult_host": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p], _c_int),
    "stmg_smooth_step_host": ([_c_void_p, _c_void_p, _c_void_p, _c_double, _c_int, _c_void_p, _c_int], _c_int),
    "stmg_vmult_host_async": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p], _c_int),
    "stmg_smooth_step_host_async": ([_c_void_p, _c_void_p, _c_void_p, _c_double, _c_int, _c_void_p, _c_int],
                                    _c_int),
    "stmg_solver_create": ([_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_double, _c_double, _c_double, _c_int,
                            _c_int, _c_int, _c_double, _c_int, _c_double, _c_double, _c_int,
                            ctypes.POINTER(_c_void_p)], _c_int),
    "stmg_solver_destroy": ([_c_void_p], _c_int),
    "stmg_solver_info": ([_c_void_p, _c_i64p], _c_int),
    "stmg_solver_level": ([_c_void_p, _c_int], _c_void_p),
    "stmg_restrict_residual": ([_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int], _c_int),
    "stmg_prolongate_correction": ([_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_int], _c_int),
    "stmg_coarse_solve": ([_c_void_p, _c_void_p, _c_void_p], _c_int),
    "stmg_vcycle": ([_c_void_p, _c_void_p, _c_void_p], _c_int),
    "stmg_gmres": ([_c_void_p, _c_void_p, _c_void_p, ctypes.POINTER(_c_int), ctypes.POINTER(_c_double), _c_int],
                   _c_int),
    "stmg_time_march": ([_c_void_p, _c_void_p, _c_void_p, ctypes.POINTER(_c_int)], _c_int),
    "stmg_time_march_ex": ([_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, ctypes.POINTER(_c_int)], _c_int),
    "stmg_time_march_problem": ([_c_void_p, _c_int, _c_void_p, ctypes.POINTER(_c_int)], _c_int),
    "stmg_time_march_host": ([_c_void_p, _c_void_p, _c_void_p, ctypes.POINTER(_c_int)], _c_int),
    "stmg_assemble_rhs": ([_c_void_p, _c_int, _c_double, _c_void_p, _c_int], _c_int),
    "stmg_interpolate_exact": ([_c_void_p, _c_int, _c_double, _c_void_p, _c_int], _c_int),
    "stmg_compute_errors": ([_c_void_p, _c_int, _c_double, _c_void_p, _c_int, ctypes.POINTER(_c_double)], _c_int),
    "stmg_solver_set_comm": ([_c_void_p, _c_void_p], _c_int),
    "stmg_solver_set_krylov": ([_c_void_p, _c_int], _c_int),
    "stmg3_solver_set_krylov": ([_c_void_p, _c_int], _c_int),
    "stmg_comm_nccl_unique_id": ([_c_void_p], _c_int),
    "stmg_comm_nccl_create": ([_c_void_p, _c_int, _c_int, _c_int, ctypes.POINTER(_c_void_p)], _c_int),
    "stmg_comm_nccl_ops": ([_c_void_p, _c_void_p], _c_int),
    "stmg_comm_destroy": ([_c_void_p], _c_int),
    "stmg_vcycle_all_at_once": ([_c_void_p, _c_void_p, _c_void_p, _c_int], _c_int),
    "stmg_solve_all_at_once": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p, ctypes.POINTER(_c_int),
                                ctypes.POINTER(_c_double), _c_int], _c_int),
    "stmg_plan_levels": ([_c_int, _c_int, _c_int, _c_int, _c_double, _c_int, _c_i64p], _c_int),
    "stmg_patch_info": ([_c_int, _c_int, _c_int, _c_int, _c_double, _c_double, _c_double, _c_int, _c_i64p,
                         ctypes.POINTER(_c_double), _c_int], _c_int),
    "stmg3_level_create": ([_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _c_double, _c_double,
                            _c_int, _c_void_p, ctypes.POINTER(_c_void_p)], _c_int),
    "stmg3_level_destroy": ([_c_void_p], _c_int),
    "stmg3_level_sizes": ([_c_void_p, _c_i64p], _c_int),
    "stmg3_level_patch_info": ([_c_void_p, ctypes.POINTER(_c_double)], _c_int),
    "stmg3_apply_block": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_int], _c_int),
    "stmg3_vmult": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p], _c_int),
    "stmg3_residual": ([_c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p, _c_int], _c_int),
    "stmg3_apply_additive": ([_c_void_p, _c_void_p, _c_void_p, _c_int], _c_int),
    "stmg3_smooth_step": ([_c_void_p, _c_void_p, _c_void_p, _c_double, _c_int, _c_void_p, _c_int, _c_void_p],
                          _c_int),
    "stmg3_vanka_update": ([_c_void_p, _c_void_p, _c_void_p, _c_double, _c_int], _c_int),
    "stmg3_project_mean_zero": ([_c_void_p, _c_void_p, _c_int], _c_int),
    "stmg3_solver_create": ([_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _c_double, _c_double,
                             _c_int, _c_int, _c_int, _c_int, _c_void_p, _c_int, _c_int, _c_double, _c_double, _c_double, _c_int,
                             ctypes.POINTER(_c_void_p)], _c_int),
    "stmg3_solver_destroy": ([_c_void_p], _c_int),
    "stmg3_plan_levels": ([_c_int] * 8 + [_c_i64p], _c_int),
    "stmg3_solver_info": ([_c_void_p, _c_i64p], _c_int),
    "stmg3_solver_level": ([_c_void_p, _c_int], _c_void_p),
    "stmg3_solver_set_comm": ([_c_void_p, _c_void_p], _c_int),
    "stmg3_restrict_residual": ([_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_int], _c_int),
    "stmg3_prolongate_correction": ([_c_void_p, _c_int, _c_void_p, _c_void_p, _c_int, _c_int, _c_int], _c_int),
    "stmg3_coarse_forward": ([_c_void_p, _c_void_p, _c_void_p, _c_int], _c_int),
    "stmg3_vcycle_all_at_once": ([_c_void_p, _c_void_p, _c_void_p, _c_int], _c_int),
    "stmg3_solve_all_at_once": ([_c_void_p, _c_void_p, _c_void_p, _c_int, _c_void_p, ctypes.POINTER(_c_int),
                                 ctypes.POINTER(_c_double), _c_int], _c_int),
    "stmg3_solver_create_split": ([_c_void_p, _c_int, _c_int, _c_int, _c_int, _c_int, _c_double, _c_double,
                                   _c_double, _c_int, _c_int, _c_int, _c_void_p, _c_int, _c_int, _c_int, _c_int,
                                   _c_double, _c_double, _c_double, _c_int, ctypes.POINTER(_c_void_p)], _c_int),
    "stmg3_solver_set_space_comm": ([_c_void_p, _c_void_p], _c_int),
    "stmg_comm_nccl_space_ops": ([_c_void_p, _c_void_p], _c_int),
}


def load_library(path: Optional[os.PathLike] = None) -> ctypes.CDLL:
    """Load (once) the in-tree CUDA library; raises if it was not built."""
    global _lib
    if _lib is not None and path is None:
        return _lib
    p = Path(path) if path else Path(os.environ.get("STMG_LIB", str(LIB_PATH)))
    if not p.exists():
        raise RuntimeError(f"stmg_b200: CUDA library {p} missing — run __graft_entry__.build() "
                           "(there is no CPU fallback)")
    lib = ctypes.CDLL(str(p))
    for name, (args, res) in _SIGNATURES.items():
        fn = getattr(lib, name)
        fn.argtypes = args
        fn.restype = res
    if path is None:
        _lib = lib
    return lib


def _check(code: int) -> None:
    if code != 0:
        raise StmgError(code, load_library().stmg_last_error().decode())


def _ptr(t, numel: Optional[int] = None, device: Optional[int] = None, name: str = "tensor") -> Optional[int]:
    """Device pointer of a contiguous float64 CUDA tensor (None passes NULL).

    ``numel``: minimum element count the C ABI will touch; ``device``: the
    context's CUDA device. A shorter, mistyped or foreign-device tensor raises
    instead of letting the kernels read or write past it."""
    if t is None:
        return None
    import torch

    if not t.is_cuda or t.dtype != torch.float64 or not t.is_contiguous():
        raise ValueError(f"stmg_b200: {name} must be a contiguous float64 CUDA tensor")
    if device is not None and t.device.index != device:
        raise ValueError(f"stmg_b200: {name} lives on cuda:{t.device.index}, the context on cuda:{device}")
    if numel is not None and t.numel() < numel:
        raise ValueError(f"stmg_b200: {name} has {t.numel()} elements, the call needs {numel}")
    return t.data_ptr()


def _hptr(a, numel: Optional[int] = None, name: str = "array") -> Optional[int]:
    """Host pointer of a C-contiguous float64 numpy array (None passes NULL)."""
    if a is None:
        return None
    import numpy as np

    if a.dtype != np.float64 or not a.flags["C_CONTIGUOUS"]:
        raise ValueError(f"stmg_b200: {name} must be a C-contiguous float64 host array")
    if numel is not None and a.size < numel:
        raise ValueError(f"stmg_b200: {name} has {a.size} elements, the call needs {numel}")
    return a.ctypes.data


_HALO_FN = ctypes.CFUNCTYPE(_c_int, _c_void_p, _c_void_p, _c_void_p, ctypes.c_int64, _c_void_p)
_REDUCE_FN = ctypes.CFUNCTYPE(_c_int, _c_void_p, _c_void_p, ctypes.c_int64, _c_void_p)


class _CommOps(ctypes.Structure):
    """struct stmg_comm_ops (include/stmg_b200.h)."""
    _fields_ = [("user", _c_void_p), ("rank", _c_int), ("world", _c_int), ("exchange_halo", _HALO_FN),
                ("allreduce_sum", _REDUCE_FN), ("allgather", _HALO_FN)]


_PLANES_FN = ctypes.CFUNCTYPE(_c_int, _c_void_p, _c_void_p, _c_void_p, _c_void_p, _c_void_p, ctypes.c_int64,
                              _c_void_p)


class _SpaceOps(ctypes.Structure):
    """struct stmg_comm_space_ops (include/stmg_b200.h): the z parts of the C5 hybrid split."""
    _fields_ = [("user", _c_void_p), ("part", _c_int), ("parts", _c_int), ("exchange_planes", _PLANES_FN),
                ("allreduce_sum", _REDUCE_FN), ("allgather", _HALO_FN)]


def _guard(fn):
    """Callbacks must not raise into C: map exceptions to a non-zero status."""
    def wrapped(*args):
        try:
            fn(*args)
            return 0
        except BaseException as exc:  # noqa: BLE001 - reported through the status code
            import traceback

            traceback.print_exception(exc)
            return 1
    return wrapped


class NcclComm:
    """The library's own NCCL time-slab communicator (stmg_comm_nccl_*): halo
    send/recv, Krylov all-reduces and the coarse all-gather run as NCCL calls
    inside libstmg_b200, with no Python in the per-iteration path. Rank 0
    makes the unique id (``NcclComm.unique_id()``); every rank passes the same
    bytes."""

    def __init__(self, rank: int, world: int, device: int, unique_id: bytes):
        if len(unique_id) != 128:
            raise ValueError("NcclComm: the NCCL unique id is 128 bytes")
        lib = load_library()
        h = _c_void_p()
        buf = ctypes.create_string_buffer(bytes(unique_id), 128)
        _check(lib.stmg_comm_nccl_create(ctypes.cast(buf, _c_void_p), rank, world, device, ctypes.byref(h)))
        self._h, self.rank, self.world, self.device = h, rank, world, device

    @staticmethod
    def unique_id() -> bytes:
        buf = ctypes.create_string_buffer(128)
        _check(load_library().stmg_comm_nccl_unique_id(ctypes.cast(buf, _c_void_p)))
        return buf.raw

    def ops(self) -> "_CommOps":
        ops = _CommOps()
        _check(load_library().stmg_comm_nccl_ops(self._h, ctypes.byref(ops)))
        return ops

    def space_ops(self) -> "_SpaceOps":
        """The same communicator as the z parts of a hybrid split (rank = part)."""
        ops = _SpaceOps()
        _check(load_library().stmg_comm_nccl_space_ops(self._h, ctypes.byref(ops)))
        return ops

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stmg_comm_destroy(self._h)
            self._h = None


class Context:
    """CUDA device + stream the library launches on (torch's current stream by default)."""

    def __init__(self, device: int = 0, stream=None):
        import torch

        lib = load_library()
        h = _c_void_p()
        _check(lib.stmg_ctx_create(device, ctypes.byref(h)))
        self._h = h
        self.device = device
        s = stream if stream is not None else torch.cuda.current_stream(device)
        _check(lib.stmg_ctx_set_stream(h, _c_void_p(s.cuda_stream)))

    @property
    def handle(self):
        return self._h

    def synchronize(self) -> None:
        _check(load_library().stmg_ctx_synchronize(self._h))

    def launch_count(self) -> int:
        return int(load_library().stmg_ctx_launch_count(self._h))

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stmg_ctx_destroy(self._h)
            self._h = None


class Level:
    """SpaceTimeBlockOperator + VankaSmoother of one Cartesian level
    (st_operator.hpp:94-165, vanka.hpp:45-89)."""

    def __init__(self, ctx: Context, nx: int, ny: int, r: int, k: int, tau: float, nu: float,
                 gamma: float = 0.0, smoother: int = SMOOTHER_CELL, _borrowed=None):
        self.ctx = ctx
        lib = load_library()
        if _borrowed is not None:
            self._h = _borrowed
            self._owned = False
        else:
            h = _c_void_p()
            _check(lib.stmg_level_create(ctx.handle, nx, ny, r, k, tau, nu, gamma, smoother, ctypes.byref(h)))
            self._h = h
            self._owned = True
        out = (ctypes.c_int64 * 10)()
        _check(lib.stmg_level_sizes(self._h, out))
        (self.n_slots, self.n_velocity, self.n_pressure, self.size, self.n_scalar, self.grid_x,
         self.n_patch_classes, self.total_matrix_elements) = [int(v) for v in out[:8]]
        self.factored = bool(out[8])           # time-diagonalised Vanka inverses in use
        self.factored_matrix_elements = int(out[9])

    # -- argument checks: every vector the C ABI touches is sized here
    def _v(self, t, n: int, name: str):
        return _ptr(t, n * self.size, self.ctx.device, name)

    def _halo(self, t, name: str = "x_prev_slot"):
        return _ptr(t, self.n_velocity, self.ctx.device, name)

    def _hv(self, a, n: int, name: str):
        return _hptr(a, n * self.size, name)

    # -- operator
    def apply_block(self, x, y, n_intervals: int = 1, raw: bool = False):
        _check(load_library().stmg_apply_block(self._h, self._v(x, n_intervals, "x"), self._v(y, n_intervals, "y"),
                                               n_intervals, int(raw)))
        return y

    def apply_block_raw(self, x, y, n_intervals: int = 1):
        return self.apply_block(x, y, n_intervals, raw=True)

    def vmult(self, x, y, n_intervals: int = 1, x_prev_slot=None):
        _check(load_library().stmg_vmult(self._h, self._v(x, n_intervals, "x"), self._v(y, n_intervals, "y"),
                                         n_intervals, self._halo(x_prev_slot)))
        return y

    def residual(self, b, x, r, n_intervals: int = 1, x_prev_slot=None, coupled: bool = True):
        _check(load_library().stmg_residual(self._h, self._v(b, n_intervals, "b"), self._v(x, n_intervals, "x"),
                                            self._v(r, n_intervals, "r"), n_intervals, self._halo(x_prev_slot),
                                            int(coupled)))
        return r

    def step_health(self, X, n_intervals: int = 1):
        """Saddle-point health per interval (solver.cpp:286-299): [(max_divergence, max_pressure_mean), ...]."""
        out = (ctypes.c_double * (2 * n_intervals))()
        _check(load_library().stmg_step_health(self._h, self._v(X, n_intervals, "X"), n_intervals, out))
        return [(out[2 * i], out[2 * i + 1]) for i in range(n_intervals)]

    def coupling_rhs(self, v_prev, out):
        _check(load_library().stmg_coupling_rhs(self._h, self._halo(v_prev, "v_prev"), self._v(out, 1, "out")))
        return out

    # -- smoother
    def apply_additive(self, residual, out, n_intervals: int = 1):
        _check(load_library().stmg_apply_additive(self._h, self._v(residual, n_intervals, "residual"),
                                                  self._v(out, n_intervals, "out"), n_intervals))
        return out

    def smooth_step(self, b, u, omega: float, n_intervals: int = 1, x_prev_slot=None, coupled: bool = False,
                    work=None):
        _check(load_library().stmg_smooth_step(self._h, self._v(b, n_intervals, "b"), self._v(u, n_intervals, "u"),
                                               omega, n_intervals, self._halo(x_prev_slot), int(coupled),
                                               self._v(work, n_intervals, "work")))
        return u

    def vanka_update(self, residual, u, omega: float, n_intervals: int = 1):
        _check(load_library().stmg_vanka_update(self._h, self._v(residual, n_intervals, "residual"),
                                                self._v(u, n_intervals, "u"), omega, n_intervals))
        return u

    # -- host-buffer (end-to-end) variants
    def assemble_rhs(self, F, t_start: float = 0.0, n_intervals: int = 1, problem: int = PROBLEM_MANUFACTURED):
        """SpaceTimeBlockOperator::assemble_rhs of a built-in force for n_intervals intervals from t_start."""
        _check(load_library().stmg_assemble_rhs(self._h, problem, t_start, self._v(F, n_intervals, "F"), n_intervals))
        return F

    def interpolate_exact(self, X, t_start: float = 0.0, n_intervals: int = 1, problem: int = PROBLEM_MANUFACTURED):
        """interpolate_exact (harness.cpp:185-239) of the built-in exact solution into X."""
        _check(load_library().stmg_interpolate_exact(self._h, problem, t_start, self._v(X, n_intervals, "X"),
                                                     n_intervals))
        return X

    def compute_errors(self, X, t_start: float = 0.0, n_intervals: int = 1,
                       problem: int = PROBLEM_MANUFACTURED) -> dict:
        """compute_errors (harness.cpp:72-183) of a trajectory against the built-in exact solution."""
        out = (ctypes.c_double * 5)()
        _check(load_library().stmg_compute_errors(self._h, problem, t_start, self._v(X, n_intervals, "X"),
                                                  n_intervals, out))
        return dict(e_v_l2=out[0], e_p_l2=out[1], e_v_h1=out[2], e_div=out[3], e_v_linf=out[4])

    def vmult_host(self, x, y, n_intervals: int = 1, x_prev_slot=None, blocking: bool = True):
        """Host (numpy) buffers; blocking=False enqueues only (stmg_vmult_host_async): keep the
        buffers alive and call ctx.synchronize() before reading y."""
        fn = load_library().stmg_vmult_host if blocking else load_library().stmg_vmult_host_async
        _check(fn(self._h, self._hv(x, n_intervals, "x"), self._hv(y, n_intervals, "y"), n_intervals,
                  _hptr(x_prev_slot, self.n_velocity, "x_prev_slot")))
        return y

    def smooth_step_host(self, b, u, omega: float, n_intervals: int = 1, x_prev_slot=None, coupled: bool = False,
                         blocking: bool = True):
        fn = load_library().stmg_smooth_step_host if blocking else load_library().stmg_smooth_step_host_async
        _check(fn(self._h, self._hv(b, n_intervals, "b"), self._hv(u, n_intervals, "u"), omega, n_intervals,
                  _hptr(x_prev_slot, self.n_velocity, "x_prev_slot"), int(coupled)))
        return u

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None) and _lib is not None:
            _lib.stmg_level_destroy(self._h)
            self._h = None


class Solver:
    """build_setup + VCycle + gmres + time_march (harness.cpp:26-70, solver.cpp:56-325)."""

    def __init__(self, ctx: Context, refinements: int, r: int, k: int = -1, n_steps: int = 0, t_end: float = 1.0,
                 nu: float = 0.1, gamma: float = 1.0, smoother: int = SMOOTHER_CELL, nu1: int = 1, nu2: int = 1,
                 omega: float = 0.8, h_only: bool = False, rtol: float = 1e-8, atol: float = 1e-14,
                 max_iterations: int = 200):
        self.ctx = ctx
        lib = load_library()
        h = _c_void_p()
        _check(lib.stmg_solver_create(ctx.handle, refinements, r, k, n_steps, t_end, nu, gamma, smoother, nu1, nu2,
                                      omega, int(h_only), rtol, atol, max_iterations, ctypes.byref(h)))
        self._h = h
        out = (ctypes.c_int64 * (2 + 5 * 64))()
        _check(lib.stmg_solver_info(h, out))
        self.n_levels, self.n_steps = int(out[0]), int(out[1])
        self.level_info = [dict(nx=int(out[2 + 5 * l]), r=int(out[3 + 5 * l]), k=int(out[4 + 5 * l]),
                                kind=TRANSFER_KINDS[int(out[5 + 5 * l])], size=int(out[6 + 5 * l]))
                           for l in range(self.n_levels)]
        self.levels = [Level(ctx, 0, 0, 0, 0, 0, 0, _borrowed=lib.stmg_solver_level(h, l))
                       for l in range(self.n_levels)]
        self.finest = self.levels[-1]

    def restrict_residual(self, l: int, fine, coarse, project_pressure: bool = True):
        _check(load_library().stmg_restrict_residual(self._h, l, self.levels[l]._v(fine, 1, "fine"),
                                                     self.levels[l - 1]._v(coarse, 1, "coarse"), int(project_pressure)))
        return coarse

    def prolongate_correction(self, l: int, coarse, fine, project_pressure: bool = True, accumulate: bool = False):
        _check(load_library().stmg_prolongate_correction(self._h, l, self.levels[l - 1]._v(coarse, 1, "coarse"),
                                                         self.levels[l]._v(fine, 1, "fine"), int(project_pressure),
                                                         int(accumulate)))
        return fine

    def coarse_solve(self, b, x):
        c = self.levels[0]
        _check(load_library().stmg_coarse_solve(self._h, c._v(b, 1, "b"), c._v(x, 1, "x")))
        return x

    def vcycle(self, b, x):
        _check(load_library().stmg_vcycle(self._h, self.finest._v(b, 1, "b"), self.finest._v(x, 1, "x")))
        return x

    def gmres(self, b, x, history_cap: int = 256):
        it = _c_int(0)
        hist = (ctypes.c_double * history_cap)()
        code = load_library().stmg_gmres(self._h, self.finest._v(b, 1, "b"), self.finest._v(x, 1, "x"),
                                         ctypes.byref(it), hist, history_cap)
        _check(code)
        return int(it.value), [hist[i] for i in range(min(history_cap, it.value + 1))]

    def time_march(self, F, X):
        iters = (ctypes.c_int * self.n_steps)()
        f = self.finest
        _check(load_library().stmg_time_march(self._h, f._v(F, self.n_steps, "F"), f._v(X, self.n_steps, "X"), iters))
        return [int(v) for v in iters]

    def time_march_problem(self, problem: int, X):
        """time_march of a built-in problem (PROBLEM_MANUFACTURED: force; PROBLEM_CAVITY: lifted lid data)."""
        iters = (ctypes.c_int * self.n_steps)()
        _check(load_library().stmg_time_march_problem(self._h, problem, self.finest._v(X, self.n_steps, "X"), iters))
        return [int(v) for v in iters]

    def time_march_ex(self, X, F=None, lifts=None, v_init=None):
        """time_march with load vectors, per-step Dirichlet lift vectors and an initial velocity (all optional)."""
        iters = (ctypes.c_int * self.n_steps)()
        f, n = self.finest, self.n_steps
        _check(load_library().stmg_time_march_ex(self._h, f._v(F, n, "F"), f._v(lifts, n, "lifts"),
                                                 f._halo(v_init, "v_init"), f._v(X, n, "X"), iters))
        return [int(v) for v in iters]

    def time_march_host(self, F, X):
        iters = (ctypes.c_int * self.n_steps)()
        f, n = self.finest, self.n_steps
        _check(load_library().stmg_time_march_host(self._h, f._hv(F, n, "F"), f._hv(X, n, "X"), iters))
        return [int(v) for v in iters]

    def set_comm(self, comm) -> None:
        """Install a time-slab communicator (``timeslab.TorchComm`` /
        ``timeslab.LoopbackComm``: attributes ``rank``, ``world`` and methods
        ``exchange_halo(send, recv, n, stream)``, ``allreduce_sum(buf, n,
        stream)``, ``allgather(send, recv, n, stream)`` taking raw device
        pointers), or remove it with None."""
        lib = load_library()
        if comm is None:
            self._comm = None
            _check(lib.stmg_solver_set_comm(self._h, None))
            return
        if isinstance(comm, NcclComm):
            self._comm = comm  # keeps the communicator alive while installed
            _check(lib.stmg_solver_set_comm(self._h, ctypes.byref(comm.ops())))
            return
        ops = _CommOps(None, comm.rank, comm.world,
                       _HALO_FN(_guard(lambda u, s, r, n, st: comm.exchange_halo(s, r, n, st))),
                       _REDUCE_FN(_guard(lambda u, b, n, st: comm.allreduce_sum(b, n, st))),
                       _HALO_FN(_guard(lambda u, s, r, n, st: comm.allgather(s, r, n, st))))
        self._comm = ops  # the C side keeps the function pointers: keep them alive
        _check(lib.stmg_solver_set_comm(self._h, ctypes.byref(ops)))

    def set_krylov(self, orthogonalization: int) -> None:
        """ORTHO_MGS (default, the reference's) or ORTHO_CGS2 (two batched all-reduces per iteration)."""
        _check(load_library().stmg_solver_set_krylov(self._h, orthogonalization))

    def vcycle_all_at_once(self, b, x, n_intervals: int):
        """One all-at-once V-cycle over n_intervals intervals (Eq. GloSys)."""
        f = self.finest
        _check(load_library().stmg_vcycle_all_at_once(self._h, f._v(b, n_intervals, "b"), f._v(x, n_intervals, "x"),
                                                      n_intervals))
        return x

    def solve_all_at_once(self, F, X, n_intervals: int, v_init=None, history_cap: int = 256):
        """FGMRES + all-at-once hp-STMG on a slab; returns (iterations, residual history)."""
        it = _c_int(0)
        hist = (ctypes.c_double * history_cap)()
        f = self.finest
        _check(load_library().stmg_solve_all_at_once(self._h, f._v(F, n_intervals, "F"), f._v(X, n_intervals, "X"),
                                                      n_intervals, f._halo(v_init, "v_init"), ctypes.byref(it), hist,
                                                      history_cap))
        return int(it.value), [hist[i] for i in range(min(history_cap, it.value + 1))]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stmg_solver_destroy(self._h)
            self._h = None


class Level3:
    """3D SpaceTimeBlockOperator + cell VankaSmoother (BASELINE C3 / C5): Q_{r+1}^3 / P_r^disc on the unit cube,
    optionally on a deformed (trilinear) mesh given by host vertex coordinates."""

    def __init__(self, ctx: Context, nx: int, ny: int, nz: int, r: int, k: int, tau: float, nu: float,
                 gamma: float = 0.0, smoother: int = SMOOTHER_CELL, vertices=None, _borrowed=None):
        self.ctx = ctx
        lib = load_library()
        if _borrowed is not None:
            self._h, self._owned = _borrowed, False
        else:
            h = _c_void_p()
            _check(lib.stmg3_level_create(ctx.handle, nx, ny, nz, r, k, tau, nu, gamma, smoother,
                                          _hptr(vertices, 3 * (nx + 1) * (ny + 1) * (nz + 1), "vertices"),
                                          ctypes.byref(h)))
            self._h, self._owned = h, True
        out = (ctypes.c_int64 * 12)()
        _check(lib.stmg3_level_sizes(self._h, out))
        (self.n_slots, self.n_velocity, self.n_pressure, self.size, self.n_scalar, self.gx, self.gy, self.gz,
         self.n_p, self.max_patch, self.n_patch_classes, self.total_matrix_elements) = [int(v) for v in out]

    def _v(self, t, n: int, name: str):
        return _ptr(t, n * self.size, self.ctx.device, name)

    def _halo(self, t, name: str = "x_prev_slot"):
        return _ptr(t, self.n_velocity, self.ctx.device, name)

    @property
    def patch_setup(self) -> dict:
        """Vanka patch setup: seconds, on_gpu (exact per-cell inverses built on the device),
        factored (time-diagonalised blocks), affine, classes."""
        out = (ctypes.c_double * 6)()
        _check(load_library().stmg3_level_patch_info(self._h, out))
        return dict(seconds=out[0], on_gpu=out[1] >= 1, factored=out[1] == 2, affine=bool(out[2]),
                    classes=int(out[3]), streamed_elements=int(out[4]), macs_per_column=int(out[5]))

    def apply_block(self, x, y, n_intervals: int = 1, raw: bool = False):
        _check(load_library().stmg3_apply_block(self._h, self._v(x, n_intervals, "x"), self._v(y, n_intervals, "y"),
                                                n_intervals, int(raw)))
        return y

    def vmult(self, x, y, n_intervals: int = 1, x_prev_slot=None):
        _check(load_library().stmg3_vmult(self._h, self._v(x, n_intervals, "x"), self._v(y, n_intervals, "y"),
                                          n_intervals, self._halo(x_prev_slot)))
        return y

    def residual(self, b, x, r, n_intervals: int = 1, x_prev_slot=None, coupled: bool = True):
        _check(load_library().stmg3_residual(self._h, self._v(b, n_intervals, "b"), self._v(x, n_intervals, "x"),
                                             self._v(r, n_intervals, "r"), n_intervals, self._halo(x_prev_slot),
                                             int(coupled)))
        return r

    def apply_additive(self, residual, out, n_intervals: int = 1):
        _check(load_library().stmg3_apply_additive(self._h, self._v(residual, n_intervals, "residual"),
                                                   self._v(out, n_intervals, "out"), n_intervals))
        return out

    def smooth_step(self, b, u, omega: float, n_intervals: int = 1, x_prev_slot=None, coupled: bool = False,
                    work=None):
        _check(load_library().stmg3_smooth_step(self._h, self._v(b, n_intervals, "b"), self._v(u, n_intervals, "u"),
                                                omega, n_intervals, self._halo(x_prev_slot), int(coupled),
                                                self._v(work, n_intervals, "work")))
        return u

    def vanka_update(self, residual, u, omega: float, n_intervals: int = 1):
        _check(load_library().stmg3_vanka_update(self._h, self._v(residual, n_intervals, "residual"),
                                                 self._v(u, n_intervals, "u"), omega, n_intervals))
        return u

    def project_mean_zero(self, x, n_intervals: int = 1):
        _check(load_library().stmg3_project_mean_zero(self._h, self._v(x, n_intervals, "x"), n_intervals))
        return x

    def __del__(self):
        if getattr(self, "_owned", False) and getattr(self, "_h", None) and _lib is not None:
            _lib.stmg3_level_destroy(self._h)
            self._h = None


class Solver3:
    """3D all-at-once hp-STMG: p-coarsening in k and r, then h-coarsening in space (and time); FGMRES."""

    def __init__(self, ctx: Context, nx: int, ny: int, nz: int, r: int, k: int, tau: float, nu: float = 1.0,
                 gamma: float = 1.0, n_hcoarse: int = 1, time_coarsen: bool = True, k_min: int = 0, vertices=None,
                 affine_patches: bool = False, nu1: int = 2,
                 nu2: int = 2, omega: float = 0.8, rtol: float = 1e-8, atol: float = 1e-14,
                 max_iterations: int = 200, z_parts: int = 1, z_part: int = 0):
        """z_parts > 1: this rank's part of the C5 hybrid split (stmg3_solver_create_split):
        `vertices` is the global vertex array, the levels hold the part's cells;
        install the parts' communicator with set_space_comm."""
        self.ctx = ctx
        lib = load_library()
        h = _c_void_p()
        vp = _hptr(vertices, 3 * (nx + 1) * (ny + 1) * (nz + 1), "vertices")
        if z_parts > 1:
            _check(lib.stmg3_solver_create_split(ctx.handle, nx, ny, nz, r, k, tau, nu, gamma, n_hcoarse,
                                                 int(time_coarsen), k_min, vp, z_parts, z_part, nu1, nu2, omega,
                                                 rtol, atol, max_iterations, ctypes.byref(h)))
        else:
            _check(lib.stmg3_solver_create(ctx.handle, nx, ny, nz, r, k, tau, nu, gamma, n_hcoarse,
                                           int(time_coarsen), k_min, int(affine_patches), vp, nu1, nu2, omega, rtol,
                                           atol, max_iterations, ctypes.byref(h)))
        self.z_parts, self.z_part = z_parts, z_part
        self._h = h
        out = (ctypes.c_int64 * (1 + 7 * 64))()
        _check(lib.stmg3_solver_info(h, out))
        self.n_levels = int(out[0])
        self.level_info = [dict(nx=int(out[1 + 7 * l]), ny=int(out[2 + 7 * l]), nz=int(out[3 + 7 * l]),
                                r=int(out[4 + 7 * l]), k=int(out[5 + 7 * l]), tshift=int(out[6 + 7 * l]),
                                size=int(out[7 + 7 * l])) for l in range(self.n_levels)]
        self.levels = [Level3(ctx, 0, 0, 0, 0, 0, 0, 0, _borrowed=lib.stmg3_solver_level(h, l))
                       for l in range(self.n_levels)]
        self.finest = self.levels[-1]

    def _n_fine(self, l: int, n_coarse: int) -> int:
        """Fine intervals of the pair (l, l-1): 2 n_coarse when it coarsens time."""
        return n_coarse << (self.level_info[l - 1]["tshift"] - self.level_info[l]["tshift"])

    def restrict_residual(self, l: int, fine, coarse, n_coarse: int = 1, project_pressure: bool = True):
        nf = self._n_fine(l, n_coarse)
        _check(load_library().stmg3_restrict_residual(self._h, l, self.levels[l]._v(fine, nf, "fine"),
                                                      self.levels[l - 1]._v(coarse, n_coarse, "coarse"), n_coarse,
                                                      int(project_pressure)))
        return coarse

    def prolongate_correction(self, l: int, coarse, fine, n_coarse: int = 1, project_pressure: bool = True,
                              accumulate: bool = False):
        nf = self._n_fine(l, n_coarse)
        _check(load_library().stmg3_prolongate_correction(self._h, l, self.levels[l - 1]._v(coarse, n_coarse, "coarse"),
                                                          self.levels[l]._v(fine, nf, "fine"), n_coarse,
                                                          int(project_pressure), int(accumulate)))
        return fine

    def coarse_forward(self, b, x, n_intervals: int):
        c = self.levels[0]
        _check(load_library().stmg3_coarse_forward(self._h, c._v(b, n_intervals, "b"), c._v(x, n_intervals, "x"),
                                                   n_intervals))
        return x

    def set_comm(self, comm) -> None:
        """Time-slab communicator, as Solver.set_comm."""
        lib = load_library()
        if comm is None:
            self._comm = None
            _check(lib.stmg3_solver_set_comm(self._h, None))
            return
        if isinstance(comm, NcclComm):
            self._comm = comm
            _check(lib.stmg3_solver_set_comm(self._h, ctypes.byref(comm.ops())))
            return
        ops = _CommOps(None, comm.rank, comm.world,
                       _HALO_FN(_guard(lambda u, s, r, n, st: comm.exchange_halo(s, r, n, st))),
                       _REDUCE_FN(_guard(lambda u, b, n, st: comm.allreduce_sum(b, n, st))),
                       _HALO_FN(_guard(lambda u, s, r, n, st: comm.allgather(s, r, n, st))))
        self._comm = ops
        _check(lib.stmg3_solver_set_comm(self._h, ctypes.byref(ops)))

    def set_space_comm(self, comm) -> None:
        """The z parts' communicator of a split solver: an NcclComm over the
        parts, or an object with part, parts, exchange_planes(send_lo, recv_lo,
        send_hi, recv_hi, n, stream), allreduce_sum(buf, n, stream) and
        allgather(send, recv, n, stream) (timeslab.LoopbackSpaceComm,
        timeslab.TorchSpaceComm)."""
        lib = load_library()
        if comm is None:
            self._space = None
            _check(lib.stmg3_solver_set_space_comm(self._h, None))
            return
        if isinstance(comm, NcclComm):
            self._space = (comm, comm.space_ops())
            _check(lib.stmg3_solver_set_space_comm(self._h, ctypes.byref(self._space[1])))
            return
        ops = _SpaceOps(None, comm.part, comm.parts,
                        _PLANES_FN(_guard(lambda u, sl, rl, sh, rh, n, st: comm.exchange_planes(sl, rl, sh, rh, n,
                                                                                               st))),
                        _REDUCE_FN(_guard(lambda u, b, n, st: comm.allreduce_sum(b, n, st))),
                        _HALO_FN(_guard(lambda u, s, r, n, st: comm.allgather(s, r, n, st))))
        self._space = ops
        _check(lib.stmg3_solver_set_space_comm(self._h, ctypes.byref(ops)))

    def set_krylov(self, orthogonalization: int) -> None:
        """As Solver.set_krylov."""
        _check(load_library().stmg3_solver_set_krylov(self._h, orthogonalization))

    def vcycle_all_at_once(self, b, x, n_intervals: int):
        f = self.finest
        _check(load_library().stmg3_vcycle_all_at_once(self._h, f._v(b, n_intervals, "b"), f._v(x, n_intervals, "x"),
                                                       n_intervals))
        return x

    def solve_all_at_once(self, F, X, n_intervals: int, v_init=None, history_cap: int = 256):
        it = _c_int(0)
        hist = (ctypes.c_double * history_cap)()
        f = self.finest
        _check(load_library().stmg3_solve_all_at_once(self._h, f._v(F, n_intervals, "F"), f._v(X, n_intervals, "X"),
                                                       n_intervals, f._halo(v_init, "v_init"), ctypes.byref(it), hist,
                                                       history_cap))
        return int(it.value), [hist[i] for i in range(min(history_cap, it.value + 1))]

    def __del__(self):
        if getattr(self, "_h", None) and _lib is not None:
            _lib.stmg3_solver_destroy(self._h)
            self._h = None


def plan_levels(refinements: int, r: int, k: int = -1, n_steps: int = 0, t_end: float = 1.0,
                h_only: bool = False) -> dict:
    """Host-only hierarchy plan (plan_hierarchy + combine_hierarchies)."""
    out = (ctypes.c_int64 * (2 + 5 * 64))()
    _check(load_library().stmg_plan_levels(refinements, r, k, n_steps, t_end, int(h_only), out))
    n = int(out[0])
    return dict(n_steps=int(out[1]),
                levels=[dict(nx=int(out[2 + 5 * l]), r=int(out[3 + 5 * l]), k=int(out[4 + 5 * l]),
                             kind=TRANSFER_KINDS[int(out[5 + 5 * l])], size=int(out[6 + 5 * l]))
                        for l in range(n)])


def plan_levels3(nx: int, ny: int, nz: int, r: int, k: int, n_hcoarse: int = 1, time_coarsen: bool = True,
                 k_min: int = 0) -> list:
    """Host-only 3D hierarchy plan (coarse first): dicts nx, ny, nz, r, k, tshift, size."""
    out = (ctypes.c_int64 * (1 + 7 * 64))()
    _check(load_library().stmg3_plan_levels(nx, ny, nz, r, k, n_hcoarse, int(time_coarsen), k_min, out))
    return [dict(nx=int(out[1 + 7 * l]), ny=int(out[2 + 7 * l]), nz=int(out[3 + 7 * l]), r=int(out[4 + 7 * l]),
                 k=int(out[5 + 7 * l]), tshift=int(out[6 + 7 * l]), size=int(out[7 + 7 * l]))
            for l in range(int(out[0]))]


def patch_info(nx: int, ny: int, r: int, k: int, tau: float, nu: float, gamma: float, smoother: int):
    """Host-only Vanka patch statistics: dict(n_patches, n_classes, sum_nt2, n_t per class, inverses...)."""
    out = (ctypes.c_int64 * 64)()
    _check(load_library().stmg_patch_info(nx, ny, r, k, tau, nu, gamma, smoother, out, None, 0))
    n_classes = int(out[1])
    return dict(n_patches=int(out[0]), n_classes=n_classes, sum_nt2=int(out[2]), n_colours=int(out[3]),
                class_sizes=[int(out[4 + i]) for i in range(min(n_classes, 56))], factored=bool(out[60]),
                n_sp=int(out[61]), factored_macs=int(out[62]))


def exported_symbols() -> Sequence[str]:
    """Function names declared in include/stmg_b200.h."""
    import re

    text = HEADER_PATH.read_text()
    return sorted(set(re.findall(r"\b(stmg3?_[a-z_0-9]+)\s*\(", text)))


__all__ = ["NcclComm", "ORTHO_MGS", "ORTHO_CGS2", "Context", "Level", "Solver", "Level3", "Solver3", "StmgError", "load_library", "plan_levels", "patch_info",
           "exported_symbols", "SMOOTHER_CELL", "SMOOTHER_VERTEX_STAR", "SMOOTHER_NONE", "PROBLEM_MANUFACTURED",
           "PROBLEM_CAVITY"]
