"""Time-slab partition of the all-at-once space-time system across ranks.

The all-at-once matrix of Eq. GloSys is lower block
bidiagonal in time: interval n couples only to interval n-1, through the
velocity of its last temporal slot (the DG upwind jump, coupling_rhs,
st_operator.cpp:409-421). Rank p owns the contiguous intervals
[p*N_local, (p+1)*N_local). Every operator application (vmult, smoother
residual) needs exactly one halo: the slot-k velocity of rank p-1's last
interval (M^v doubles), sent point-to-point with NCCL (GPU) or gloo (CPU
tests). Everything else -- the Vanka patch solves, the spatial transfers --
is interval-local.
"""
from __future__ import annotations

from typing import Optional


def owned_intervals(n_global: int, rank: int, world: int) -> range:
    """Contiguous block of intervals owned by `rank` (remainder to the first ranks)."""
    base, rem = divmod(n_global, world)
    start = rank * base + min(rank, rem)
    return range(start, start + base + (1 if rank < rem else 0))


def last_slot_velocity(x, n_local: int, interval_size: int, n_velocity: int, n_slots: int):
    """View of the slot-k velocity block of the last local interval."""
    start = (n_local - 1) * interval_size + (n_slots - 1) * n_velocity
    return x[start:start + n_velocity]


def exchange_halo(x, halo, n_local: int, interval_size: int, n_velocity: int, n_slots: int,
                  rank: int, world: int, group=None) -> Optional[object]:
    """Send my last interval's slot-k velocity to rank+1, receive rank-1's
    into `halo`. Returns `halo` on ranks > 0 and None on rank 0 (its first
    interval is coupled to the initial value, zero here)."""
    import torch.distributed as dist

    if world == 1:
        return None
    ops = []
    if rank + 1 < world:
        send = last_slot_velocity(x, n_local, interval_size, n_velocity, n_slots).contiguous()
        ops.append(dist.P2POp(dist.isend, send, rank + 1, group=group))
    if rank > 0:
        ops.append(dist.P2POp(dist.irecv, halo, rank - 1, group=group))
    for w in dist.batch_isend_irecv(ops):
        w.wait()
    return halo if rank > 0 else None


# ---------------------------------------------------------------- communicators
# Implementations of the library's stmg_comm_ops (include/stmg_b200.h) for the
# all-at-once solve: Solver.set_comm(comm). The library passes raw pointers
# and its stream; every exchange is stream-ordered on that stream.

def _view(ptr: int, n: int, device):
    """Zero-copy float64 tensor over a raw pointer (device or host memory)."""
    import ctypes

    import torch

    if n == 0:
        return torch.empty(0, dtype=torch.float64, device=device)
    if torch.device(device).type == "cuda":
        class _Iface:
            __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                        "version": 3, "strides": None}
        return torch.as_tensor(_Iface(), device=device)
    return torch.frombuffer((ctypes.c_double * int(n)).from_address(int(ptr)), dtype=torch.float64)


def _on_stream(stream, device):
    import contextlib

    import torch

    if stream and torch.device(device).type == "cuda":
        return torch.cuda.stream(torch.cuda.ExternalStream(int(stream), device=device))
    return contextlib.nullcontext()


class TorchComm:
    """Time-slab communicator over torch.distributed (NCCL over NVLink on
    the GPU box; gloo for CPU tests): point-to-point halo, all-reduce of the
    Krylov dots, all-gather of the coarse right-hand sides."""

    def __init__(self, device="cuda", group=None):
        import torch.distributed as dist

        self.group = group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device

    def exchange_halo(self, send, recv, n, stream=None):
        import torch.distributed as dist

        with _on_stream(stream, self.device):
            ops = []
            peer = (lambda r: r) if self.group is None else (lambda r: dist.get_global_rank(self.group, r))
            if self.rank + 1 < self.world:
                ops.append(dist.P2POp(dist.isend, _view(send, n, self.device), peer(self.rank + 1), group=self.group))
            if self.rank > 0:
                ops.append(dist.P2POp(dist.irecv, _view(recv, n, self.device), peer(self.rank - 1), group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()

    def allreduce_sum(self, buf, n, stream=None):
        import torch.distributed as dist

        with _on_stream(stream, self.device):
            dist.all_reduce(_view(buf, n, self.device), group=self.group)

    def allgather(self, send, recv, n, stream=None):
        import torch.distributed as dist

        with _on_stream(stream, self.device):
            out = _view(recv, n * self.world, self.device)
            src = _view(send, n, self.device)
            if hasattr(dist, "all_gather_into_tensor") and out.is_cuda:
                dist.all_gather_into_tensor(out, src, group=self.group)
            else:
                dist.all_gather(list(out.split(n)), src, group=self.group)


class LoopbackHub:
    """Shared state of `world` in-process ranks (one thread each). Every
    exchange is host-synchronised: a rank finishes its stream, hands over a
    copy, and the receiver copies it in. No kernel ever waits on another
    rank's kernel, so several ranks can share one GPU safely. This is how the
    partitioned solve is tested on a single B200."""

    def __init__(self, world: int, timeout: float = 120.0):
        import queue
        import threading

        self.world = world
        self.timeout = timeout
        self.barrier = threading.Barrier(world)
        self.lock = threading.Lock()
        self.slots = {}
        self.mail = [queue.Queue() for _ in range(world)]

    def gather(self, rank, t):
        with self.lock:
            self.slots[rank] = t
        self.barrier.wait(self.timeout)
        parts = [self.slots[r] for r in range(self.world)]
        self.barrier.wait(self.timeout)  # all read before the next round writes
        return parts


class LoopbackComm:
    def __init__(self, hub: LoopbackHub, rank: int, device="cuda"):
        self.hub, self.rank, self.world, self.device = hub, rank, hub.world, device

    def _sync(self, stream):
        import torch

        if torch.device(self.device).type == "cuda":
            if stream:
                torch.cuda.ExternalStream(int(stream), device=self.device).synchronize()
            else:
                torch.cuda.synchronize(self.device)

    def _snapshot(self, ptr, n, stream):
        with _on_stream(stream, self.device):
            t = _view(ptr, n, self.device).clone()
        self._sync(stream)
        return t

    def exchange_halo(self, send, recv, n, stream=None):
        self._sync(stream)
        if self.rank + 1 < self.world:
            self.hub.mail[self.rank + 1].put(self._snapshot(send, n, stream))
        if self.rank > 0:
            data = self.hub.mail[self.rank].get(timeout=self.hub.timeout)
            with _on_stream(stream, self.device):
                _view(recv, n, self.device).copy_(data)
            self._sync(stream)

    def allreduce_sum(self, buf, n, stream=None):
        self._sync(stream)
        parts = self.hub.gather(self.rank, self._snapshot(buf, n, stream))
        with _on_stream(stream, self.device):
            total = parts[0].clone()
            for p in parts[1:]:  # fixed rank order: identical sums on every rank
                total += p
            _view(buf, n, self.device).copy_(total)
        self._sync(stream)

    def allgather(self, send, recv, n, stream=None):
        self._sync(stream)
        parts = self.hub.gather(self.rank, self._snapshot(send, n, stream))
        with _on_stream(stream, self.device):
            out = _view(recv, n * self.world, self.device)
            for r, p in enumerate(parts):
                out[r * n:(r + 1) * n].copy_(p)
        self._sync(stream)


# ---------------------------------------------------------------- z parts
# The C5 hybrid split (stmg3_solver_create_split, stmg_comm_space_ops): the
# part's neighbours exchange their shared interface planes; pressure means
# and Krylov sums are reduced over the parts; the coarse level is gathered.

def z_part_dofs(nx: int, ny: int, nz: int, r: int, k: int, parts: int, part: int):
    """Whole-mesh index (within one interval) of every dof of z part `part`,
    in the part's own BlockVector order (3D layout of include/stmg_b200.h):
    velocity (slot, component, node (Z, Y, X)), then pressure (slot, cell, mode)."""
    import numpy as np

    if nz % parts:
        raise ValueError("nz must be divisible by the number of z parts")
    p, S = r + 1, k + 1
    npm = (r + 1) * (r + 2) * (r + 3) // 6
    gx, gy, gz = nx * p + 1, ny * p + 1, nz * p + 1
    nsc = gx * gy * gz
    mv, mp = 3 * nsc, nx * ny * nz * npm
    nzl = nz // parts
    gzl = nzl * p + 1
    plane = gx * gy
    nodes = (np.arange(gzl)[:, None] + part * nzl * p) * plane + np.arange(plane)[None, :]
    vel = (np.arange(S)[:, None, None] * mv + np.arange(3)[None, :, None] * nsc + nodes.reshape(1, 1, -1)).ravel()
    cells = np.arange(nx * ny * nzl) + part * nzl * nx * ny
    pre = (S * mv + np.arange(S)[:, None, None] * mp + cells[None, :, None] * npm
           + np.arange(npm)[None, None, :]).ravel()
    return np.concatenate([vel, pre]).astype(np.int64)


class LoopbackSpaceHub:
    """Shared state of the `parts` in-process z parts of one time slab
    (host-synchronised, as LoopbackHub)."""

    def __init__(self, parts: int, timeout: float = 120.0):
        import queue

        self.hub = LoopbackHub(parts, timeout)
        self.parts = parts
        # from_below[p]: planes sent up by part p-1; from_above[p]: sent down by p+1
        self.from_below = [queue.Queue() for _ in range(parts)]
        self.from_above = [queue.Queue() for _ in range(parts)]


class LoopbackSpaceComm:
    """stmg_comm_space_ops for in-process z parts (threads) on one GPU."""

    def __init__(self, hub: LoopbackSpaceHub, part: int, device="cuda"):
        self.hub, self.part, self.parts, self.device = hub, part, hub.parts, device
        self._inner = LoopbackComm(hub.hub, part, device)

    def exchange_planes(self, send_lo, recv_lo, send_hi, recv_hi, n, stream=None):
        c = self._inner
        c._sync(stream)
        if send_lo and self.part > 0:
            self.hub.from_above[self.part - 1].put(c._snapshot(send_lo, n, stream))
        if send_hi and self.part + 1 < self.parts:
            self.hub.from_below[self.part + 1].put(c._snapshot(send_hi, n, stream))
        for ptr, q in ((recv_lo, self.hub.from_below[self.part]), (recv_hi, self.hub.from_above[self.part])):
            if ptr:
                data = q.get(timeout=self.hub.hub.timeout)
                with _on_stream(stream, self.device):
                    _view(ptr, n, self.device).copy_(data)
        c._sync(stream)

    def allreduce_sum(self, buf, n, stream=None):
        self._inner.allreduce_sum(buf, n, stream)

    def allgather(self, send, recv, n, stream=None):
        self._inner.allgather(send, recv, n, stream)


class TorchSpaceComm:
    """stmg_comm_space_ops over a torch.distributed group of the z parts
    (group rank = part): interface planes by send/recv with the neighbours."""

    def __init__(self, device="cuda", group=None):
        import torch.distributed as dist

        self.group = group
        self.part = dist.get_rank(group)
        self.parts = dist.get_world_size(group)
        self.device = device
        self._inner = TorchComm(device, group)

    def _peer(self, part):
        import torch.distributed as dist

        return part if self.group is None else dist.get_global_rank(self.group, part)

    def exchange_planes(self, send_lo, recv_lo, send_hi, recv_hi, n, stream=None):
        import torch.distributed as dist

        with _on_stream(stream, self.device):
            ops = []
            if send_lo and self.part > 0:
                ops.append(dist.P2POp(dist.isend, _view(send_lo, n, self.device), self._peer(self.part - 1),
                                      group=self.group))
                ops.append(dist.P2POp(dist.irecv, _view(recv_lo, n, self.device), self._peer(self.part - 1),
                                      group=self.group))
            if send_hi and self.part + 1 < self.parts:
                ops.append(dist.P2POp(dist.isend, _view(send_hi, n, self.device), self._peer(self.part + 1),
                                      group=self.group))
                ops.append(dist.P2POp(dist.irecv, _view(recv_hi, n, self.device), self._peer(self.part + 1),
                                      group=self.group))
            if ops:
                for w in dist.batch_isend_irecv(ops):
                    w.wait()

    def allreduce_sum(self, buf, n, stream=None):
        self._inner.allreduce_sum(buf, n, stream)

    def allgather(self, send, recv, n, stream=None):
        self._inner.allgather(send, recv, n, stream)


def nccl_comm(device: Optional[int] = None, group=None):
    """The library's C++ NCCL communicator (``NcclComm``) for the ranks of a
    torch.distributed process group: rank 0 makes the NCCL unique id, the
    group broadcasts its 128 bytes once, every rank creates its communicator.
    Afterwards every halo, all-reduce and all-gather of the all-at-once solve
    is an NCCL call inside libstmg_b200 (no Python per exchange)."""
    import torch
    import torch.distributed as dist

    from . import NcclComm

    rank, world = dist.get_rank(group), dist.get_world_size(group)
    dev = torch.cuda.current_device() if device is None else device
    uid = torch.zeros(128, dtype=torch.uint8)
    if rank == 0:
        uid.copy_(torch.frombuffer(bytearray(NcclComm.unique_id()), dtype=torch.uint8))
    backend = dist.get_backend(group)
    src = 0 if group is None else dist.get_global_rank(group, 0)  # broadcast takes a global rank
    if backend == "nccl":
        uid_dev = uid.to(f"cuda:{dev}")
        dist.broadcast(uid_dev, src, group=group)
        uid = uid_dev.cpu()
    else:
        dist.broadcast(uid, src, group=group)
    return NcclComm(rank, world, dev, bytes(uid.numpy().tobytes()))
