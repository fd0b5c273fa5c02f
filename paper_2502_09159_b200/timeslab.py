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
