"""CPU tier, world_size 2 over gloo: the time-slab partition (halo exchange of
the slot-k velocity) reproduces the unpartitioned all-at-once vmult and
smoother step. The per-rank compute is the oracle (test infrastructure), so
this checks the partition protocol that bench.py runs over NCCL."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle_ctypes as oc
from paper_2502_09159_b200 import timeslab

NC, R, K, TAU, NU, GAMMA, N_GLOBAL = 8, 1, 1, 1.0 / 8, 1.0, 1.0, 6


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, out):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    lvl = oc.OracleLevel(NC, R, K, TAU, NU, GAMMA, 0)
    isz, mv, S = lvl.size, lvl.n_velocity, lvl.n_slots
    x = oc.seeded(N_GLOBAL * isz, 5)
    b = oc.seeded(N_GLOBAL * isz, 6)
    mine = timeslab.owned_intervals(N_GLOBAL, rank, world)
    nl = len(mine)
    xl = torch.from_numpy(x[mine.start * isz: mine.stop * isz].copy())
    bl = b[mine.start * isz: mine.stop * isz].copy()
    halo = torch.zeros(mv, dtype=torch.float64)
    h = timeslab.exchange_halo(xl, halo, nl, isz, mv, S, rank, world)
    h_np = None if h is None else h.numpy().copy()
    y = lvl.vmult_all(xl.numpy().copy(), nl, h_np)
    u = lvl.smooth_step_all(bl, xl.numpy().copy(), 0.8, nl, h_np)
    parts_y = [None] * world
    parts_u = [None] * world
    dist.all_gather_object(parts_y, y)
    dist.all_gather_object(parts_u, u)
    if rank == 0:
        out.put((np.concatenate(parts_y), np.concatenate(parts_u)))
    dist.destroy_process_group()


def test_owned_intervals_cover_all():
    for n, w in [(64, 8), (7, 3), (5, 5), (3, 1)]:
        seen = [i for r in range(w) for i in timeslab.owned_intervals(n, r, w)]
        assert seen == list(range(n))


def test_time_slab_partition_matches_single_process(oracle):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    y_part, u_part = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    lvl = oc.OracleLevel(NC, R, K, TAU, NU, GAMMA, 0)
    x = oc.seeded(N_GLOBAL * lvl.size, 5)
    b = oc.seeded(N_GLOBAL * lvl.size, 6)
    y_ref = lvl.vmult_all(x, N_GLOBAL, None)
    u_ref = lvl.smooth_step_all(b, x, 0.8, N_GLOBAL, None)
    assert np.array_equal(y_part, y_ref)
    assert np.array_equal(u_part, u_ref)
