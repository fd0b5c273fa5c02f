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


# ------------------------------------------------ communicator callbacks
# The library's stmg_comm_ops receive raw pointers. TorchComm is the
# implementation bench.py installs over NCCL; here it runs over gloo on host
# buffers (same code, device "cpu") and LoopbackComm on host threads.

def _comm_worker(rank, world, port, out):
    import ctypes

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = timeslab.TorchComm(device="cpu")
    n = 5
    send = np.arange(n, dtype=np.float64) + 100 * rank
    recv = np.full(n, -1.0)
    comm.exchange_halo(send.ctypes.data, recv.ctypes.data, n, None)
    buf = np.full(3, rank + 1.0)
    comm.allreduce_sum(buf.ctypes.data, 3, None)
    gat = np.zeros(n * world)
    comm.allgather(send.ctypes.data, gat.ctypes.data, n, None)
    out.put((rank, recv.copy(), buf.copy(), gat.copy()))
    dist.destroy_process_group()
    del ctypes


@pytest.mark.parametrize("world", [2, 3])
def test_torch_comm_callbacks_over_gloo(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_comm_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, recv, buf, gat = q.get(timeout=300)
        res[rank] = (recv, buf, gat)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    n = 5
    every = np.concatenate([np.arange(n) + 100.0 * r for r in range(world)])
    for rank, (recv, buf, gat) in res.items():
        if rank == 0:
            assert np.all(recv == -1.0)  # first rank receives nothing
        else:
            assert np.array_equal(recv, np.arange(n) + 100.0 * (rank - 1))
        assert np.all(buf == world * (world + 1) / 2)
        assert np.array_equal(gat, every)


def test_loopback_comm_threads_on_host():
    import threading

    world, n = 3, 4
    hub = timeslab.LoopbackHub(world, timeout=30)
    res, errs = {}, []

    def run(rank):
        try:
            c = timeslab.LoopbackComm(hub, rank, device="cpu")
            send = np.arange(n, dtype=np.float64) + 10 * rank
            recv = np.full(n, -1.0)
            c.exchange_halo(send.ctypes.data, recv.ctypes.data, n, None)
            buf = np.array([rank + 0.5, 1.0])
            c.allreduce_sum(buf.ctypes.data, 2, None)
            gat = np.zeros(n * world)
            c.allgather(send.ctypes.data, gat.ctypes.data, n, None)
            res[rank] = (recv, buf, gat)
        except BaseException as exc:
            errs.append(exc)
            hub.barrier.abort()

    ts = [threading.Thread(target=run, args=(r,)) for r in range(world)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(60)
    assert not errs, errs
    every = np.concatenate([np.arange(n) + 10.0 * r for r in range(world)])
    for rank, (recv, buf, gat) in res.items():
        assert np.array_equal(recv, np.full(n, -1.0) if rank == 0 else np.arange(n) + 10.0 * (rank - 1))
        assert np.allclose(buf, [sum(r + 0.5 for r in range(world)), world])
        assert np.array_equal(gat, every)
