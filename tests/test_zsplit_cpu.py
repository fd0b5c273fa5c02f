"""CPU tier: host logic of the C5 hybrid split -- the z parts' dof maps cover
the whole mesh with exactly the interface planes shared, and the parts'
communicator (timeslab.TorchSpaceComm) exchanges interface planes, sums and
gathers correctly over gloo with 3 ranks."""
import os
import socket

import numpy as np
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2502_09159_b200 import timeslab


def test_z_part_dofs_cover_mesh_once_except_interfaces():
    nx, ny, nz, r, k, parts = 3, 2, 6, 2, 1, 3
    p, S, npm = r + 1, k + 1, (r + 1) * (r + 2) * (r + 3) // 6
    gx, gy, gz = nx * p + 1, ny * p + 1, nz * p + 1
    size = S * 3 * gx * gy * gz + S * nx * ny * nz * npm
    count = np.zeros(size, dtype=int)
    for part in range(parts):
        idx = timeslab.z_part_dofs(nx, ny, nz, r, k, parts, part)
        assert len(np.unique(idx)) == len(idx)
        count[idx] += 1
    assert count.min() == 1
    # exactly the velocity nodes of the parts' interface planes are held twice
    twice = np.flatnonzero(count == 2)
    plane = gx * gy
    nzl = nz // parts
    z_of = (twice % (gx * gy * gz)) // plane
    assert set(z_of.tolist()) == {q * nzl * p for q in range(1, parts)}
    assert len(twice) == (parts - 1) * S * 3 * plane
    assert count.max() == 2


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    comm = timeslab.TorchSpaceComm(device="cpu")
    n = 5
    lo = torch.full((n,), 10.0 * rank + 1)
    hi = torch.full((n,), 10.0 * rank + 2)
    rlo = torch.zeros(n, dtype=torch.float64)
    rhi = torch.zeros(n, dtype=torch.float64)
    lo, hi = lo.double(), hi.double()
    has_lo, has_hi = rank > 0, rank + 1 < world
    comm.exchange_planes(lo.data_ptr() if has_lo else 0, rlo.data_ptr() if has_lo else 0,
                         hi.data_ptr() if has_hi else 0, rhi.data_ptr() if has_hi else 0, n)
    s = torch.tensor([float(rank + 1)], dtype=torch.float64)
    comm.allreduce_sum(s.data_ptr(), 1)
    g = torch.zeros(2 * world, dtype=torch.float64)
    mine = torch.tensor([rank, -rank], dtype=torch.float64)
    comm.allgather(mine.data_ptr(), g.data_ptr(), 2)
    q.put((rank, rlo.tolist(), rhi.tolist(), float(s[0]), g.tolist()))
    dist.destroy_process_group()


def test_space_comm_over_gloo():
    world = 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(world):
        rank, rlo, rhi, s, g = q.get(timeout=120)
        res[rank] = (rlo, rhi, s, g)
    for p in procs:
        p.join(60)
        assert p.exitcode == 0
    for rank in range(world):
        rlo, rhi, s, g = res[rank]
        # lower neighbour sent its upper plane (10 (rank-1) + 2), upper one its lower (10 (rank+1) + 1)
        assert rlo == ([10.0 * (rank - 1) + 2] * 5 if rank > 0 else [0.0] * 5)
        assert rhi == ([10.0 * (rank + 1) + 1] * 5 if rank + 1 < world else [0.0] * 5)
        assert s == 6.0
        assert g == [0.0, -0.0, 1.0, -1.0, 2.0, -2.0]
