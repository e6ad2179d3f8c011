"""Multi-GPU plumbing of SURVEY 8(e) on the CPU: z-slab bounds and the periodic halo exchange over a
torch.distributed gloo group with world sizes 2 and 3 (the GPU run uses the same code with NCCL)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2209_08001_b200.shard import GHOST, halo_exchange, local_from_global, slab_bounds


def test_slab_bounds_partition():
    for nz in (5, 8, 17, 256):
        for world in (1, 2, 3, 4, 8):
            if world * 2 > nz:
                continue
            b = [slab_bounds(nz, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == nz
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            sizes = [hi - lo for lo, hi in b]
            assert max(sizes) - min(sizes) <= 1


def test_single_rank_exchange_is_periodic_copy():
    g = np.random.default_rng(0).standard_normal((3, 7, 4, 5))
    loc = torch.from_numpy(local_from_global(g, 0, 7))
    loc[:, :GHOST] = 0
    loc[:, -GHOST:] = 0
    halo_exchange(loc)
    np.testing.assert_array_equal(loc.numpy(), local_from_global(g, 0, 7))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, nz, out):
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        g = np.random.default_rng(42).standard_normal((5, nz, 3, 4))       # (fields, z, y, x)
        lo, hi = slab_bounds(nz, world, rank)
        want = local_from_global(g, lo, hi)
        loc = torch.from_numpy(want.copy())
        loc[:, :GHOST] = np.nan
        loc[:, -GHOST:] = np.nan
        halo_exchange(loc)
        out[rank] = float(np.abs(loc.numpy() - want).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nz", [(2, 8), (3, 10), (2, 5)])
def test_halo_exchange_gloo(world, nz):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker, args=(world, _free_port(), nz, out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    assert all(v == 0.0 for v in out.values()), dict(out)
