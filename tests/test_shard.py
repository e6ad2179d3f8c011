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


def _worker_wide(rank, world, port, nz, ghost, out):
    """Ghost width 3 (RAS overlap 2 + 1) and the fixed-order allreduce of the sharded step."""
    from paper_2209_08001_b200.shard import allreduce_fixed_order
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        g = np.random.default_rng(7).standard_normal((5, nz, 3, 4))
        lo, hi = slab_bounds(nz, world, rank)
        idx = [(z % nz) for z in range(lo - ghost, hi + ghost)]
        want = g[:, idx].copy()
        loc = torch.from_numpy(want.copy())
        loc[:, :ghost] = np.nan
        loc[:, -ghost:] = np.nan
        halo_exchange(loc, ghost=ghost)
        err = float(np.abs(loc.numpy() - want).max())
        # allreduce: the per-rank partial sums of a global vector, added in rank order 0..world-1
        vals = np.random.default_rng(11).standard_normal((world, 6))
        buf = torch.from_numpy(vals[rank].copy())
        allreduce_fixed_order(buf)
        ref = vals[0].copy()
        for r in range(1, world):
            ref = ref + vals[r]
        out[rank] = (err, buf.numpy().tobytes() == ref.tobytes())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,nz,ghost", [(2, 12, 3), (3, 18, 3), (2, 16, 4)])
def test_wide_halo_and_fixed_order_allreduce_gloo(world, nz, ghost):
    mgr = mp.Manager()
    out = mgr.dict()
    mp.spawn(_worker_wide, args=(world, _free_port(), nz, ghost, out), nprocs=world, join=True)
    assert sorted(out.keys()) == list(range(world))
    for r, (err, exact) in out.items():
        assert err == 0.0, (r, err)
        assert exact, r              # bitwise identical on every rank, and equal to the rank-ordered sum


def test_box_slab_bounds_keep_whole_boxes():
    from paper_2209_08001_b200.shard import box_slab_bounds
    for nz, nb in ((16, 4), (10, 4), (18, 6), (256, 8), (129, 8)):
        base, rem = divmod(nz, nb)
        starts = {b * base + min(b, rem) for b in range(nb + 1)}
        for world in (1, 2, 3, 4, 8):
            if world > nb:
                continue
            b = [box_slab_bounds(nz, nb, world, r) for r in range(world)]
            assert b[0][0] == 0 and b[-1][1] == nz
            assert all(b[r][1] == b[r + 1][0] for r in range(world - 1))
            assert all(lo in starts and hi in starts for lo, hi, _ in b)
            assert sum(k for _, _, k in b) == nb


# ---------------------------------------------------------------------------------------- the library's own plan
def _plan_worker(rank, world, port, out):
    """Each rank takes its slab from the library (nks_decompose) and executes the library's halo message list
    (nks_halo_plan -- the ncclSend/ncclRecv sequence the library issues) over gloo.  NCCL pairs the messages of
    two ranks in issue order; gloo pairs them by tag, so the k-th message between a given sender and receiver
    gets tag k on both sides -- the same matching."""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        import nks_inputs as ni
        from paper_2209_08001_b200 import nks
        nz, ny, nx, nf = 24, 6, 5, 5
        params = nks.make_params(ni.model_default(), ni.solver_default())
        lg = nks.decompose(nks.make_grid((nz, ny, nx), 0.25, (world * 2, 1, 1), 2), params, rank, world)
        zg, nzl = lg.zghost, lg.n[2]
        g = np.random.default_rng(7).standard_normal((nf, nz, ny, nx))
        idx = [(z % nz) for z in range(lg.z_offset - zg, lg.z_offset - zg + nzl)]
        want = g[:, idx]
        vec = torch.from_numpy(want.copy()).reshape(-1)
        flat = vec.view(nf, nzl, ny, nx)
        flat[:, :zg] = np.nan
        flat[:, -zg:] = np.nan
        plan = nks.halo_plan(lg, rank, world, nf)
        assert len(plan) == 4 * nf
        seq_send, seq_recv, reqs = {}, {}, []
        for kind, peer, off, cnt in plan:
            if kind == 0:
                tag = seq_send.get(peer, 0)
                seq_send[peer] = tag + 1
                reqs.append(dist.isend(vec[off:off + cnt].clone(), peer, tag=tag))
            else:
                tag = seq_recv.get(peer, 0)
                seq_recv[peer] = tag + 1
                buf = torch.empty(cnt, dtype=vec.dtype)
                reqs.append((dist.irecv(buf, peer, tag=tag), off, buf))
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                vec[r[1]:r[1] + r[2].numel()] = r[2]
            else:
                r.wait()
        out[rank] = float(np.abs(vec.view(nf, nzl, ny, nx).numpy() - want).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2, 3, 4])
def test_library_halo_plan_over_gloo(world):
    out = mp.Manager().dict()
    mp.spawn(_plan_worker, args=(world, _free_port(), out), nprocs=world, join=True)
    assert all(out[r] == 0.0 for r in range(world)), dict(out)


# ---------------------------------------------------------------------------------------- pencils (z x y)
def _pencil_worker(rank, world, pz, py, port, out):
    """Each rank takes its pencil from the library (nks_decompose_pencil) and runs the library's pencil halo
    plan (y blocks, then whole planes) over gloo; every ghost cell -- the (y, z) edges included, which the
    J.v stencil's (0, +-1, +-1) offsets read -- must equal the global periodic field."""
    dist.init_process_group("gloo", init_method=f"tcp://127.0.0.1:{port}", rank=rank, world_size=world)
    try:
        from paper_2209_08001_b200 import nks
        from paper_2209_08001_b200.shard import run_halo_plan
        nz, ny, nx, nf = 12, 10, 5, 5
        import nks_inputs as ni
        p0 = nks.make_params(ni.model_default(), ni.solver_default(), nks.PC_NONE)
        lg = nks.decompose_pencil(nks.make_grid((nz, ny, nx), 0.25, (1, 1, 1), 2), p0, rank, pz, py)
        zg, yg, nzl, nyl = lg.zghost, lg.yghost, lg.n[2], lg.n[1]
        g = np.random.default_rng(11).standard_normal((nf, nz, ny, nx))
        zi = [(z % nz) for z in range(lg.z_offset - zg, lg.z_offset - zg + nzl)]
        yi = [(y % ny) for y in range(lg.y_offset - yg, lg.y_offset - yg + nyl)]
        want = g[:, zi][:, :, yi]
        arr = want.copy()
        arr[:, :zg] = np.nan
        arr[:, -zg:] = np.nan
        arr[:, :, :yg] = np.nan
        arr[:, :, -yg:] = np.nan
        vec = torch.from_numpy(arr).reshape(-1)
        plan = nks.halo_plan(lg, rank, world, nf)
        assert len(plan) == 8 * nf
        assert [m[0] for m in plan[:4 * nf]] == [2, 2, 3, 3] * nf      # y phase first
        run_halo_plan(vec, plan, lg, rank)
        out[rank] = float(np.abs(vec.view(nf, nzl, nyl, nx).numpy() - want).max())
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("pz,py", [(1, 2), (2, 1), (1, 3), (3, 1), (2, 2), (4, 1), (1, 4)])
def test_library_pencil_halo_plan_over_gloo(pz, py):
    world = pz * py
    out = mp.Manager().dict()
    mp.spawn(_pencil_worker, args=(world, pz, py, _free_port(), out), nprocs=world, join=True)
    assert all(out[r] == 0.0 for r in range(world)), dict(out)


def test_pencil_plan_single_rank_is_the_periodic_copy():
    """One rank (pz = py = 1, no process group): every message of the library's pencil plan goes to this rank
    itself and the executor pairs them locally -- the ghosts become the periodic images (RAS ghost width 3)."""
    import nks_inputs as ni
    from paper_2209_08001_b200 import nks
    from paper_2209_08001_b200.shard import run_halo_plan
    nz, ny, nx, nf = 12, 10, 6, 5
    p = nks.make_params(ni.model_default(), ni.solver_default(), nks.PC_RAS_BILU0)
    lg = nks.decompose_pencil(nks.make_grid((nz, ny, nx), 0.25, (2, 2, 1), 2), p, 0, 1, 1)
    assert lg.zghost == lg.yghost == 3
    zg, yg, nzl, nyl = lg.zghost, lg.yghost, lg.n[2], lg.n[1]
    g = np.random.default_rng(5).standard_normal((nf, nz, ny, nx))
    want = g[:, [(z - zg) % nz for z in range(nzl)]][:, :, [(y - yg) % ny for y in range(nyl)]]
    arr = want.copy()
    arr[:, :zg] = np.nan
    arr[:, -zg:] = np.nan
    arr[:, :, :yg] = np.nan
    arr[:, :, -yg:] = np.nan
    vec = torch.from_numpy(arr).reshape(-1)
    run_halo_plan(vec, nks.halo_plan(lg, 0, 1, nf), lg, 0)
    assert np.array_equal(vec.view(nf, nzl, nyl, nx).numpy(), want)
