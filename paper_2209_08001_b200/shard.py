"""z-slab sharding of a 3D periodic grid over the ranks of a torch.distributed process group
(DESIGN.md section 8).  Plumbing only -- the arithmetic runs in the library's kernels.

A rank owns the planes [z_lo, z_hi) of the global grid and holds them in a local array with 2 ghost
planes on each side (F and J.v are radius-2 stencils): local plane p <-> global plane
z_lo - 2 + p.  `halo_exchange` fills the ghosts from the periodic neighbours with point-to-point
send/recv (NCCL over NVLink on GPUs, gloo on CPU); with one rank it is the periodic self-copy.  A
library state created with ``zghost=2`` on the local shape (nz_own + 4) evaluates F and J.v on its own
planes without z wrap.
"""
from __future__ import annotations

import numpy as np

GHOST = 2


def slab_bounds(nz: int, world: int, rank: int):
    """Balanced contiguous z ranges: the first nz % world ranks get one extra plane."""
    base, rem = divmod(nz, world)
    lo = rank * base + min(rank, rem)
    return lo, lo + base + (1 if rank < rem else 0)


def local_from_global(field, lo: int, hi: int):
    """Slab [lo-2, hi+2) of a global periodic field (leading axes kept), as a new array/tensor."""
    nz = field.shape[-3]
    idx = [(z % nz) for z in range(lo - GHOST, hi + GHOST)]
    if isinstance(field, np.ndarray):
        return field[..., idx, :, :].copy()
    import torch
    return field[..., torch.tensor(idx, device=field.device), :, :].contiguous()


def _world(group=None):
    import torch.distributed as dist
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def halo_exchange(t, group=None):
    """Fill the 2 ghost planes on each side of t[..., nz_own + 4, ny, nx] from the periodic neighbours.

    t is a torch tensor (CPU with gloo, CUDA with NCCL); its own planes are t[..., 2:-2, :, :].
    group: a torch.distributed ProcessGroup or None (the default group; no group initialised means
    one rank).  Uses batched isend/irecv; returns after the exchange completed.
    """
    import torch
    nz_loc = t.shape[-3]
    own = nz_loc - 2 * GHOST
    if own < GHOST:
        raise ValueError("a slab must own at least 2 planes")
    # contiguous send/recv buffers (the planes are strided when leading field axes exist)
    send_lo = t[..., GHOST:2 * GHOST, :, :].contiguous()             # my first own planes -> rank-1's top ghosts
    send_hi = t[..., own:own + GHOST, :, :].contiguous()            # my last own planes -> rank+1's bottom ghosts
    world, rank = _world(group)
    if world == 1:
        t[..., nz_loc - GHOST:, :, :] = send_lo
        t[..., :GHOST, :, :] = send_hi
        return t
    import torch.distributed as dist
    up, dn = (rank + 1) % world, (rank - 1) % world
    gu = dist.get_global_rank(group, up) if group is not None else up
    gd = dist.get_global_rank(group, dn) if group is not None else dn
    recv_lo = torch.empty_like(send_lo)     # from rank-1: its last own planes -> my bottom ghosts
    recv_hi = torch.empty_like(send_hi)     # from rank+1: its first own planes -> my top ghosts
    # order (and tag) the messages so that they also match when up == dn (two ranks): the upward stream
    # (my last planes -> the next rank's bottom ghosts) first, then the downward one
    ops = [dist.P2POp(dist.isend, send_hi, gu, group=group, tag=0), dist.P2POp(dist.isend, send_lo, gd, group=group, tag=1),
           dist.P2POp(dist.irecv, recv_lo, gd, group=group, tag=0), dist.P2POp(dist.irecv, recv_hi, gu, group=group, tag=1)]
    for req in dist.batch_isend_irecv(ops):
        req.wait()
    t[..., :GHOST, :, :] = recv_lo
    t[..., nz_loc - GHOST:, :, :] = recv_hi
    return t


class SlabOperators:
    """F and J.v of one z-slab through the C ABI (the library state has zghost = 2).

    The caller supplies X^n, X^b, v as local arrays with ghosts; `residual` / `jv` exchange the ghosts
    of every input first (the exchange is part of the operator) and return the own planes.
    """

    def __init__(self, shape_global, model, solver, group=None, h=0.25, device=None, world=None, rank=None):
        import torch
        from .nks import PC_NONE, Solver
        self.group = group
        w, r = _world(group)
        world = w if world is None else world       # world/rank may be given explicitly (single-process emulation)
        rank = r if rank is None else rank
        # exchange through the group when there is one; the periodic self-copy for one rank; none when a
        # single process emulates several slabs (the caller fills the ghosts from the global field)
        self.exchange = w > 1 or world == 1
        nz, ny, nx = shape_global
        self.lo, self.hi = slab_bounds(nz, world, rank)
        self.own = self.hi - self.lo
        self.local_shape = (self.own + 2 * GHOST, ny, nx)
        sol = dict(solver)
        sol["gmres_restart"] = 1
        self.solver = Solver(self.local_shape, model, sol, h=h, pc_type=PC_NONE, zghost=GHOST, device=device)
        self.torch = torch

    def set_level_n(self, Xa, cbar0):
        """X^n (local, ghosts filled or not: they are exchanged here); cbar0 = the global mean of c^0."""
        Xa = halo_exchange(Xa, self.group) if self.exchange else Xa
        self.solver.set_fields(Xa[0], Xa[1], Xa[2:])
        self.solver.set_cbar0(cbar0)

    def residual(self, Xb, dt):
        Xb = halo_exchange(Xb, self.group) if self.exchange else Xb
        return self.solver.eval_residual(Xb, dt)[:, GHOST:-GHOST]

    def jv(self, Xb, v, dt):
        if self.exchange:
            Xb = halo_exchange(Xb, self.group)
            v = halo_exchange(v, self.group)
        return self.solver.eval_jv(Xb, v, dt)[:, GHOST:-GHOST]
