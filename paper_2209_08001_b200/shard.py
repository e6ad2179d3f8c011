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


def _is_gloo(group=None):
    import torch.distributed as dist
    return dist.get_backend(group) == "gloo"


def halo_exchange(t, group=None, ghost: int = GHOST):
    """Fill the `ghost` ghost planes on each side of t[..., nz_own + 2*ghost, ny, nx] from the periodic
    neighbours.

    t is a torch tensor (CPU or CUDA); its own planes are t[..., ghost:-ghost, :, :].  group: a
    torch.distributed ProcessGroup or None (the default group; no group initialised means one rank).
    NCCL exchanges device tensors directly (send/recv over NVLink); gloo stages CUDA tensors through
    host memory.  Uses batched isend/irecv; returns after the exchange completed.
    """
    import torch
    g = int(ghost)
    nz_loc = t.shape[-3]
    own = nz_loc - 2 * g
    if own < g:
        raise ValueError(f"a slab must own at least {g} planes")
    # contiguous send/recv buffers (the planes are strided when leading field axes exist)
    send_lo = t[..., g:2 * g, :, :].contiguous()             # my first own planes -> rank-1's top ghosts
    send_hi = t[..., own:own + g, :, :].contiguous()         # my last own planes -> rank+1's bottom ghosts
    world, rank = _world(group)
    if world == 1:
        t[..., nz_loc - g:, :, :] = send_lo
        t[..., :g, :, :] = send_hi
        return t
    import torch.distributed as dist
    stage = t.is_cuda and _is_gloo(group)
    if stage:
        send_lo, send_hi = send_lo.cpu(), send_hi.cpu()
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
    t[..., :g, :, :] = recv_lo.to(t.device, non_blocking=False) if stage else recv_lo
    t[..., nz_loc - g:, :, :] = recv_hi.to(t.device, non_blocking=False) if stage else recv_hi
    return t


def allreduce_fixed_order(buf, group=None):
    """In-place sum of buf over the ranks, added in rank order 0, 1, ..., world-1 on every rank.

    An all-gather followed by a left-to-right sum: every rank obtains bitwise identical values (so
    control decisions taken from them agree across ranks) and the result does not depend on the
    collective's internal algorithm (reading R37; SURVEY Z34 fixed-order reductions).
    """
    import torch
    import torch.distributed as dist
    world, _ = _world(group)
    if world == 1:
        return buf
    src = buf.cpu() if (buf.is_cuda and _is_gloo(group)) else buf.contiguous()
    parts = [torch.empty_like(src) for _ in range(world)]
    dist.all_gather(parts, src, group=group)
    acc = parts[0].clone()
    for r in range(1, world):
        acc += parts[r]
    buf.copy_(acc)
    return buf


def box_slab_bounds(nz: int, nsub_z: int, world: int, rank: int):
    """z range and box count of `rank` when the nsub_z global boxes along z (split like the library's
    split: the first nz % nsub_z boxes one plane longer) are dealt out contiguously.  A slab made of
    whole boxes keeps the global subdomain grid -- and so GMRES's iteration counts -- independent of
    the number of ranks."""
    if nsub_z < world:
        raise ValueError(f"nsub_z = {nsub_z} boxes cannot be dealt to {world} ranks")
    base, rem = divmod(nz, nsub_z)
    starts = [b * base + min(b, rem) for b in range(nsub_z + 1)]
    b0, b1 = slab_bounds(nsub_z, world, rank)
    return starts[b0], starts[b1], b1 - b0


class SlabOperators:
    """F and J.v of one z-slab through the C ABI (the library state has zghost = 2).

    The caller supplies X^n, X^b, v as local arrays with ghosts; `residual` / `jv` exchange the ghosts
    of every input first (the exchange is part of the operator) and return the own planes.
    """

    def __init__(self, shape_global, model, solver, group=None, h=0.25, device=None, world=None, rank=None):
        import torch
        from .nks import PC_NONE, Solver, make_grid
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
        grid = make_grid(self.local_shape, h, None, 2, GHOST, z_offset=self.lo, nz_global=nz)
        self.solver = Solver(self.local_shape, model, sol, h=h, pc_type=PC_NONE, device=device, grid=grid)
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


class ShardedSolver:
    """One z-slab of a 3D periodic grid per rank, stepped by the library's full NKS step.

    The library decomposes the grid (nks_decompose: every rank owns whole layers of the global RAS box
    grid, so the preconditioner -- and the iteration counts -- do not depend on the number of ranks) and,
    with comm="nccl", owns the communication: rank 0's nks_get_unique_id is broadcast over the torch
    process group, nks_create builds an NCCL communicator, and the halo exchanges (grouped ncclSend/ncclRecv)
    and fixed-order reductions (ncclAllGather + rank-ordered sum) run inside the library on its stream --
    no Python in the per-iteration path.  comm="callbacks" attaches this object's host callbacks instead
    (torch.distributed exchanges; gloo stages through host memory) -- used to emulate several ranks on one
    GPU or on CPU process groups.  comm="auto": "nccl" when the group's backend is NCCL or it has one rank.

    shape_global / nsub: C order (nz, ny, nx).  group: a torch.distributed process group or None (the
    default group; none initialised = one rank).
    """

    def __init__(self, shape_global, model, solver, h=0.25, nsub=(1, 1, 1), overlap=2, pc_type=None,
                 pc_reuse=1, group=None, device=None, comm="auto"):
        import torch
        from .nks import PC_RAS_BILU0, Solver, decompose, make_grid, make_params, unique_id
        if len(shape_global) != 3:
            raise ValueError("z-slab sharding is 3D")
        self.torch = torch
        self.group = group
        self.world, self.rank = _world(group)
        self.shape_global = tuple(int(v) for v in shape_global)
        nz, ny, nx = self.shape_global
        self.pc_type = PC_RAS_BILU0 if pc_type is None else pc_type
        self.nsub_z = int(nsub[0])
        params = make_params(model, solver, self.pc_type, pc_reuse)
        self.lgrid = decompose(make_grid(self.shape_global, h, nsub, overlap), params, self.rank, self.world)
        self.zghost = zg = int(self.lgrid.zghost)
        self.lo = int(self.lgrid.z_offset)
        self.own = int(self.lgrid.n[2]) - 2 * zg
        self.hi = self.lo + self.own
        self.local_shape = (self.own + 2 * zg, ny, nx)
        self.model, self.solver_cfg, self.h = model, solver, h
        if comm == "auto":
            comm = "nccl" if (self.world == 1 or not _is_gloo(group)) else "callbacks"
        self.comm = comm
        self.halo_calls = 0
        self.allreduce_calls = 0
        nccl_id = None
        if comm == "nccl":
            nccl_id = unique_id() if self.rank == 0 else None
            if self.world > 1:
                import torch.distributed as dist
                box = [nccl_id]
                src = dist.get_global_rank(group, 0) if group is not None else 0
                dist.broadcast_object_list(box, src=src, group=group)
                nccl_id = box[0]
        self.solver = Solver(self.local_shape, model, solver, h=h, pc_type=self.pc_type, pc_reuse=pc_reuse,
                             device=device, grid=self.lgrid, rank=self.rank, nranks=self.world, nccl_id=nccl_id)
        self.device = self.solver.device
        if comm == "callbacks":
            self.solver.set_comm(self._allreduce, self._halo)

    # ---------------------------------------------------------------- callbacks (library -> here)
    def _allreduce(self, ptr, n, stream):
        self.allreduce_calls += 1
        with self.torch.cuda.stream(self.solver.stream):
            allreduce_fixed_order(self.solver.device_view(ptr, n), self.group)
        return 0

    def _halo(self, ptr, nf, stride, stream):
        self.halo_calls += 1
        nz_loc, ny, nx = self.local_shape
        if stride != nz_loc * ny * nx:
            raise ValueError("unexpected field stride")
        v = self.solver.device_view(ptr, nf * stride).view(nf, nz_loc, ny, nx)
        with self.torch.cuda.stream(self.solver.stream):
            halo_exchange(v, self.group, self.zghost)
        return 0

    # ---------------------------------------------------------------- API (global arrays in, local work)
    def local(self, field):
        """This rank's local slab (own planes + ghosts) of a global (..., nz, ny, nx) field."""
        nz = self.shape_global[0]
        idx = [(z % nz) for z in range(self.lo - self.zghost, self.hi + self.zghost)]
        if isinstance(field, np.ndarray):
            return field[..., idx, :, :].copy()
        t = self.torch
        return field[..., t.tensor(idx, device=field.device), :, :].contiguous()

    def set_fields(self, c, eta, u=None):
        """Global c, eta (nz, ny, nx) and optionally u (3, nz, ny, nx), the same on every rank; each rank
        passes its slab.  Without u the library solves u^0 on the slabs themselves (conjugate gradients on
        the elastic block with halo exchanges and allreduces, reading R13) -- no rank holds the whole grid."""
        t = self.torch
        c = t.as_tensor(np.asarray(c) if not isinstance(c, t.Tensor) else c, dtype=t.float64).to(self.device)
        eta = t.as_tensor(np.asarray(eta) if not isinstance(eta, t.Tensor) else eta, dtype=t.float64).to(self.device)
        if u is not None:
            u = t.as_tensor(np.asarray(u) if not isinstance(u, t.Tensor) else u, dtype=t.float64).to(self.device)
            u = self.local(u)
        self.solver.set_fields(self.local(c), self.local(eta), u)

    def step(self, dt, raise_on_fail=True):
        return self.solver.step(dt, raise_on_fail=raise_on_fail)

    def run_adaptive(self, max_steps, t_end=0.0):
        return self.solver.run_adaptive(max_steps, t_end)

    def energy(self):
        return self.solver.energy()

    def own_state(self):
        """X^n on the own planes, (5, own, ny, nx) device tensor."""
        zg = self.zghost
        return self.solver.get_state_device()[:, zg:zg + self.own]

    def gather_state(self):
        """The global X^n (5, nz, ny, nx) as numpy, on every rank (all-gather of the own planes)."""
        import torch.distributed as dist
        own = self.own_state()
        if self.world == 1:
            return own.cpu().numpy()
        nz, ny, nx = self.shape_global
        src = own.contiguous().cpu() if _is_gloo(self.group) else own.contiguous()
        sizes = [hi - lo for lo, hi in (self.slab_of(r) for r in range(self.world))]
        parts = [self.torch.empty((5, sz, ny, nx), dtype=src.dtype, device=src.device) for sz in sizes]
        if len(set(sizes)) == 1:
            dist.all_gather(parts, src, group=self.group)
        else:      # unequal slabs: pad to the largest
            m = max(sizes)
            pad = self.torch.zeros((5, m, ny, nx), dtype=src.dtype, device=src.device)
            pad[:, :src.shape[1]] = src
            full = [self.torch.empty_like(pad) for _ in range(self.world)]
            dist.all_gather(full, pad, group=self.group)
            parts = [f[:, :sz] for f, sz in zip(full, sizes)]
        return self.torch.cat([p.cpu() for p in parts], dim=1).numpy()

    def slab_of(self, r):
        """(lo, hi) global z range of rank r (the library's decomposition)."""
        from .nks import decompose, make_grid, make_params
        params = make_params(self.model, self.solver_cfg, self.pc_type)
        nz, ny, nx = self.shape_global
        lg = decompose(make_grid(self.shape_global, self.h, (self.nsub_z, 1, 1), self.lgrid.overlap), params, r,
                       self.world)
        return int(lg.z_offset), int(lg.z_offset) + int(lg.n[2]) - 2 * int(lg.zghost)


def run_halo_plan(vec, plan, local, rank: int, group=None):
    """Execute the library's halo message list (nks_halo_plan: the ncclSend/ncclRecv sequence the library
    issues) with torch.distributed point-to-point calls on a flat tensor `vec` of one local vector.

    Kinds 0 / 1 send / receive `count` contiguous doubles at `offset`; kinds 2 / 3 (pencils) a y block of
    `count` doubles per own plane, packed plane after plane.  Messages are matched per peer in issue order
    (the k-th message between two ranks gets tag k on both sides, NCCL's rule); a pencil's y phase completes
    before its plane phase starts.  Messages to this rank itself (a process-grid axis of length 1) pair up
    locally in the same order."""
    import torch
    import torch.distributed as dist
    nx, nyl, nzl = local.n[0], local.n[1], local.n[2]
    nxy, zg = nx * nyl, local.zghost
    nzo = nzl - 2 * zg

    def gather(off, cnt, kind):
        if kind < 2:
            return vec[off:off + cnt].clone()
        return torch.stack([vec[off + p * nxy: off + p * nxy + cnt] for p in range(nzo)]).reshape(-1).clone()

    def scatter(off, cnt, kind, buf):
        if kind < 2:
            vec[off:off + cnt] = buf
            return
        b = buf.view(nzo, cnt)
        for p in range(nzo):
            vec[off + p * nxy: off + p * nxy + cnt] = b[p]

    seq_send, seq_recv = {}, {}
    for phase in ((2, 3), (0, 1)):
        reqs, self_q, pending_self = [], [], []
        for kind, peer, off, cnt in plan:
            if kind not in phase:
                continue
            sending = kind in (0, 2)
            if peer == rank:
                (self_q if sending else pending_self).append(gather(off, cnt, kind) if sending else (off, cnt, kind))
                continue
            if sending:
                tag = seq_send.get(peer, 0)
                seq_send[peer] = tag + 1
                reqs.append(dist.isend(gather(off, cnt, kind), peer, tag=tag, group=group))
            else:
                tag = seq_recv.get(peer, 0)
                seq_recv[peer] = tag + 1
                buf = torch.empty(cnt * (nzo if kind == 3 else 1), dtype=vec.dtype)
                reqs.append((dist.irecv(buf, peer, tag=tag, group=group), off, cnt, kind, buf))
        for (off, cnt, kind), buf in zip(pending_self, self_q):
            scatter(off, cnt, kind, buf)
        for r in reqs:
            if isinstance(r, tuple):
                r[0].wait()
                scatter(r[1], r[2], r[3], r[4])
            else:
                r.wait()


class PencilSolver:
    """One z x y pencil of a 3D periodic grid per rank on a pz x py process grid (rank = rz * py + ry), for the
    full NKS step and for F / J.v alone ("pencil z x y (2x2, 2x4) for 4 and 8 GPUs"; BASELINE
    configs 4/5 "slab- then pencil-sharded").

    The library decomposes the grid (nks_decompose_pencil: with RAS every rank owns whole layers of the global
    box grid along z AND y, so the preconditioner -- and the iteration counts -- do not depend on the process
    grid) and fills the ghost planes and rows itself: with comm="nccl" through its own communicator (y blocks
    packed and exchanged in one NCCL group, then whole planes, so the (y, z) edge cells arrive), with
    comm="callbacks" through this object's host callbacks, which run the library's own message list
    (nks_halo_plan) over the torch process group (host-staged; emulated ranks on one GPU)."""

    def __init__(self, shape_global, model, solver, pz, py, h=0.25, nsub=(1, 1, 1), overlap=2, pc_type=None,
                 pc_reuse=1, group=None, device=None, comm="auto"):
        import torch
        from .nks import PC_NONE, Solver, decompose_pencil, halo_plan, make_grid, make_params, unique_id
        self.torch = torch
        self.group = group
        self.world, self.rank = _world(group)
        if self.world != pz * py:
            raise ValueError("the process grid pz x py must match the group size")
        self.shape_global = tuple(int(v) for v in shape_global)
        self.pc_type = PC_NONE if pc_type is None else pc_type
        params = make_params(model, solver, self.pc_type, pc_reuse)
        self.lgrid = decompose_pencil(make_grid(self.shape_global, h, nsub, overlap), params, self.rank, pz, py)
        g = self.lgrid
        self.zg, self.yg = int(g.zghost), int(g.yghost)
        self.z0, self.y0 = int(g.z_offset), int(g.y_offset)
        self.local_shape = (int(g.n[2]), int(g.n[1]), int(g.n[0]))
        self.nzo, self.nyo = self.local_shape[0] - 2 * self.zg, self.local_shape[1] - 2 * self.yg
        if comm == "auto":
            comm = "nccl" if (self.world == 1 or not _is_gloo(group)) else "callbacks"
        self.comm = comm
        self.halo_calls = 0
        self.allreduce_calls = 0
        nccl_id = None
        if comm == "nccl":
            nccl_id = unique_id() if self.rank == 0 else None
            if self.world > 1:
                import torch.distributed as dist
                box = [nccl_id]
                src = dist.get_global_rank(group, 0) if group is not None else 0
                dist.broadcast_object_list(box, src=src, group=group)
                nccl_id = box[0]
        self.solver = Solver(self.local_shape, model, solver, h=h, pc_type=self.pc_type, pc_reuse=pc_reuse,
                             device=device, grid=g, rank=self.rank, nranks=self.world, nccl_id=nccl_id)
        self.device = self.solver.device
        self._plan = {}
        self._halo_plan = halo_plan
        if comm == "callbacks":
            self.solver.set_comm(self._allreduce, self._halo)

    def _allreduce(self, ptr, n, stream):
        self.allreduce_calls += 1
        with self.torch.cuda.stream(self.solver.stream):
            allreduce_fixed_order(self.solver.device_view(ptr, n), self.group)
        return 0

    def _halo(self, ptr, nf, stride, stream):
        self.halo_calls += 1
        if nf not in self._plan:
            self._plan[nf] = self._halo_plan(self.lgrid, self.rank, self.world, nf)
        v = self.solver.device_view(ptr, nf * stride)
        self.solver.stream.synchronize()
        host = v.cpu() if (self.world > 1 and _is_gloo(self.group)) else v
        run_halo_plan(host, self._plan[nf], self.lgrid, self.rank, self.group)
        if host is not v:
            with self.torch.cuda.stream(self.solver.stream):
                v.copy_(host.to(self.device))
        return 0

    def local(self, field):
        """This rank's pencil (own planes / rows + ghosts, periodic) of a global (..., nz, ny, nx) field."""
        nz, ny, _ = self.shape_global
        zi = [(z % nz) for z in range(self.z0 - self.zg, self.z0 + self.nzo + self.zg)]
        yi = [(y % ny) for y in range(self.y0 - self.yg, self.y0 + self.nyo + self.yg)]
        a = np.asarray(field)
        return a[..., zi, :, :][..., yi, :].copy()

    def own(self, local_field):
        """The own planes / rows of a local (..., nzl, nyl, nx) field."""
        return local_field[..., self.zg:self.zg + self.nzo, self.yg:self.yg + self.nyo, :]

    def set_fields(self, c, eta, u=None):
        """Global c, eta (nz, ny, nx) and optionally u (3, nz, ny, nx); without u the library solves u^0 by
        conjugate gradients on the pencils (reading R13).  The ghosts are refilled by the library."""
        self.solver.set_fields(self.local(c), self.local(eta), None if u is None else self.local(u))

    def step(self, dt, raise_on_fail=True):
        return self.solver.step(dt, raise_on_fail=raise_on_fail)

    def own_state(self):
        """(5, nzo, nyo, nx) numpy array of this rank's own points of X^n."""
        return np.ascontiguousarray(self.own(self.solver.get_state()))

    def _nan_ghosts(self, a):
        a[:, :self.zg] = np.nan
        a[:, -self.zg:] = np.nan
        a[:, :, :self.yg] = np.nan
        a[:, :, -self.yg:] = np.nan
        return a

    def residual(self, Xb, dt):
        """F on the own points for a global state Xb (5, nz, ny, nx); the local ghosts are sent as NaN and
        refilled by the library's halo exchange."""
        return self.own(self.solver.eval_residual(self._nan_ghosts(self.local(Xb)), dt))

    def jv(self, Xb, v, dt):
        return self.own(self.solver.eval_jv(self._nan_ghosts(self.local(Xb)), self._nan_ghosts(self.local(v)), dt))
