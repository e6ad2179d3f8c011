"""Thin ctypes binding of ``lib/libnks.so`` (include/nks.h).  Argument marshalling only: every
step of the NKS time step runs in the library's CUDA kernels.  PyTorch supplies device memory
(the workspace), the CUDA stream and the current device.

The library is loaded from the package's ``lib/`` directory; there is no fallback -- importing
this module without a built library or without a CUDA device raises.
"""
from __future__ import annotations

import ctypes as C
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("NKS_LIB", os.path.join(_HERE, "lib", "libnks.so"))   # NKS_LIB: experiments only

NKS_OK, NKS_E_INVALID, NKS_E_DOMAIN, NKS_E_DIVERGED, NKS_E_CUDA, NKS_E_NCCL, NKS_E_OOM, NKS_E_STATE = range(8)
STATUS = {0: "OK", 1: "INVALID", 2: "DOMAIN", 3: "DIVERGED", 4: "CUDA", 5: "NCCL", 6: "OOM", 7: "STATE"}
PC_NONE, PC_RAS_BILU0, PC_AS_BILU0, PC_RRAS_BILU0, PC_SPECTRAL, PC_RAS_SPECTRAL = 0, 2, 3, 4, 5, 6
REASONS = {0: "none", 1: "newton_maxit", 2: "line_search", 3: "gmres_maxit", 4: "domain", 5: "dt_floor",
           6: "gmres_stagnation", 7: "gmres_projected"}
PHASES = ["residual", "jv", "ras_apply", "assemble", "factor", "gmres_vec", "reductions", "other"]


class Grid(C.Structure):
    _fields_ = [("dim", C.c_int32), ("n", C.c_int32 * 3), ("h", C.c_double), ("nsub", C.c_int32 * 3),
                ("overlap", C.c_int32), ("zghost", C.c_int32), ("z_offset", C.c_int32), ("nz_global", C.c_int32),
                ("bc", C.c_int32), ("yghost", C.c_int32), ("y_offset", C.c_int32), ("ny_global", C.c_int32),
                ("pz", C.c_int32), ("py", C.c_int32), ("pad_", C.c_int32)]


class Params(C.Structure):
    _fields_ = [
        ("theta", C.c_double), ("gamma_c", C.c_double), ("gamma_eta", C.c_double), ("kappa", C.c_double),
        ("eps0", C.c_double), ("C11", C.c_double), ("C12", C.c_double), ("C44", C.c_double),
        ("Lscale", C.c_double), ("w_c", C.c_double),
        ("L0", C.c_double), ("L1", C.c_double), ("L2", C.c_double), ("L3", C.c_double),
        ("U1", C.c_double), ("U4", C.c_double), ("dE0", C.c_double), ("S", C.c_int32),
        ("newton_rtol", C.c_double), ("newton_atol", C.c_double), ("gmres_rtol", C.c_double),
        ("gmres_atol", C.c_double), ("newton_maxit", C.c_int32), ("gmres_restart", C.c_int32),
        ("gmres_maxit", C.c_int32), ("pc_type", C.c_int32), ("pc_reuse", C.c_int32),
        ("ls_alpha", C.c_double), ("ls_max_halvings", C.c_int32),
        ("zeta", C.c_double), ("dt_min", C.c_double), ("dt_max", C.c_double), ("dt_init", C.c_double),
        ("dt_floor_factor", C.c_double), ("xd_norm", C.c_int32), ("factor_fp32", C.c_int32),
        ("gmres_stall_cycles", C.c_int32), ("ilu_level", C.c_int32), ("u0_cg", C.c_int32),
        ("ras_cta_per_box", C.c_int32),
    ]


class HaloMsg(C.Structure):
    _fields_ = [("kind", C.c_int32), ("peer", C.c_int32), ("offset", C.c_int64), ("count", C.c_int64)]


class StepInfo(C.Structure):
    _fields_ = [
        ("converged", C.c_int32), ("reason", C.c_int32), ("newton_its", C.c_int32), ("gmres_its", C.c_int32),
        ("retries", C.c_int32), ("ls_halvings", C.c_int32), ("pc_setups", C.c_int32), ("pad_", C.c_int32),
        ("dt", C.c_double), ("time", C.c_double), ("energy", C.c_double), ("energy_parts", C.c_double * 4),
        ("mass", C.c_double), ("fnorm0", C.c_double), ("fnorm", C.c_double), ("zeta", C.c_double),
        ("xd", C.c_double),
    ]

    def to_dict(self):
        d = {k: getattr(self, k) for k, _ in self._fields_ if k != "pad_"}
        d["energy_parts"] = list(self.energy_parts)
        d["reason"] = REASONS.get(self.reason, str(self.reason))
        return d


_P = C.c_void_p
_D = C.POINTER(C.c_double)
# communication callbacks of a z-sharded state (nks.h: nks_allreduce_fn, nks_halo_fn)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p)
HALO_FN = C.CFUNCTYPE(C.c_int32, C.c_void_p, C.c_void_p, C.c_int32, C.c_int64, C.c_void_p)
_SIGS = {
    "nks_workspace_bytes": (C.c_size_t, [C.POINTER(Grid), C.POINTER(Params)]),
    "nks_create": (C.c_int, [C.POINTER(Grid), C.POINTER(Params), C.c_int32, C.c_int32, _P, _P, C.c_size_t, _P,
                             C.POINTER(_P)]),
    "nks_get_unique_id": (C.c_int, [_P]),
    "nks_decompose": (C.c_int, [C.POINTER(Grid), C.POINTER(Params), C.c_int32, C.c_int32, C.POINTER(Grid)]),
    "nks_halo_plan": (C.c_int32, [C.POINTER(Grid), C.c_int32, C.c_int32, C.c_int32, C.POINTER(HaloMsg), C.c_int32]),
    "nks_decompose_pencil": (C.c_int, [C.POINTER(Grid), C.POINTER(Params), C.c_int32, C.c_int32, C.c_int32, C.POINTER(Grid)]),
    "nks_set_fields": (C.c_int, [_P, _P, _P, _P, C.c_int32]),
    "nks_get_fields": (C.c_int, [_P, _P, _P, _P, C.c_int32]),
    "nks_set_state": (C.c_int, [_P, _P, _P, _P, C.c_int32]),
    "nks_set_cbar0": (C.c_int, [_P, C.c_double]),
    "nks_set_comm": (C.c_int, [_P, ALLREDUCE_FN, HALO_FN, _P]),
    "nks_step": (C.c_int, [_P, C.c_double, C.POINTER(StepInfo)]),
    "nks_run_adaptive": (C.c_int, [_P, C.c_int32, C.c_double, C.POINTER(StepInfo), C.POINTER(C.c_int32)]),
    "nks_energy": (C.c_int, [_P, _D, _D]),
    "nks_eval_residual": (C.c_int, [_P, C.c_double, _P, _P, C.c_int32]),
    "nks_eval_jv": (C.c_int, [_P, C.c_double, _P, _P, _P, C.c_int32]),
    "nks_pc_setup": (C.c_int, [_P, C.c_double, _P, C.c_int32]),
    "nks_pc_apply": (C.c_int, [_P, _P, _P, C.c_int32]),
    "nks_gmres_solve": (C.c_int, [_P, C.c_double, _P, _P, _P, C.c_int32, C.POINTER(C.c_int32)]),
    "nks_counters": (C.c_int, [_P, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    "nks_set_profiling": (C.c_int, [_P, C.c_int32]),
    "nks_phase_times": (C.c_int, [_P, _D, C.POINTER(C.c_int64), C.c_int32]),
    "nks_destroy": (C.c_int, [_P]),
    "nks_last_error": (C.c_char_p, [_P]),
    "nks_version": (C.c_char_p, []),
}

_lib = None


def load_library(path: str = LIB_PATH):
    """Load libnks.so and declare every ABI signature.  Raises if the library is missing."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise RuntimeError(f"libnks.so not built ({path}); run `python -m paper_2209_08001_b200.build`")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


class NKSError(RuntimeError):
    def __init__(self, status, msg):
        super().__init__(f"{STATUS.get(status, status)}: {msg}")
        self.status = status


def make_grid(shape, h=0.25, nsub=None, overlap=2, zghost=0, z_offset=0, nz_global=0, bc=0) -> Grid:
    """shape and nsub in C order: (ny, nx) or (nz, ny, nx)."""
    d = len(shape)
    g = Grid()
    g.dim = d
    n = list(reversed(shape)) + [1] * (3 - d)
    for j in range(3):
        g.n[j] = int(n[j])
    g.h = float(h)
    ns = list(reversed(nsub)) if nsub is not None else [1] * d     # nsub in C order like shape
    ns = ns + [1] * (3 - len(ns))
    for j in range(3):
        g.nsub[j] = int(ns[j])
    g.overlap = int(overlap)
    g.zghost = int(zghost)
    g.z_offset = int(z_offset)
    g.nz_global = int(nz_global)
    g.bc = int(bc)
    return g


def unique_id() -> bytes:
    """nks_get_unique_id: the 128-byte NCCL id rank 0 hands to every rank of a sharded run."""
    buf = C.create_string_buffer(128)
    rc = load_library().nks_get_unique_id(buf)
    if rc != NKS_OK:
        raise NKSError(rc, "nks_get_unique_id failed")
    return buf.raw


def halo_plan(local: Grid, rank: int, nranks: int, nfields: int):
    """nks_halo_plan: the ordered (kind, peer, offset, count) messages of the library's halo exchange (host only)."""
    lib = load_library()
    n = lib.nks_halo_plan(C.byref(local), int(rank), int(nranks), int(nfields), None, 0)
    if n < 0:
        raise NKSError(NKS_E_INVALID, "nks_halo_plan: invalid slab / pencil")
    buf = (HaloMsg * n)()
    lib.nks_halo_plan(C.byref(local), int(rank), int(nranks), int(nfields), buf, n)
    return [(m.kind, m.peer, m.offset, m.count) for m in buf]


def decompose_pencil(global_grid: Grid, params: Params, rank: int, pz: int, py: int) -> Grid:
    """nks_decompose_pencil: the z x y pencil grid of `rank` = rz * py + ry on a pz x py process grid (host only);
    with RAS each rank owns whole box layers along z and y."""
    out = Grid()
    rc = load_library().nks_decompose_pencil(C.byref(global_grid), C.byref(params), int(rank), int(pz), int(py),
                                             C.byref(out))
    if rc != NKS_OK:
        raise NKSError(rc, "nks_decompose_pencil: no valid pencil for this grid / process grid")
    return out


def decompose(global_grid: Grid, params: Params, rank: int, nranks: int) -> Grid:
    """nks_decompose: the z-slab grid of `rank` (host only)."""
    out = Grid()
    rc = load_library().nks_decompose(C.byref(global_grid), C.byref(params), int(rank), int(nranks), C.byref(out))
    if rc != NKS_OK:
        raise NKSError(rc, "nks_decompose: no valid slab for this grid / rank count")
    return out


def make_params(model: dict, solver: dict, pc_type=PC_RAS_BILU0, pc_reuse=1) -> Params:
    p = Params()
    for k in ["theta", "gamma_c", "gamma_eta", "kappa", "eps0", "C11", "C12", "C44", "Lscale", "w_c",
              "L0", "L1", "L2", "L3", "U1", "U4", "dE0"]:
        setattr(p, k, float(model[k]))
    p.S = int(model["S"])
    for k in ["newton_rtol", "newton_atol", "gmres_rtol", "gmres_atol", "ls_alpha", "zeta", "dt_min",
              "dt_max", "dt_init", "dt_floor_factor"]:
        setattr(p, k, float(solver[k]))
    for k in ["newton_maxit", "gmres_restart", "gmres_maxit"]:
        setattr(p, k, int(solver[k]))
    p.ls_max_halvings = int(solver["ls_max_halvings"])
    p.pc_type = int(pc_type)
    p.pc_reuse = int(pc_reuse)
    p.xd_norm = {"rms": 0, "l2": 1, "ceta_l2": 2}[solver.get("xd_norm", "rms")]
    p.factor_fp32 = int(solver.get("factor_fp32", 0))
    p.gmres_stall_cycles = int(solver.get("gmres_stall_cycles", 0))
    p.ilu_level = int(solver.get("ilu_level", 0))
    p.u0_cg = int(solver.get("u0_cg", 0))
    p.ras_cta_per_box = int(solver.get("ras_cta_per_box", 0))
    return p


class Solver:
    """One NKS state on the current CUDA device (single GPU)."""

    def __init__(self, shape, model: dict, solver: dict, h=0.25, nsub=None, overlap=2,
                 pc_type=PC_RAS_BILU0, pc_reuse=1, device=None, zghost=0, grid: Grid = None, rank=0, nranks=1,
                 nccl_id: bytes = None, bc=0):
        """shape: the (local) grid in C order; `grid` overrides the grid built from shape/nsub/overlap/zghost
        (a slab from `decompose`).  nccl_id (slab states): the library creates its own NCCL communicator."""
        import torch
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2209_08001_b200 needs a CUDA device (B200, sm_100a)")
        self.torch = torch
        self.lib = load_library()
        self.shape = tuple(shape)
        self.d = len(shape)
        self.nf = 2 + self.d
        self.N = int(np.prod(shape))
        self.device = torch.device(device) if device is not None else torch.device("cuda", torch.cuda.current_device())
        self.grid = grid if grid is not None else make_grid(shape, h, nsub, overlap, zghost, bc=bc)
        self.rank, self.nranks = int(rank), int(nranks)
        self._nccl_id = C.create_string_buffer(bytes(nccl_id), 128) if nccl_id is not None else None
        self.params = make_params(model, solver, pc_type, pc_reuse)
        nbytes = self.lib.nks_workspace_bytes(C.byref(self.grid), C.byref(self.params))
        if nbytes == 0:
            raise NKSError(NKS_E_INVALID, "invalid grid/params")
        with torch.cuda.device(self.device):
            self.workspace = torch.empty(int(nbytes), dtype=torch.uint8, device=self.device)
            self.stream = torch.cuda.current_stream(self.device)
            st = C.c_void_p()
            rc = self.lib.nks_create(C.byref(self.grid), C.byref(self.params), self.rank, self.nranks, self._nccl_id,
                                     C.c_void_p(self.workspace.data_ptr()), C.c_size_t(nbytes),
                                     C.c_void_p(self.stream.cuda_stream), C.byref(st))
        if rc != NKS_OK:
            raise NKSError(rc, "nks_create failed")
        self.st = st
        self.workspace_bytes = nbytes

    # ---------------------------------------------------------------- helpers
    def _check(self, rc, what):
        if rc != NKS_OK:
            extra = f" ({self.comm_error!r})" if getattr(self, "comm_error", None) is not None else ""
            raise NKSError(rc, f"{what}: {self.lib.nks_last_error(self.st).decode()}{extra}")

    def _dev(self, a, n):
        """Device fp64 contiguous tensor for an array-like (numpy or torch)."""
        t = self.torch
        if isinstance(a, t.Tensor):
            x = a.to(device=self.device, dtype=t.float64).contiguous()
        else:
            x = t.from_numpy(np.ascontiguousarray(a, dtype=np.float64)).to(self.device)
        if x.numel() != n:
            raise ValueError(f"expected {n} values, got {x.numel()}")
        return x

    def __del__(self):
        try:
            if getattr(self, "st", None):
                self.lib.nks_destroy(self.st)
                self.st = None
        except Exception:
            pass

    # ---------------------------------------------------------------- API
    def set_fields(self, c, eta, u=None):
        tc, te = self._dev(c, self.N), self._dev(eta, self.N)
        tu = self._dev(u, self.d * self.N) if u is not None else None
        rc = self.lib.nks_set_fields(self.st, C.c_void_p(tc.data_ptr()), C.c_void_p(te.data_ptr()),
                                     C.c_void_p(tu.data_ptr()) if tu is not None else None, 1)
        self._check(rc, "nks_set_fields")

    def set_fields_host(self, c, eta, u=None):
        """Same as set_fields from host (numpy) memory through the ABI's on_device = 0 path."""
        c = np.ascontiguousarray(c, dtype=np.float64)
        eta = np.ascontiguousarray(eta, dtype=np.float64)
        uu = np.ascontiguousarray(u, dtype=np.float64) if u is not None else None
        rc = self.lib.nks_set_fields(self.st, c.ctypes.data_as(C.c_void_p), eta.ctypes.data_as(C.c_void_p),
                                     uu.ctypes.data_as(C.c_void_p) if uu is not None else None, 0)
        self._check(rc, "nks_set_fields")

    def set_state(self, c, eta, u):
        """Replace X^n without restarting the run (nks_set_state): controller history, time, zeta kept."""
        tc, te, tu = self._dev(c, self.N), self._dev(eta, self.N), self._dev(u, self.d * self.N)
        rc = self.lib.nks_set_state(self.st, C.c_void_p(tc.data_ptr()), C.c_void_p(te.data_ptr()),
                                    C.c_void_p(tu.data_ptr()), 1)
        self._check(rc, "nks_set_state")

    def set_comm(self, allreduce, halo):
        """Attach host communication callbacks to this z-slab state (nks_set_comm; the callback backend of a
        state created without an NCCL id).  allreduce(ptr, n, stream) and halo(ptr, nfields, field_stride,
        stream) are Python callables on raw device pointers that return 0 on success; the ctypes
        trampolines are kept alive by this object."""
        def _ar(user, buf, n, stream):
            try:
                return int(allreduce(buf, n, stream) or 0)
            except Exception as e:          # never let an exception unwind through C
                self.comm_error = e
                return 1

        def _halo(user, vec, nf, stride, stream):
            try:
                return int(halo(vec, nf, stride, stream) or 0)
            except Exception as e:
                self.comm_error = e
                return 1
        self._comm_cbs = (ALLREDUCE_FN(_ar), HALO_FN(_halo))
        self.comm_error = None
        self._check(self.lib.nks_set_comm(self.st, self._comm_cbs[0], self._comm_cbs[1], None), "nks_set_comm")

    def device_view(self, ptr, n):
        """fp64 tensor aliasing n doubles at device pointer ptr inside this state's workspace."""
        base = self.workspace.data_ptr()
        off = int(ptr) - base
        if off < 0 or off % 8 or off + 8 * int(n) > self.workspace_bytes:
            raise ValueError("pointer outside the workspace")
        return self.workspace[off:off + 8 * int(n)].view(self.torch.float64)

    def set_cbar0(self, cbar0):
        self._check(self.lib.nks_set_cbar0(self.st, C.c_double(cbar0)), "nks_set_cbar0")

    def get_state(self):
        """X^n as a (2+d, *shape) float64 numpy array."""
        out = np.empty((self.nf,) + self.shape)
        rc = self.lib.nks_get_fields(self.st, out[0].ctypes.data_as(C.c_void_p), out[1].ctypes.data_as(C.c_void_p),
                                     out[2:].ctypes.data_as(C.c_void_p), 0)
        self._check(rc, "nks_get_fields")
        return out

    def get_state_device(self):
        t = self.torch
        out = t.empty((self.nf,) + self.shape, dtype=t.float64, device=self.device)
        rc = self.lib.nks_get_fields(self.st, C.c_void_p(out[0].data_ptr()), C.c_void_p(out[1].data_ptr()),
                                     C.c_void_p(out[2].data_ptr()), 1)
        self._check(rc, "nks_get_fields")
        return out

    def step(self, dt, raise_on_fail=True):
        info = StepInfo()
        rc = self.lib.nks_step(self.st, C.c_double(dt), C.byref(info))
        if rc != NKS_OK and raise_on_fail:
            self._check(rc, "nks_step")
        d = info.to_dict()
        d["status"] = STATUS.get(rc, rc)
        return d

    def run_adaptive(self, max_steps, t_end=0.0):
        recs = (StepInfo * max(1, max_steps))()
        done = C.c_int32(0)
        rc = self.lib.nks_run_adaptive(self.st, int(max_steps), C.c_double(t_end), recs, C.byref(done))
        self._check(rc, "nks_run_adaptive")
        return [recs[k].to_dict() for k in range(done.value)]

    def energy(self):
        parts = (C.c_double * 4)()
        mass = C.c_double()
        self._check(self.lib.nks_energy(self.st, parts, C.byref(mass)), "nks_energy")
        return list(parts), mass.value

    def eval_residual(self, x_b, dt):
        xb = self._dev(x_b, self.nf * self.N)
        F = self.torch.empty_like(xb)
        self._check(self.lib.nks_eval_residual(self.st, C.c_double(dt), C.c_void_p(xb.data_ptr()),
                                               C.c_void_p(F.data_ptr()), 1), "nks_eval_residual")
        return F.reshape((self.nf,) + self.shape)

    def eval_jv(self, x_b, v, dt):
        xb = self._dev(x_b, self.nf * self.N)
        vv = self._dev(v, self.nf * self.N)
        out = self.torch.empty_like(xb)
        self._check(self.lib.nks_eval_jv(self.st, C.c_double(dt), C.c_void_p(xb.data_ptr()),
                                         C.c_void_p(vv.data_ptr()), C.c_void_p(out.data_ptr()), 1), "nks_eval_jv")
        return out.reshape((self.nf,) + self.shape)

    def pc_setup(self, x_b, dt):
        xb = self._dev(x_b, self.nf * self.N)
        self._check(self.lib.nks_pc_setup(self.st, C.c_double(dt), C.c_void_p(xb.data_ptr()), 1), "nks_pc_setup")

    def pc_apply(self, r):
        rr = self._dev(r, self.nf * self.N)
        z = self.torch.empty_like(rr)
        self._check(self.lib.nks_pc_apply(self.st, C.c_void_p(rr.data_ptr()), C.c_void_p(z.data_ptr()), 1),
                    "nks_pc_apply")
        return z.reshape((self.nf,) + self.shape)

    def gmres_solve(self, x_b, rhs, dt):
        xb = self._dev(x_b, self.nf * self.N)
        b = self._dev(rhs, self.nf * self.N)
        s = self.torch.empty_like(b)
        its = C.c_int32(0)
        rc = self.lib.nks_gmres_solve(self.st, C.c_double(dt), C.c_void_p(xb.data_ptr()), C.c_void_p(b.data_ptr()),
                                      C.c_void_p(s.data_ptr()), 1, C.byref(its))
        self._check(rc, "nks_gmres_solve")
        return s.reshape((self.nf,) + self.shape), its.value

    def counters(self):
        a, b, r = C.c_int64(), C.c_int64(), C.c_int64()
        self._check(self.lib.nks_counters(self.st, C.byref(a), C.byref(b), C.byref(r)), "nks_counters")
        return {"kernel_launches": a.value, "host_syncs": b.value, "reductions": r.value}

    def set_profiling(self, on=True):
        self._check(self.lib.nks_set_profiling(self.st, 1 if on else 0), "nks_set_profiling")

    def phase_times(self, reset=False):
        ms = (C.c_double * 8)()
        cnt = (C.c_int64 * 8)()
        self._check(self.lib.nks_phase_times(self.st, ms, cnt, 1 if reset else 0), "nks_phase_times")
        return {PHASES[k]: {"ms": ms[k], "count": cnt[k]} for k in range(8)}


def version():
    return load_library().nks_version().decode()
