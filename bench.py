#!/usr/bin/env python
"""Benchmark of the B200 NKS time step (arXiv 2209.08001) -- the driver's bench contract.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl nks|reference] [--config 2]

One "step" = one accepted adaptive NKS time step (Eq. NSOA-1 solved by Newton-Krylov-Schwarz,
P:474-488) of BASELINE.json configs[1] = config 2: 2D 512x512 periodic, fp64,
adaptive dt, RAS 4x4 boxes delta = 2 with point-block ILU(0), GMRES(30).  Steps
are consecutive steps of one trajectory (W untimed warm-up steps first, then K timed steps).

value  = NKS time steps per second of the whole job (the inverse of BASELINE's "NKS time-step
         wall time"; ms_per_step is that wall time), inputs resident in HBM;
e2e    = the same through the C ABI with HOST buffers: every step uploads X^n from pinned host
         memory (nks_set_fields, on_device = 0), runs nks_step with the dt the device run
         accepted and downloads X^{n+1} (nks_get_fields) -- copies inside the timed region;
roofline = the dominant kernel of the step (per-phase CUDA events recorded by the library on
         its own stream in a profiled pass of 2 steps right after the unprofiled timed region),
         algorithmic bytes per launch / mean duration, against MEASURED_PEAKS.json hbm_gbs;
cpu_baseline = the oracle (oracle/, plain NumPy/SciPy) as it stands, timed on one step of the same
         trajectory on the full grid (and compared with the GPU's result of that step).

N > 1: config 2 (2D) runs independent replicas per rank (the 2D sweep is not sharded; DESIGN.md
"Multi-GPU"), scaling "weak", value = all ranks' steps / max-over-ranks time.  3D configs
(--config 3/4) run the z-slab SHARDED step at N > 1 (or with --sharded at N = 1): every rank owns
whole RAS boxes of the global box grid, the library calls back for NCCL halo exchanges and
fixed-order allreduces (paper_2209_08001_b200/shard.py), value = steps/s of the one global run.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import nks_inputs as ni  # noqa: E402

# fp64 thread-level operations per grid point (DFMA + DADD + DMUL), counted by ncu at 3D 256^3
# (profiles/r01_ncu_F_Jv_fp64_ops_3d256.txt): F is bound by the fp64 pipe, J.v by HBM
FP64_OPS_PER_POINT = {"residual": 515.7, "jv": 138.5}
# measured fp64 peak: 36.77 TFLOP/s DFMA = 18.4e12 fp64 pipe operations/s (profiles/r01_fp64_peak_probe.txt,
# tools/lat_probe.cu); nominal 148 SMs x 64 lanes x 1.965 GHz = 18.6e12
FP64_OPS_PEAK = 36.77e12 / 2
METRIC = "NKS time steps/s (inverse NKS time-step wall time; BASELINE: NKS time-step wall time and F/J.v GDOF/s)"
UNIT = "steps/s"


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="nks", choices=["nks", "reference"])
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-micro", action="store_true")
    ap.add_argument("--no-variants", action="store_true")
    ap.add_argument("--no-extra", action="store_true")
    ap.add_argument("--scaling", default="strong", choices=["strong", "weak"],
                    help="3D sharded runs: strong (a fixed grid split over N ranks) or weak (128^3 per rank)")
    ap.add_argument("--decomp", default="slab", choices=["slab", "pencil"],
                    help="sharded 3D runs: z-slabs (default) or z x y pencils on the most square pz x py grid")
    ap.add_argument("--sharded", action="store_true",
                    help="3D configs: run the z-slab sharded NKS step (ShardedSolver, NCCL halos/allreduces); "
                         "implied for 3D configs at N > 1")
    return ap.parse_args()


# ------------------------------------------------------------------------------------------- dist
def dist_setup(ngpus):
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    pg = None
    if world > 1:
        import torch
        import torch.distributed as dist
        backend = "nccl" if torch.cuda.is_available() else "gloo"
        if torch.cuda.is_available():
            torch.cuda.set_device(local)
        dist.init_process_group(backend=backend)
        pg = dist
    return world, rank, local, pg


def barrier(pg):
    if pg is not None:
        pg.barrier()


def max_over_ranks(pg, x):
    if pg is None:
        return x
    import torch
    dev = "cuda" if torch.cuda.is_available() else "cpu"
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    pg.all_reduce(t, op=pg.ReduceOp.MAX)
    return float(t.item())


# ------------------------------------------------------------------------------------------- clocks
class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms during the timed region."""
    Q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, index=0):
        self.index = index
        self.rows = []
        self.proc = None
        self.th = None

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.Q}", "--format=csv,noheader,nounits",
                 "-lms", "200"], stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
            return
        self.th = threading.Thread(target=self._read, daemon=True)
        self.th.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 7:
                self.rows.append(parts)

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        time.sleep(0.25)
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        if self.th:
            self.th.join(timeout=2)
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        smax = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[k] for r in self.rows for k in range(4) if r[3 + k].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(smax) if smax else None,
                "reasons": reasons, "samples": len(self.rows)}


# ------------------------------------------------------------------------------------------- oracle
def oracle_model_sol(cfg, sol):
    from oracle import scheme
    return scheme.Model.from_dict(len(cfg["shape"]), cfg["h"], ni.model_default()), dict(sol)


def oracle_threads():
    """Host threads the oracle can use: NumPy elementwise work runs on one core, scipy.fft (the
    spectral preconditioner) on os.cpu_count() workers."""
    return os.cpu_count() or 1


def oracle_step_sample(cfg, sol, Xn, cbar0, dt):
    """One oracle NKS step (oracle/, plain NumPy/SciPy as it stands) of the FULL config grid: Newton
     with the oracle's large-grid Krylov path (matrix-free J v + spectral-preconditioned
    GMRES(30), oracle/krylov.py) from X^n with the given dt.  Returns (X^{n+1}, info, seconds)."""
    from oracle import krylov, solver
    m, sol = oracle_model_sol(cfg, sol)
    t0 = time.perf_counter()
    X, info = solver.newton_step(m, Xn, dt, cbar0, sol, linsolve=krylov.make_linsolve())
    return X, info, time.perf_counter() - t0


def run_reference(args, world, rank, pg):
    """--impl reference: the oracle (the CPU definition of the method, oracle/) running config 2's own
    adaptive trajectory from the seeded initial state -- its own controller (Eq. sencondt),
    exact Newton through its Krylov path.  Warm-up and timed steps are real full-grid steps; because
    one oracle step takes ~10-25 s, at most 1 warm-up step and as many timed steps as fit in a
    ~150 s budget are run (`steps` is the number actually timed; `steps_requested` = K)."""
    if rank != 0:
        return
    from oracle import krylov, solver
    cfg = ni.CONFIGS[args.config]
    sol = bench_solver(cfg)
    m, sol = oracle_model_sol(cfg, sol)
    shape = cfg["shape"]
    c, eta = ni.initial_fields(shape, 0)
    cbar = c.mean()
    X = solver.gauge_project(np.concatenate([c[None], eta[None], solver.init_displacement_fft(m, c, cbar)]))
    lin = krylov.make_linsolve()
    Xprev, dt_prev, zeta = None, None, sol["zeta"]
    per, recs = [], []
    budget = float(os.environ.get("NKS_REFERENCE_BUDGET_S", "150"))
    t_start = time.perf_counter()
    n = 0
    while n < min(args.warmup, 1) + args.steps:
        dt = sol["dt_init"] if Xprev is None else solver.predict_dt(
            solver.change_rate(X, Xprev, dt_prev, sol["xd_norm"]), zeta, sol["dt_min"], sol["dt_max"])
        t0 = time.perf_counter()
        while True:
            Xb, info = solver.newton_step(m, X, dt, cbar, sol, linsolve=lin)
            if info["converged"]:
                break
            dt /= np.sqrt(2)
            zeta *= 2
        el = time.perf_counter() - t0
        if n >= min(args.warmup, 1):
            per.append(el)
            recs.append({"dt": dt, "newton_its": info["newton_its"]})
        Xprev, X, dt_prev = X, Xb, dt
        n += 1
        if time.perf_counter() - t_start > budget and per:
            break
    mean_s = float(np.mean(per))
    sample = (f"{len(per)} timed oracle steps (after {min(args.warmup, 1)} warm-up) of config 2's own adaptive "
              f"trajectory on the full {'x'.join(map(str, shape))} grid, seed 0: exact Newton via oracle/krylov.py "
              f"(matrix-free J.v, spectral-preconditioned GMRES(30)); dt {[round(r['dt'], 4) for r in recs]}")
    line = {"impl": "reference", "metric": METRIC, "value": 1.0 / mean_s, "unit": UNIT, "n_gpus": args.gpus,
            "steps": len(per), "steps_requested": args.steps, "warmup": min(args.warmup, 1),
            "ms_per_step": mean_s * 1e3, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": "f64", "data": "synthetic", "config": config_dict(cfg, args.gpus),
            "cpu_baseline": {"value": 1.0 / mean_s, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
                             "sample": sample},
            "e2e": {"value": 1.0 / mean_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "per_step_s": per}
    print(json.dumps(line), flush=True)


def bench_solver(cfg):
    """Solver settings of the benchmark: SURVEY 8(c).2 defaults + the opt-in GMRES stagnation rule
    (gmres_stall_cycles = 3, R18) so that a BILU(0)-RAS solve that stalls is retried by the
    controller instead of running to gmres_maxit = 10,000."""
    sol = dict(ni.solver_default())
    sol["gmres_stall_cycles"] = 3
    return sol


def config_dict(cfg, ngpus, sharded=False, decomp="slab"):
    d = len(cfg["shape"])
    return {"workload": f"config {2 if cfg['name'] == '2d_512' else cfg['name']}: {cfg['name']} "
                        f"{'x'.join(map(str, cfg['shape']))} periodic, adaptive dt (P:596-607), "
                        f"RAS {'x'.join(map(str, cfg['nsub']))} boxes delta={cfg['overlap']} BILU(0), GMRES(30)",
            "grid": list(cfg["shape"]), "dof": (2 + d) * int(np.prod(cfg["shape"])),
            "nsub": list(cfg["nsub"]), "overlap": cfg["overlap"], "newton_rtol": 1e-11, "gmres_rtol": 1e-10,
            "init": "c=0.1622+U(-0.005,0.005), eta=0.1+U(-0.01,0.01), seed 0, " +
                    ("u0 = conjugate gradients on the elastic block (sharded)" if sharded else "u0=FFT equilibrium"),
            "parallelism": ((f"z x y pencils {'x'.join(map(str, pencil_grid(ngpus)))} (sharded NKS step, NCCL halo "
                             f"exchange + allreduce)" if decomp == "pencil" else
                             f"z-slabs x {ngpus} (sharded NKS step, NCCL halo exchange + allreduce)") if sharded
                            else ("replicas" if ngpus > 1 else "1 GPU")),
            "l2": l2_note(cfg)}


def l2_note(cfg):
    """Working set of the timed step against the 126 MB L2: the BILU factors over the overlapped boxes
    (13 / 25 point blocks of nf x nf doubles per box position) and the GMRES(30) basis."""
    d = len(cfg["shape"])
    nf = 2 + d
    ext = [n // s + 2 * cfg["overlap"] for n, s in zip(cfg["shape"], cfg["nsub"])]
    P = int(np.prod(ext)) * int(np.prod(cfg["nsub"]))
    fac = 8 * (13 if d == 2 else 25) * nf * nf * P
    basis = 8 * 31 * nf * int(np.prod(cfg["shape"]))
    return (f"working set > 126 MB L2 (BILU factors ~{fac / 1e9:.2f} GB + Krylov basis ~{basis / 1e9:.2f} GB); "
            "no flush")


# ------------------------------------------------------------------------------------------- GPU arm
def ras_bytes(solver_obj, cfg):
    """Algorithmic bytes of one RAS apply: every stored factor entry once, r gathered over the
    overlapped boxes, z written on owned points."""
    d = len(cfg["shape"])
    nf = 2 + d
    N = int(np.prod(cfg["shape"]))
    nslots = 13 if d == 2 else 25
    ext = [n // s + 2 * cfg["overlap"] for n, s in zip(cfg["shape"], cfg["nsub"])]
    P = int(np.prod(ext)) * int(np.prod(cfg["nsub"]))
    return 8 * (nslots * nf * nf * P + nf * P + nf * N), P


def micro_kernels(shape, reps=10):
    """F (K1) and J.v (K2) alone on one grid (SURVEY 8(d) config 5 recipe): X^n = common init (u = 0),
    X^b = X^n + U(-1e-3, 1e-3) on c and eta, v ~ U(-1, 1), dt = 0.01; library CUDA events around each
    launch (nks_phase_times), mean over `reps` launches after warm-up.  Algorithmic bytes per point:
    F = 8 (2 nf + 3) (X^b, c^a, eta^a, T^n in; F out); J.v = 8 (2 nf + 5) (v, 4 partials, c^a in; out)."""
    import torch
    from paper_2209_08001_b200 import PC_NONE, Solver
    d = len(shape)
    nf = 2 + d
    N = int(np.prod(shape))
    sol = dict(ni.solver_default())
    sol["gmres_restart"] = 1                      # no Krylov basis needed here
    g = Solver(shape, ni.model_default(), sol, pc_type=PC_NONE)
    gen = torch.Generator(device="cuda").manual_seed(0)
    c = 0.1622 + (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.01
    eta = 0.1 + (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.02
    u = torch.zeros((d,) + tuple(shape), device="cuda", dtype=torch.float64)
    g.set_fields(c, eta, u)
    xb = torch.cat([c[None], eta[None], u]).contiguous()
    xb[0] += (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2e-3
    xb[1] += (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2e-3
    v = (torch.rand((nf,) + tuple(shape), device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2
    del c, eta, u
    for _ in range(2):
        g.eval_residual(xb, 0.01)
        g.eval_jv(xb, v, 0.01)
    torch.cuda.synchronize()
    g.set_profiling(True)
    g.phase_times(reset=True)
    for _ in range(reps):
        g.eval_residual(xb, 0.01)
        g.eval_jv(xb, v, 0.01)
    ph = g.phase_times(reset=True)
    out = {}
    for key, per_pt in (("residual", 2 * nf + 3), ("jv", 2 * nf + 5)):
        ms = ph[key]["ms"] / ph[key]["count"]
        out[key] = {"ms": ms, "GDOF_s": nf * N / (ms * 1e-3) / 1e9, "alg_bytes": per_pt * 8 * N,
                    "GB_s": per_pt * 8 * N / (ms * 1e-3) / 1e9}
    del g, xb, v
    torch.cuda.empty_cache()
    return out


def micro_sharded(shape, pg, reps=10):
    """Config 5: F and J.v of a z-sharded 3D grid (each rank one slab, 2 ghost planes per side), the
    NCCL halo exchange of every input included in the timed operator; time = max over ranks."""
    import torch
    from paper_2209_08001_b200.shard import SlabOperators
    ops = SlabOperators(shape, ni.model_default(), ni.solver_default())
    d = 3
    nf = 2 + d
    ls = ops.local_shape
    gen = torch.Generator(device="cuda").manual_seed(1234 + ops.lo)
    Xa = torch.empty((nf,) + ls, device="cuda", dtype=torch.float64)
    Xa[0] = 0.1622 + (torch.rand(ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.01
    Xa[1] = 0.1 + (torch.rand(ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.02
    Xa[2:] = 0.0
    ops.set_level_n(Xa, 0.1622)
    Xb = Xa.clone()
    Xb[:2] += (torch.rand((2,) + ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2e-3
    v = (torch.rand((nf,) + ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2
    del Xa
    for _ in range(2):
        ops.residual(Xb, 0.01)
        ops.jv(Xb, v, 0.01)
    res = {}
    for key in ("residual", "jv"):
        barrier(pg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            if key == "residual":
                ops.residual(Xb, 0.01)
            else:
                ops.jv(Xb, v, 0.01)
        e1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(pg, e0.elapsed_time(e1) / reps)
        Ng = int(np.prod(shape))
        res[key] = {"ms_incl_halo_exchange": ms, "GDOF_s": nf * Ng / (ms * 1e-3) / 1e9}
    del ops, Xb, v
    torch.cuda.empty_cache()
    return res


def micro_pencil(shape, pg, world, reps=10):
    """Config 5 on z x y pencils (a pz x py process grid, the most square factorisation of the rank count):
    F and J.v through the library's pencil state (nks_decompose_pencil; nks_eval_residual / nks_eval_jv fill
    the ghost planes AND rows with the library's NCCL exchange: packed y blocks, then planes), the exchange
    of every input included in the timed operator; time = max over ranks."""
    import torch
    import torch.distributed as dist
    from paper_2209_08001_b200.shard import PencilSolver
    pz = max(p for p in range(1, int(world ** 0.5) + 1) if world % p == 0)
    py = world // pz
    ps = PencilSolver(shape, ni.model_default(), ni.solver_default(), pz, py,
                      group=None if not dist.is_initialized() else dist.group.WORLD, comm="nccl")
    nf, ls = 5, ps.local_shape
    gen = torch.Generator(device="cuda").manual_seed(4321 + ps.rank)
    c = 0.1622 + (torch.rand(ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.01
    eta = 0.1 + (torch.rand(ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.02
    u = torch.zeros((3,) + ls, device="cuda", dtype=torch.float64)
    ps.solver.set_fields(c, eta, u)
    Xb = torch.cat([c[None], eta[None], u])
    Xb[:2] += (torch.rand((2,) + ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2e-3
    v = (torch.rand((nf,) + ls, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2
    del c, eta, u
    for _ in range(2):
        ps.solver.eval_residual(Xb, 0.01)
        ps.solver.eval_jv(Xb, v, 0.01)
    res = {"process_grid_pz_py": [pz, py]}
    for key in ("residual", "jv"):
        barrier(pg)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            if key == "residual":
                ps.solver.eval_residual(Xb, 0.01)
            else:
                ps.solver.eval_jv(Xb, v, 0.01)
        e1.record()
        torch.cuda.synchronize()
        ms = max_over_ranks(pg, e0.elapsed_time(e1) / reps)
        Ng = int(np.prod(shape))
        res[key] = {"ms_incl_halo_exchange_and_d2d_copies": ms, "GDOF_s": nf * Ng / (ms * 1e-3) / 1e9}
    del ps, Xb, v
    torch.cuda.empty_cache()
    return res


def step_stats(per_ms):
    a = np.asarray(per_ms)
    return {"mean": float(a.mean()), "p50": float(np.percentile(a, 50)), "p90": float(np.percentile(a, 90)),
            "min": float(a.min()), "max": float(a.max())}


def run_variant(args, cfg, model, sol, c, eta, pg, pc_type):
    """W warm-up + K timed adaptive steps of config 2's workload with another preconditioner."""
    import torch
    from paper_2209_08001_b200 import Solver
    g = Solver(cfg["shape"], model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_type=pc_type,
               pc_reuse=1)
    g.set_fields(c, eta, None)
    for _ in range(args.warmup):
        g.run_adaptive(1)
    torch.cuda.synchronize()
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier(pg)
    torch.cuda.synchronize()
    evs[0].record(g.stream)
    recs = []
    for k in range(args.steps):
        recs += g.run_adaptive(1)
        evs[k + 1].record(g.stream)
    torch.cuda.synchronize()
    t_ms = max_over_ranks(pg, evs[0].elapsed_time(evs[-1]))
    per = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    out = {"pc": {5: "spectral (cuFFT, mean-coefficient inverse per wave number)",
                  2: "left-RAS, point-block ILU(0)",
                  6: "two-level: spectral global correction + left-RAS 4x4 boxes delta=2 BILU(0)"}.get(pc_type, pc_type),
           "value": args.steps / (t_ms / 1e3), "unit": UNIT, "ms_per_step": t_ms / args.steps, "step_ms": step_stats(per),
           "newton_its": [r["newton_its"] for r in recs], "gmres_its": [r["gmres_its"] for r in recs],
           "dt": [r["dt"] for r in recs], "retries": [r["retries"] for r in recs],
           "time_simulated": recs[-1]["time"] if recs else None,
           "note": "same grid, model, controller and tolerances as the headline; its own adaptive trajectory"}
    del g
    torch.cuda.empty_cache()
    return out


def pencil_grid(world):
    """The most square pz x py factorisation of the rank count (pz <= py)."""
    pz = max(p for p in range(1, int(world ** 0.5) + 1) if world % p == 0)
    return pz, world // pz


def run_sharded_point(args, cfg, model, sol, pg, steps, warmup, decomp="slab"):
    """Config 3 through the sharded path (library decomposition into z-slabs -- ShardedSolver -- or z x y
    pencils -- PencilSolver --, library-owned NCCL communicator) with the ranks of pg (one rank here): W + K
    adaptive steps, max-over-ranks time."""
    import torch
    from paper_2209_08001_b200 import PC_RAS_BILU0
    from paper_2209_08001_b200.shard import PencilSolver, ShardedSolver
    c, eta = ni.initial_fields(cfg["shape"], 0)
    if decomp == "pencil":
        import torch.distributed as dist
        pz, py = pencil_grid(dist.get_world_size() if dist.is_initialized() else 1)
        sh = PencilSolver(cfg["shape"], model, sol, pz, py, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"],
                          pc_type=PC_RAS_BILU0, pc_reuse=1, comm="nccl")
        sh.run_adaptive = sh.solver.run_adaptive
    else:
        sh = ShardedSolver(cfg["shape"], model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
    sh.set_fields(c, eta)
    for _ in range(warmup):
        sh.run_adaptive(1)
    torch.cuda.synchronize()
    st = sh.solver.stream
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(pg)
    e0.record(st)
    recs = []
    for _ in range(steps):
        recs += sh.run_adaptive(1)
    e1.record(st)
    torch.cuda.synchronize()
    t = max_over_ranks(pg, e0.elapsed_time(e1))
    out = {"grid": list(cfg["shape"]), "nsub": list(cfg["nsub"]), "ranks": sh.world, "comm": sh.comm,
           "value": steps / (t / 1e3), "unit": UNIT, "ms_per_step": t / steps, "warmup": warmup, "steps": steps,
           "newton_its": [r["newton_its"] for r in recs], "gmres_its": [r["gmres_its"] for r in recs],
           "dt": [r["dt"] for r in recs], "retries": [r["retries"] for r in recs]}
    del sh
    return out


def run_gpu(args, world, rank, local, pg):
    import torch
    from paper_2209_08001_b200 import PC_SPECTRAL, Solver
    from paper_2209_08001_b200.build import build
    build()
    torch.cuda.set_device(local)
    # N > 1: the sharded 3D step (strong scaling) on config 3 (128^3) as the stated proxy of config 4 --
    # the 2D sweep of config 2 is not sharded, and config 4's one-level RAS/BILU(0) step takes ~15 min on
    # one GPU.  N = 1 also reports config 3 through the same sharded code path (one rank, library-owned
    # NCCL communicator) in configs_3d_one_gpu.config3_sharded_1rank -- the N = 1 point of that curve.
    cid = 3 if (world > 1 and args.config == 2) else args.config
    cfg = dict(ni.CONFIGS[cid])
    if args.scaling == "weak" and len(cfg["shape"]) == 3:
        # weak scaling (128^3 per GPU): the per-rank block stacked along z, with its
        # box layers, so every rank owns one 128^3 block of 8x8x8 boxes whatever N
        b = ni.CONFIGS[3]
        cfg["shape"] = (b["shape"][0] * world,) + tuple(b["shape"][1:])
        cfg["nsub"] = (b["nsub"][0] * world,) + tuple(b["nsub"][1:])
        cfg["name"] = f"3d_128_weak_x{world}"
    shape = cfg["shape"]
    d = len(shape)
    nf = 2 + d
    N = int(np.prod(shape))
    model, sol = ni.model_default(), bench_solver(cfg)
    sharded = d == 3 and (world > 1 or args.sharded)
    c, eta = ni.initial_fields(shape, 0)
    if sharded:
        # one z-slab (or z x y pencil, --decomp pencil) per rank; the library exchanges halos and reduces
        from paper_2209_08001_b200 import PC_RAS_BILU0
        from paper_2209_08001_b200.shard import PencilSolver, ShardedSolver
        if args.decomp == "pencil":
            pz, py = pencil_grid(world)
            sh = PencilSolver(shape, model, sol, pz, py, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"],
                              pc_type=PC_RAS_BILU0, pc_reuse=1)
        else:
            sh = ShardedSolver(shape, model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
        sh.set_fields(c, eta)
        g = sh.solver
    else:
        sh = None
        g = Solver(shape, model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
        g.set_fields(c, eta, None)
    for _ in range(args.warmup):
        g.run_adaptive(1)
    torch.cuda.synchronize()
    X_warm = g.get_state() if (rank == 0 and world == 1 and not args.no_cpu) else None

    # ---- timed region: K accepted adaptive steps, library profiling OFF, one event pair per step
    clk = ClockSampler(local)
    clk.start()
    l0 = g.counters()["kernel_launches"]
    stream = g.stream
    evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
    barrier(pg)
    torch.cuda.synchronize()
    evs[0].record(stream)
    timed = []
    for k in range(args.steps):
        timed += g.run_adaptive(1)
        evs[k + 1].record(stream)
    torch.cuda.synchronize()
    barrier(pg)
    clocks = clk.stop()
    t_ms = evs[0].elapsed_time(evs[-1])
    per_step_ms = [evs[k].elapsed_time(evs[k + 1]) for k in range(args.steps)]
    launches = g.counters()["kernel_launches"] - l0
    t_max = max_over_ranks(pg, t_ms)
    ms_per_step = t_max / args.steps
    # sharded: all ranks advance ONE global grid (strong scaling); replicas: world independent runs
    value = (1 if sharded else world) * args.steps / (t_max / 1e3)

    # ---- profiled pass (after the timed region, same trajectory): per-launch CUDA events on the library
    # stream give every phase's share of the step and the dominant kernel's mean launch duration
    nprof = max(1, min(2, args.steps))
    g.set_profiling(True)
    g.phase_times(reset=True)
    ep0, ep1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ep0.record(stream)
    prof_recs = []
    for _ in range(nprof):
        prof_recs += g.run_adaptive(1)
    ep1.record(stream)
    phases = g.phase_times(reset=True)
    g.set_profiling(False)
    prof_ms = ep0.elapsed_time(ep1)

    dom = max(phases, key=lambda k: phases[k]["ms"])
    rb, P = ras_bytes(g, cfg)
    alg = {
        "ras_apply": rb,
        "residual": 8 * (2 * nf + 3) * N,            # read X^b (nf), c^a, eta^a, T^n; write F (nf)
        "jv": 8 * (2 * nf + 5) * N,                  # read v (nf), jac4 (4), c^a; write (nf)
    }
    peaks = {}
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            peaks = json.load(f)
    except Exception:
        pass
    hbm = float(peaks.get("hbm_gbs", 6650.0))
    peak_src = "MEASURED_PEAKS.json hbm_gbs (measured)" if "hbm_gbs" in peaks else "fallback 6650 GB/s"
    per_launch_ms = {k: (v["ms"] / v["count"] if v["count"] else None) for k, v in phases.items()}
    kern = {}
    for k in ("ras_apply", "residual", "jv"):
        if per_launch_ms.get(k):
            gbs = alg[k] / (per_launch_ms[k] * 1e-3) / 1e9
            kern[k] = {"ms_per_launch": per_launch_ms[k], "launches": phases[k]["count"],
                       "alg_bytes": alg[k], "GB_s": gbs, "frac_hbm": gbs / hbm,
                       "GDOF_s": nf * N / (per_launch_ms[k] * 1e-3) / 1e9}
    if dom in alg and per_launch_ms.get(dom):
        ach = alg[dom] / (per_launch_ms[dom] * 1e-3) / 1e9
        roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": hbm, "unit": "GB/s", "frac": ach / hbm,
                "traffic": None, "peak_source": peak_src, "alg_bytes_per_launch": alg[dom],
                "ms_per_launch": per_launch_ms[dom],
                "share_of_step": phases[dom]["ms"] / prof_ms if prof_ms > 0 else None,
                "measured_in": f"profiled pass of {nprof} steps right after the timed region (per-launch CUDA "
                               "events on the library stream); the timed region itself ran unprofiled"}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                "traffic": None, "peak_source": peak_src}
    if dom == "ras_apply" and d == 2 and per_launch_ms.get(dom):
        # the 2D BILU(0) sweep is a dependency chain: (ex + 2(ey-1)) forward + as many backward wavefront
        # steps per apply (reading R21); its latency roofline is that step count x the measured minimum step
        ex = cfg["shape"][1] // cfg["nsub"][1] + 2 * cfg["overlap"]
        ey = cfg["shape"][0] // cfg["nsub"][0] + 2 * cfg["overlap"]
        nsteps = 2 * (ex + 2 * (ey - 1))
        roof["critical_path_steps"] = nsteps
        roof["ns_per_wavefront_step"] = per_launch_ms[dom] * 1e6 / nsteps
        # minimum latency of one wavefront step: step barrier 22.6 + exchange LDS 29.1 + 4 dependent DFMA
        # x 8.3 + DADD 8.3 + exchange store ~20 cycles (probes: profiles/r01_bar_probe2.txt,
        # profiles/r01_fp64_peak_probe.txt); the apply cannot beat nsteps x that at the measured SM clock
        min_cyc = 22.6 + 29.1 + 4 * 8.3 + 8.3 + 20.0
        sm_mhz = clocks.get("sm_mhz") or 1965.0
        lat_ms = nsteps * min_cyc / (sm_mhz * 1e3)
        roof["latency_roofline"] = {"min_step_cycles": min_cyc, "sm_mhz": sm_mhz, "bound_ms": lat_ms,
                                    "frac": lat_ms / per_launch_ms[dom],
                                    "note": "critical-path steps x minimum step latency (barrier, exchange load, "
                                            "4-deep DFMA chain, add, exchange store)"}

    # ---- the same workload with the B200-native spectral preconditioner (not the configured one-level RAS;
    # DESIGN.md section 9): its own adaptive trajectory from the same seeded state, W + K steps
    variants = {}
    if not sharded and not args.no_variants:
        # the variants' own trajectories, W warm-up + min(K, 6) timed steps (bounded bench time)
        va = argparse.Namespace(warmup=args.warmup, steps=min(args.steps, 6))
        variants["spectral_pc"] = run_variant(va, cfg, model, sol, c, eta, pg, PC_SPECTRAL)
        variants["two_level_ras_spectral"] = run_variant(va, cfg, model, sol, c, eta, pg, 6)

    # ---- the 3D configurations on this GPU, a few steps each: config 3
    # (128^3, RAS 8x8x8 boxes, BILU(0)) with the configured preconditioner and with the spectral one;
    # config 4 (256^3) with the spectral one (its one-level RAS/BILU(0) step takes ~15 min on one GPU,
    # DESIGN.md section 7)
    extra = {}
    if not sharded and world == 1 and not args.no_extra and args.config == 2:
        del g
        torch.cuda.empty_cache()
        g = None
        try:
            extra["config3_sharded_1rank"] = run_sharded_point(args, ni.CONFIGS[3], model, sol, pg, steps=2, warmup=1)
            try:       # the pencil-sharded step at one rank (NCCL self-exchange along z and y), one step
                extra["config3_pencil_1rank"] = run_sharded_point(args, ni.CONFIGS[3], model, sol, pg, steps=1,
                                                                  warmup=0, decomp="pencil")
            except Exception as e:
                extra["config3_pencil_1rank"] = {"error": str(e)[:300]}
        except Exception as e:
            extra["config3_sharded_1rank"] = {"error": str(e)[:300]}
        torch.cuda.empty_cache()
        for key, ecid, pct, w, k in (("config3_spectral", 3, PC_SPECTRAL, 1, 3), ("config4_spectral", 4, PC_SPECTRAL, 1, 2)):
            try:
                ecfg = ni.CONFIGS[ecid]
                ec, ee = ni.initial_fields(ecfg["shape"], 0)
                ea = argparse.Namespace(warmup=w, steps=k)
                extra[key] = run_variant(ea, ecfg, model, sol, ec, ee, pg, pct if pct is not None else 2)
                extra[key]["grid"] = list(ecfg["shape"])
                extra[key]["nsub"] = list(ecfg["nsub"])
                extra[key]["warmup"], extra[key]["steps"] = w, k
            except Exception as e:
                extra[key] = {"error": str(e)[:300]}
            torch.cuda.empty_cache()

    # ---- end to end through the C ABI with host buffers: every step uploads X^n from pinned host memory
    # (nks_set_state, on_device = 0: keeps the controller's history), advances one adaptive step
    # (nks_run_adaptive, retries included, exactly the device leg's work) and downloads X^{n+1}
    e2e = None
    X_e2e_first = None
    if not args.no_e2e and not sharded:
        import ctypes as C
        from paper_2209_08001_b200.nks import StepInfo
        g = None
        torch.cuda.empty_cache()
        g2 = Solver(shape, model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
        g2.set_fields(c, eta, None)
        for _ in range(args.warmup):
            g2.run_adaptive(1)
        Xh = torch.from_numpy(g2.get_state()).pin_memory()
        n_e2e = min(args.steps, 6)       # the first min(K, 6) steps of the timed trajectory (bounded bench time)
        lib = g2.lib
        rec = (StepInfo * 1)()
        done = C.c_int32(0)
        barrier(pg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(g2.stream)
        for k in range(n_e2e):
            rc = lib.nks_set_state(g2.st, C.c_void_p(Xh[0].data_ptr()), C.c_void_p(Xh[1].data_ptr()),
                                   C.c_void_p(Xh[2].data_ptr()), 0)
            assert rc == 0, rc
            rc = lib.nks_run_adaptive(g2.st, 1, C.c_double(0.0), rec, C.byref(done))
            assert rc == 0 and done.value == 1, rc
            rc = lib.nks_get_fields(g2.st, C.c_void_p(Xh[0].data_ptr()), C.c_void_p(Xh[1].data_ptr()),
                                    C.c_void_p(Xh[2].data_ptr()), 0)
            assert rc == 0, rc
            if k == 0 and X_warm is not None:
                X_e2e_first = Xh.numpy().copy()      # host copy of step W+1 (already on the host)
        e1.record(g2.stream)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(pg, e0.elapsed_time(e1))
        del g2
        torch.cuda.empty_cache()
        e2e = {"value": world * n_e2e / (t_e2e / 1e3), "unit": UNIT, "steps": n_e2e,
               "h2d_bytes_per_step": nf * N * 8, "d2h_bytes_per_step": nf * N * 8,
               "wall_s": time.perf_counter() - t0,
               "note": "per step: nks_set_state (pinned host X^n, on_device=0) + nks_run_adaptive(1) + "
                       "nks_get_fields (pinned host); same trajectory and warm-up as the device leg"}

    # ---- CPU baseline: the oracle takes step W+1 of this very trajectory (X^n = the GPU state after the
    # W warm-up steps, dt forced to the GPU's accepted dt) on the full grid; its result is also compared
    # with the GPU's step W+1 (taken from the e2e leg's host copy, same deterministic trajectory)
    cpu = None
    parity = None
    if X_warm is not None:
        cbar0 = float(ni.initial_fields(shape, 0)[0].mean())
        Xo, oinfo, el = oracle_step_sample(cfg, sol, X_warm, cbar0, timed[0]["dt"])
        cpu = {"value": 1.0 / el, "unit": UNIT, "cores": oracle_threads(), "kind": "oracle",
               "sample": f"1 oracle NKS step of the timed trajectory (step {args.warmup + 1}: X^n = the GPU state "
                         f"after {args.warmup} warm-up steps, dt forced to the GPU's accepted "
                         f"{timed[0]['dt']:.6g}) on the full {'x'.join(map(str, shape))} grid, exact Newton via "
                         f"oracle/krylov.py ({oinfo['newton_its']} Newton its), {el:.1f} s",
               "threads_note": "NumPy elementwise work on 1 core, scipy.fft on all cores"}
        if X_e2e_first is not None and oinfo["converged"]:
            rel = [float(np.linalg.norm(X_e2e_first[f] - Xo[f]) / np.linalg.norm(Xo[f])) for f in range(nf)]
            parity = {"step": args.warmup + 1, "dt": timed[0]["dt"], "field_rel_l2": rel,
                      "bar": 1e-8, "ok": max(rel) <= 1e-8}

    micro_sh = None
    if world > 1 and not args.no_micro:
        g = None
        sh = None
        torch.cuda.empty_cache()
        try:
            micro_sh = {"grid": [512, 512, 512], "sharding": f"z-slabs x {world}", **micro_sharded((512, 512, 512), pg)}
            try:
                micro_sh["pencils"] = micro_pencil((512, 512, 512), pg, world)
            except Exception as e:            # reported, never silent
                micro_sh["pencils"] = {"error": repr(e)[:300]}
        except Exception as e:
            micro_sh = {"error": str(e)[:200]}
    micro = {}
    if not args.no_micro and world == 1:
        g = None
        torch.cuda.empty_cache()
        for name, shp in (("2d512", (512, 512)), ("3d256", (256, 256, 256)), ("3d512", (512, 512, 512))):
            try:
                r = micro_kernels(shp)
            except Exception as e:           # e.g. out of memory on a smaller part
                micro[name] = {"error": str(e)[:200]}
                continue
            for k in r:
                r[k]["frac_hbm"] = r[k]["GB_s"] / hbm
                # fp64 ALU roofline: thread-level fp64 ops per point counted by ncu (DFMA+DADD+DMUL,
                # profiles/r01_ncu_F_Jv_fp64_ops_3d256.txt) against 148 SMs x 64 fp64 lanes x max SM clock
                ops = FP64_OPS_PER_POINT.get(k)
                if ops and len(shp) == 3:
                    peak_ops = FP64_OPS_PEAK
                    npts = float(np.prod(shp))
                    r[k]["fp64_ops_per_point"] = ops
                    r[k]["frac_fp64_alu"] = ops * npts / (r[k]["ms"] * 1e-3) / peak_ops
                    r[k]["bound"] = "alu" if k == "residual" else "hbm"
            micro[name] = r

    # DRAM traffic of the roofline kernel from the committed ncu --set full capture (per launch), if any
    traffic = None
    try:
        with open(os.path.join(ROOT, "profiles", "ncu_traffic.json")) as f:
            tr = json.load(f)
        if roof.get("kernel") in tr and tuple(tr[roof["kernel"]].get("grid", [])) == tuple(shape):
            traffic = tr[roof["kernel"]]["dram_bytes_per_launch"]
    except Exception:
        pass
    roof["traffic"] = traffic

    if rank == 0:
        conf = config_dict(cfg, world, sharded, args.decomp)
        conf["gmres_stall_cycles"] = sol["gmres_stall_cycles"]
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": (args.scaling if sharded else "weak"), "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": conf, "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clocks,
                "step_ms": step_stats(per_step_ms), "per_step_ms": [round(x, 3) for x in per_step_ms],
                "parity_vs_oracle": parity, "variants": variants, "configs_3d_one_gpu": extra,
                "kernels": kern, "kernels_micro": micro, "kernels_micro_sharded": micro_sh,
                "phases_ms_profiled_pass": {k: round(v["ms"], 3) for k, v in phases.items()},
                "profiled_pass_ms": prof_ms, "profiled_pass_steps": nprof,
                "solver": {"newton_its": [r["newton_its"] for r in timed], "gmres_its": [r["gmres_its"] for r in timed],
                           "dt": [r["dt"] for r in timed], "retries": [r["retries"] for r in timed],
                           "energy": [r["energy"] for r in timed], "mass": [r["mass"] for r in timed]}}
        print(json.dumps(line), flush=True)


def main():
    args = parse()
    world, rank, local, pg = dist_setup(args.gpus)
    if args.impl == "reference":
        run_reference(args, world, rank, pg)
    else:
        run_gpu(args, world, rank, local, pg)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
