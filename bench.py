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
         its own stream during the timed region), algorithmic bytes per launch / mean duration,
         against MEASURED_PEAKS.json hbm_gbs;
cpu_baseline = the oracle (oracle/, plain NumPy/SciPy) as it stands, on a bounded sample.

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
def oracle_sample(cfg, seconds_hint=20.0):
    """Oracle (plain NumPy/SciPy, as it stands) NKS steps on a bounded sample of the workload.

    The oracle's exact-Newton step (sparse direct LU) on the full 512^2 grid takes tens of
    minutes, so the sample is the same recipe (seed 0, dt = 0.01, same model and tolerances)
    on a 64x64 periodic grid; the time per step is scaled linearly by the point count to the
    workload's grid (a LOWER bound on the oracle's true time: the direct LU is superlinear).
    """
    from oracle import scheme, solver
    import torch
    shape = (64, 64)
    d = len(shape)
    m = scheme.Model.from_dict(d, 0.25, ni.model_default())
    sol = ni.solver_default()
    c, eta = ni.initial_fields(shape, 0)
    cbar = c.mean()
    X = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
    t0 = time.perf_counter()
    n = 0
    while True:
        X, info = solver.newton_step(m, X, 0.01, cbar, sol)
        n += 1
        if time.perf_counter() - t0 >= seconds_hint or n >= 8:
            break
    el = time.perf_counter() - t0
    scale = float(np.prod(shape)) / float(np.prod(cfg["shape"]))
    sps = n / el * scale
    cores = torch.get_num_threads()
    return {"value": sps, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{n} oracle exact-Newton steps (sparse LU) on 2D 64x64, dt=0.01, seed 0, {el:.1f} s; "
                      f"steps/s scaled by points 64^2/{'x'.join(map(str, cfg['shape']))} (lower bound)",
            "os_cpu_count": os.cpu_count()}


def run_reference(args, world, rank, pg):
    if rank != 0:
        return
    cfg = ni.CONFIGS[args.config]
    per = []
    for k in range(args.warmup + args.steps):
        s = oracle_sample(cfg, seconds_hint=5.0)
        if k >= args.warmup:
            per.append(1.0 / s["value"])
    mean_s = float(np.mean(per))
    cb = oracle_sample(cfg, seconds_hint=5.0)
    line = {"impl": "reference", "metric": METRIC, "value": 1.0 / mean_s, "unit": UNIT, "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": mean_s * 1e3, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": config_dict(cfg, args.gpus),
            "cpu_baseline": {"value": 1.0 / mean_s, "unit": UNIT, "cores": cb["cores"], "kind": "oracle",
                             "sample": cb["sample"]},
            "e2e": {"value": 1.0 / mean_s, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)


def config_dict(cfg, ngpus, sharded=False):
    d = len(cfg["shape"])
    return {"workload": f"config {2 if cfg['name'] == '2d_512' else cfg['name']}: {cfg['name']} "
                        f"{'x'.join(map(str, cfg['shape']))} periodic, adaptive dt (P:596-607), "
                        f"RAS {'x'.join(map(str, cfg['nsub']))} boxes delta={cfg['overlap']} BILU(0), GMRES(30)",
            "grid": list(cfg["shape"]), "dof": (2 + d) * int(np.prod(cfg["shape"])),
            "nsub": list(cfg["nsub"]), "overlap": cfg["overlap"], "newton_rtol": 1e-11, "gmres_rtol": 1e-10,
            "init": "c=0.1622+U(-0.005,0.005), eta=0.1+U(-0.01,0.01), seed 0, u0=FFT equilibrium",
            "parallelism": (f"z-slabs x {ngpus} (sharded NKS step, NCCL halo exchange + allreduce)" if sharded
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


def run_gpu(args, world, rank, local, pg):
    import torch
    from paper_2209_08001_b200 import Solver
    from paper_2209_08001_b200.build import build
    build()
    torch.cuda.set_device(local)
    cfg = ni.CONFIGS[args.config]
    shape = cfg["shape"]
    d = len(shape)
    nf = 2 + d
    N = int(np.prod(shape))
    model, sol = ni.model_default(), ni.solver_default()
    sharded = d == 3 and (world > 1 or args.sharded)
    c, eta = ni.initial_fields(shape, 0)
    if sharded:
        # one z-slab per rank; the library calls back for halo exchanges and fixed-order allreduces
        from paper_2209_08001_b200.shard import ShardedSolver
        sh = ShardedSolver(shape, model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
        sh.set_fields(c, eta)
        g = sh.solver
    else:
        sh = None
        g = Solver(shape, model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
        g.set_fields(c, eta, None)
    recs = []
    for _ in range(args.warmup):
        recs += g.run_adaptive(1)
    torch.cuda.synchronize()
    clk = ClockSampler(local)
    clk.start()
    g.set_profiling(True)
    g.phase_times(reset=True)
    l0 = g.counters()["kernel_launches"]
    stream = g.stream
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    barrier(pg)
    torch.cuda.synchronize()
    ev0.record(stream)
    timed = []
    for _ in range(args.steps):
        timed += g.run_adaptive(1)
    ev1.record(stream)
    torch.cuda.synchronize()
    barrier(pg)
    clocks = clk.stop()
    t_ms = ev0.elapsed_time(ev1)
    launches = g.counters()["kernel_launches"] - l0
    phases = g.phase_times(reset=True)
    g.set_profiling(False)
    t_max = max_over_ranks(pg, t_ms)
    ms_per_step = t_max / args.steps
    # sharded: all ranks advance ONE global grid (strong scaling); replicas: world independent runs
    value = (1 if sharded else world) * args.steps / (t_max / 1e3)

    # ---- roofline of the dominant kernel (phase with the largest share of the timed region)
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
                "ms_per_launch": per_launch_ms[dom]}
    else:
        roof = {"kernel": dom, "bound": "hbm", "achieved": None, "peak": hbm, "unit": "GB/s", "frac": None,
                "traffic": None, "peak_source": peak_src}

    # ---- end to end through the C ABI with host buffers: every step uploads X^n from pinned host memory
    # (nks_set_state, on_device = 0: keeps the controller's history), advances one adaptive step
    # (nks_run_adaptive, retries included, exactly the device leg's work) and downloads X^{n+1}
    e2e = None
    if not args.no_e2e and not sharded:
        import ctypes as C
        from paper_2209_08001_b200.nks import StepInfo
        g2 = Solver(shape, model, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
        g2.set_fields(c, eta, None)
        for _ in range(args.warmup):
            g2.run_adaptive(1)
        Xh = torch.from_numpy(g2.get_state()).pin_memory()
        lib = g2.lib
        rec = (StepInfo * 1)()
        done = C.c_int32(0)
        barrier(pg)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(g2.stream)
        for _ in range(args.steps):
            rc = lib.nks_set_state(g2.st, C.c_void_p(Xh[0].data_ptr()), C.c_void_p(Xh[1].data_ptr()),
                                   C.c_void_p(Xh[2].data_ptr()), 0)
            assert rc == 0, rc
            rc = lib.nks_run_adaptive(g2.st, 1, C.c_double(0.0), rec, C.byref(done))
            assert rc == 0 and done.value == 1, rc
            rc = lib.nks_get_fields(g2.st, C.c_void_p(Xh[0].data_ptr()), C.c_void_p(Xh[1].data_ptr()),
                                    C.c_void_p(Xh[2].data_ptr()), 0)
            assert rc == 0, rc
        e1.record(g2.stream)
        torch.cuda.synchronize()
        t_e2e = max_over_ranks(pg, e0.elapsed_time(e1))
        del g2
        e2e = {"value": world * args.steps / (t_e2e / 1e3), "unit": UNIT,
               "h2d_bytes_per_step": nf * N * 8, "d2h_bytes_per_step": nf * N * 8,
               "wall_s": time.perf_counter() - t0,
               "note": "per step: nks_set_state (pinned host X^n, on_device=0) + nks_run_adaptive(1) + "
                       "nks_get_fields (pinned host); same trajectory and warm-up as the device leg"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = oracle_sample(cfg)

    micro_sh = None
    if world > 1 and not args.no_micro:
        del g
        torch.cuda.empty_cache()
        try:
            micro_sh = {"grid": [512, 512, 512], "sharding": f"z-slabs x {world}", **micro_sharded((512, 512, 512), pg)}
        except Exception as e:
            micro_sh = {"error": str(e)[:200]}
        g = None
        sh = None
    micro = {}
    if not args.no_micro and world == 1:
        del g
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
        line = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": ms_per_step, "higher_is_better": True,
                "scaling": "strong" if sharded else "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
                "config": config_dict(cfg, world, sharded), "roofline": roof, "cpu_baseline": cpu, "e2e": e2e,
                "gpu_launches": int(launches), "clocks": clocks,
                "kernels": kern, "kernels_micro": micro, "kernels_micro_sharded": micro_sh,
                "phases_ms": {k: round(v["ms"], 3) for k, v in phases.items()},
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
