#!/usr/bin/env python
"""Subdomain-solver / preconditioner table at BASELINE config 2 (paper Table 1).

    python tools/pc_table.py [--warmup 3] [--dts 0.986,2.0] [--solvers ilu0,ilu1,ilu2,spectral,none] [--lu-grid 128]

X^n = the state after W accepted adaptive steps of the configured run (RAS 4x4 boxes, delta = 2, BILU(0),
GMRES(30), the bench's gmres_stall_cycles = 3).  From that SAME X^n every solver takes one step at each
forced dt: Newton iterations, GMRES iterations per Newton, preconditioner setups, wall time of the step
(CUDA events on the library stream), and whether it converged (a stalled BILU(0) solve is reported as
DIVERGED / gmres_stagnation, which the adaptive controller would retry with dt/sqrt(2)).
The exact block LU (ilu_level = -1) is run on a smaller grid (--lu-grid, 4x4 boxes) because its
sequential natural-order factorisation of 132^2-point boxes is impractically slow.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import nks_inputs as ni  # noqa: E402

SOLVERS = {"ilu0": (2, 0), "ilu1": (2, 1), "ilu2": (2, 2), "lu": (2, -1), "spectral": (5, 0), "two_level": (6, 0),
           "none": (0, 0)}


def one(shape, nsub, X, sol, pc, level, dt):
    import torch
    from paper_2209_08001_b200 import Solver
    s = dict(sol, ilu_level=level)
    t0 = time.perf_counter()
    g = Solver(shape, ni.model_default(), s, nsub=nsub, overlap=2, pc_type=pc, pc_reuse=1)
    g.set_fields(X[0], X[1], X[2:])
    torch.cuda.synchronize()
    t_create = time.perf_counter() - t0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(g.stream)
    info = g.step(dt, raise_on_fail=False)
    e1.record(g.stream)
    torch.cuda.synchronize()
    out = {"dt": dt, "status": info["status"], "reason": info["reason"], "newton_its": info["newton_its"],
           "gmres_its": info["gmres_its"], "gmres_per_newton": info["gmres_its"] / max(info["newton_its"], 1),
           "pc_setups": info["pc_setups"], "step_ms": e0.elapsed_time(e1), "create_s": t_create,
           "workspace_GB": g.workspace_bytes / 1e9}
    del g
    torch.cuda.empty_cache()
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--dts", default="0.986,1.414,2.0")
    ap.add_argument("--solvers", default="ilu0,ilu1,ilu2,spectral,two_level")
    ap.add_argument("--lu-grid", type=int, default=128)
    args = ap.parse_args()
    import torch
    from paper_2209_08001_b200 import Solver
    from paper_2209_08001_b200.build import build
    build()
    cfg = ni.CONFIGS[2]
    sol = dict(ni.solver_default(), gmres_stall_cycles=3)
    c, eta = ni.initial_fields(cfg["shape"], 0)
    g = Solver(cfg["shape"], ni.model_default(), sol, nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
    g.set_fields(c, eta, None)
    for _ in range(args.warmup):
        g.run_adaptive(1)
    X = g.get_state()
    del g
    torch.cuda.empty_cache()
    dts = [float(v) for v in args.dts.split(",")]
    for name in args.solvers.split(","):
        pc, lv = SOLVERS[name]
        for dt in dts:
            r = one(cfg["shape"], cfg["nsub"], X, sol, pc, lv, dt)
            print(json.dumps({"grid": list(cfg["shape"]), "solver": name, **r}), flush=True)
    # exact LU on a smaller grid: same recipe (W adaptive steps first), ILU(0) beside it for the trend
    n = args.lu_grid
    shp = (n, n)
    c, eta = ni.initial_fields(shp, 0)
    g = Solver(shp, ni.model_default(), sol, nsub=(4, 4), overlap=2, pc_reuse=1)
    g.set_fields(c, eta, None)
    for _ in range(args.warmup):
        g.run_adaptive(1)
    X = g.get_state()
    del g
    for name in ("ilu0", "ilu1", "ilu2", "lu"):
        pc, lv = SOLVERS[name]
        for dt in dts:
            r = one(shp, (4, 4), X, sol, pc, lv, dt)
            print(json.dumps({"grid": list(shp), "solver": name, **r}), flush=True)


if __name__ == "__main__":
    main()
