"""Does the opt-in early-divergence rule (gmres_stall_cycles, R18) change the controller's
decisions?  Runs the bench's config-2 trajectory (STEPS adaptive steps from the common seeded init) once per
value in STALL and prints, per step, the accepted dt, retries, Newton / GMRES counts, energy and wall time.
With STALL=0 every failed attempt runs to gmres_maxit (the paper's behaviour), so identical dt / retries
sequences mean the rule only cut work.

    STALL=0,3 STEPS=9 python tools/trajectory_check.py
"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import nks_inputs as ni
from paper_2209_08001_b200 import Solver

cfg = ni.CONFIGS[2]
shape = cfg["shape"]
steps = int(os.environ.get("STEPS", "9"))
c, eta = ni.initial_fields(shape, 0)
runs = {}
for stall in [int(s) for s in os.environ.get("STALL", "0,3").split(",")]:
    sol = dict(ni.solver_default())
    sol["gmres_stall_cycles"] = stall
    g = Solver(shape, ni.model_default(), sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
    g.set_fields(c, eta, None)
    recs = []
    for k in range(steps):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        r = g.run_adaptive(1)[0]
        torch.cuda.synchronize()
        rec = {"step": k, "dt": r["dt"], "retries": r["retries"], "newton": r["newton_its"], "gmres": r["gmres_its"],
               "energy": r["energy"], "zeta": r["zeta"], "s": round(time.perf_counter() - t0, 3)}
        recs.append(rec)
        print(json.dumps({"stall": stall, **rec}), flush=True)
    runs[stall] = recs
    del g
keys = sorted(runs)
if len(keys) > 1:
    a, b = runs[keys[0]], runs[keys[1]]
    same = all(x["dt"] == y["dt"] and x["retries"] == y["retries"] for x, y in zip(a, b))
    print(json.dumps({"same_dt_and_retries": same,
                      "max_energy_rel_diff": max(abs(x["energy"] - y["energy"]) / abs(y["energy"]) for x, y in zip(a, b)),
                      "seconds": {k: round(sum(r["s"] for r in runs[k]), 1) for k in keys}}))
