"""Debug helper: run a few NKS steps on the GPU against the oracle and print per-step diagnostics."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np

import nks_inputs as ni
from oracle import scheme, solver
from paper_2209_08001_b200 import Solver

shape = tuple(int(s) for s in os.environ.get("SHAPE", "64,64").split(","))
nsub = tuple(int(s) for s in os.environ.get("NSUB", "1,1").split(","))
dt = float(os.environ.get("DT", "0.01"))
steps = int(os.environ.get("STEPS", "3"))
d = len(shape)
MODEL, SOL = ni.model_default(), ni.solver_default()
m = scheme.Model.from_dict(d, 0.25, MODEL)
c, eta = ni.initial_fields(shape, 0)
cbar = c.mean()
Xo = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
g = Solver(shape, MODEL, SOL, h=0.25, nsub=nsub, overlap=2)
g.set_fields(c, eta, None)
for k in range(steps):
    t0 = time.perf_counter()
    Xo, io = solver.newton_step(m, Xo, dt, cbar, SOL)
    t1 = time.perf_counter()
    ig = g.step(dt, raise_on_fail=False)
    t2 = time.perf_counter()
    Xg = g.get_state()
    rel = [float(np.linalg.norm(Xg[f] - Xo[f]) / np.linalg.norm(Xo[f])) for f in range(2 + d)]
    print(f"step {k}: oracle {io.get('newton_its')} its {t1-t0:.2f}s | gpu {ig['status']} newton {ig['newton_its']} "
          f"gmres {ig['gmres_its']} fnorm0 {ig['fnorm0']:.3e} fnorm {ig['fnorm']:.3e} {t2-t1:.3f}s | rel {rel}", flush=True)
    if ig["status"] != "OK":
        break
