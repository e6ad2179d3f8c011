"""Cost of the controller's attempts at config 2: after the bench's 3 warm-up steps, one nks_step from the
same X^n at each trial dt (the accepted one and the rejected ones the controller tries first), reporting
Newton / GMRES iterations, the failure reason and the wall time; for gmres_stall_cycles in STALL.

    STALL=3,0 DTS=2,1.414,1 NKS_DEBUG=1 python tools/attempt_cost.py   (NKS_DEBUG: per-cycle GMRES residuals on stderr)
"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import nks_inputs as ni
from paper_2209_08001_b200 import Solver

cfg = ni.CONFIGS[2]
shape = cfg["shape"]
c, eta = ni.initial_fields(shape, 0)
for stall in [int(s) for s in os.environ.get("STALL", "3").split(",")]:
    sol = dict(ni.solver_default())
    sol["gmres_stall_cycles"] = stall
    g = Solver(shape, ni.model_default(), sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)
    g.set_fields(c, eta, None)
    for _ in range(3):
        r = g.run_adaptive(1)[0]
        print(f"warm-up step: dt {r['dt']:.4f} retries {r['retries']} newton {r['newton_its']} gmres {r['gmres_its']}",
              flush=True)
    X = g.get_state()
    for dt in [float(x) for x in os.environ.get("DTS", "2.0,1.41421356,1.0").split(",")]:
        g.set_state(X[0], X[1], X[2:])
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        info = g.step(dt, raise_on_fail=False)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        print(f"stall {stall} dt {dt:.4f}: {info['status']} reason {info['reason']} newton {info['newton_its']} "
              f"gmres {info['gmres_its']} ls {info['ls_halvings']} {ms:.0f} ms", flush=True)
    g.set_state(X[0], X[1], X[2:])
    t0 = time.perf_counter()
    r = g.run_adaptive(1)[0]
    torch.cuda.synchronize()
    print(f"stall {stall} adaptive step: dt {r['dt']:.4f} retries {r['retries']} newton {r['newton_its']} gmres "
          f"{r['gmres_its']} {(time.perf_counter() - t0) * 1e3:.0f} ms", flush=True)
    del g
