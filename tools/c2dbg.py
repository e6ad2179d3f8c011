import sys, time; sys.path.insert(0, ".")
import numpy as np, torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver
cfg = ni.CONFIGS[2]
g = Solver(cfg["shape"], ni.model_default(), ni.solver_default(), nsub=cfg["nsub"], overlap=2)
c, eta = ni.initial_fields(cfg["shape"], 0)
g.set_fields(c, eta, None)
for k in range(5):
    t = time.perf_counter(); r = g.run_adaptive(1); torch.cuda.synchronize()
    print("STEP", k, "%.2f s"%(time.perf_counter() - t), r[0]["newton_its"], r[0]["gmres_its"], r[0]["dt"], r[0]["retries"], flush=True)
