"""Time the GMRES vector kernels inside real iterations: config 2 state, one preconditioned GMRES solve
(nks_gmres_solve), per-phase CUDA events; prints ms per launch of each phase."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver
cfg = ni.CONFIGS[int(os.environ.get("CFG", "2"))]
shape = cfg["shape"]; nf = 2 + len(shape)
sol = ni.solver_default(); sol["gmres_maxit"] = int(os.environ.get("ITS", "300"))
g = Solver(shape, ni.model_default(), sol, nsub=cfg["nsub"], overlap=cfg["overlap"])
c, eta = ni.initial_fields(shape, 0)
g.set_fields(c, eta, None)
X = g.get_state()
rhs = torch.from_numpy(ni.random_direction(nf, shape, 5)).cuda()
g.set_profiling(True); g.phase_times(reset=True)
try:
    g.gmres_solve(X, rhs, 0.5)
except Exception as e:
    print("gmres:", str(e)[:80])
ph = g.phase_times(reset=True)
for k, v in ph.items():
    if v["count"]:
        print(f"{k:12s} {v['count']:6d} launches {v['ms']:9.3f} ms  {1e3 * v['ms'] / v['count']:8.1f} us/launch")
