"""Time the RAS apply (and J.v, F) at a config's grid on the GPU; check pipelined vs level kernel."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver

cfg = dict(ni.CONFIGS[int(os.environ.get("CFG", "2"))])
if "SHAPE" in os.environ:
    cfg["shape"] = tuple(int(v) for v in os.environ["SHAPE"].split(","))
    cfg["nsub"] = tuple(int(v) for v in os.environ["NSUB"].split(","))
shape = cfg["shape"]; d = len(shape); nf = 2 + d
sol = ni.solver_default()
sol["factor_fp32"] = int(os.environ.get("FP32", "0"))
g = Solver(shape, ni.model_default(), sol, nsub=cfg["nsub"], overlap=cfg["overlap"])
c, eta = ni.initial_fields(shape, 0)
g.set_fields(c, eta, None)
X = g.get_state()
g.pc_setup(X, 0.3)
r = torch.from_numpy(ni.random_direction(nf, shape, 11)).cuda()
z = g.pc_apply(r)
torch.cuda.synchronize()
g.set_profiling(True); g.phase_times(reset=True)
for _ in range(20):
    g.pc_apply(r)
ph = g.phase_times(reset=True)
print("ras_apply ms/launch", ph["ras_apply"]["ms"] / ph["ras_apply"]["count"])
if "OUT" in os.environ:
    np.save(os.environ["OUT"], z.cpu().numpy())
