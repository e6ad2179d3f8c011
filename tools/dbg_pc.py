"""Debug: RAS apply on a small 2D grid vs the oracle; print where the error lives (box-local rows)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import nks_inputs as ni
from oracle import jacobian, pc, scheme
from paper_2209_08001_b200 import Solver

shape = tuple(int(v) for v in os.environ.get("SHAPE", "16,16").split(","))
nsub = tuple(int(v) for v in os.environ.get("NSUB", "2,2").split(","))
delta = int(os.environ.get("DELTA", "2"))
d = 2
MODEL = ni.model_default()
ca, ea = ni.initial_fields(shape, 0)
ua = ni.random_displacement(d, shape, 2, 1e-3)
Xa = np.concatenate([ca[None], ea[None], ua])
cb, eb = ni.perturbed_state(ca, ea, 1, 2e-3)
Xb = np.concatenate([cb[None], eb[None], ua])
g = Solver(shape, MODEL, ni.solver_default(), nsub=nsub, overlap=delta)
g.set_fields(Xa[0], Xa[1], Xa[2:])
g.pc_setup(Xb, 0.3)
r = ni.random_direction(4, shape, 11)
zg = g.pc_apply(r).cpu().numpy()
m = scheme.Model.from_dict(d, 0.25, MODEL)
J = jacobian.assemble(m, Xa, Xb, 0.3)
zo = pc.RAS(J, shape, 4, tuple(reversed(nsub)), delta).apply(r)
err = np.abs(zg - zo).max(axis=0)
print("max rel err", np.abs(zg - zo).max() / np.abs(zo).max())
np.set_printoptions(linewidth=250, precision=1)
print((np.log10(err + 1e-30)).round(0))
