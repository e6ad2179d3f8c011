import os, sys
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver
shape=(512,512); nsub=(4,4)
g = Solver(shape, ni.model_default(), ni.solver_default(), nsub=nsub, overlap=2)
c, eta = ni.initial_fields(shape, 0)
g.set_fields(c, eta, None)
X = g.get_state()
print("set ok", flush=True)
g.pc_setup(X, 0.3)
torch.cuda.synchronize()
print("pc_setup ok", flush=True)
r = torch.from_numpy(ni.random_direction(4, shape, 11)).cuda()
z = g.pc_apply(r)
torch.cuda.synchronize()
print("apply ok", float(z.abs().max()), flush=True)
