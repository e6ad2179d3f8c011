"""Preconditioner family study: one NKS step from the config-2 initial state on a 2D
grid, for RAS / AS / RRAS and overlap delta in {0, 1, 2}: Newton iterations, GMRES iterations per Newton
iteration and wall time per step (the trends of the paper's Tables 1-2; synthetic input)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import nks_inputs as ni
from paper_2209_08001_b200 import PC_AS_BILU0, PC_RAS_BILU0, PC_RRAS_BILU0, Solver

shape = tuple(int(v) for v in os.environ.get("SHAPE", "256,256").split(","))
nsub = tuple(int(v) for v in os.environ.get("NSUB", "4,4").split(","))
dt = float(os.environ.get("DT", "0.5"))
c, eta = ni.initial_fields(shape, 0)
print(f"grid {shape} boxes {nsub} dt {dt}")
for name, pct in (("RAS", PC_RAS_BILU0), ("AS", PC_AS_BILU0), ("RRAS", PC_RRAS_BILU0)):
    for delta in (0, 1, 2):
        g = Solver(shape, ni.model_default(), ni.solver_default(), nsub=nsub, overlap=delta, pc_type=pct)
        g.set_fields(c, eta, None)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        info = g.step(dt, raise_on_fail=False)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
        nn = max(1, info["newton_its"])
        print(f"{name:5s} delta {delta}: {info['status']:8s} newton {info['newton_its']:2d}  gmres {info['gmres_its']:6d} "
              f"({info['gmres_its'] / nn:7.1f} per Newton)  {t:7.3f} s  energy {info['energy']:.10e}", flush=True)
        del g
