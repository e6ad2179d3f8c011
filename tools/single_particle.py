"""the paper's single-particle workload on the GPU path:
80^3, h = 0.25, a sphere of radius 7.5 at the centre with c = 0.238, eta = 0.01 inside and c = 0.1375,
eta = 0.99 outside, adaptive dt, RAS 8x8x8 boxes delta = 2.  Prints per accepted step the
dt, Newton/GMRES counts, the energy parts E~1..E~4 (E~3 elastic, E~4 interfacial) and the mass.

    STEPS=20 LSCALE=1 python tools/single_particle.py
"""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver

n = int(os.environ.get("N", "80"))
shape = (n, n, n)
model = ni.model_default()
model["Lscale"] = float(os.environ.get("LSCALE", "1"))
c, eta = ni.sphere_fields(shape, 0.25, 7.5, 0.238, 0.01, 0.1375, 0.99)
g = Solver(shape, model, ni.solver_default(), h=0.25, nsub=(8, 8, 8), overlap=2)
g.set_fields(c, eta, None)
print(f"single particle {n}^3, L = {model['Lscale']}")
print("step      dt  retries newton gmres       E1            E2            E3            E4           mass     s")
for k in range(int(os.environ.get("STEPS", "10"))):
    t0 = time.perf_counter()
    r = g.run_adaptive(1)[0]
    torch.cuda.synchronize()
    e = r["energy_parts"]
    print(f"{k:4d} {r['dt']:8.4f} {r['retries']:4d} {r['newton_its']:6d} {r['gmres_its']:6d} "
          f"{e[0]:13.6e} {e[1]:13.6e} {e[2]:13.6e} {e[3]:13.6e} {r['mass']:13.8e} {time.perf_counter()-t0:6.2f}",
          flush=True)
