"""Per-phase timing of the first adaptive steps of a config (library CUDA events)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver
cfg = ni.CONFIGS[int(os.environ.get("CFG", "2"))]
g = Solver(cfg["shape"], ni.model_default(), ni.solver_default(), nsub=cfg["nsub"], overlap=cfg["overlap"])
c, eta = ni.initial_fields(cfg["shape"], 0)
g.set_fields(c, eta, None)
g.set_profiling(True)
for k in range(int(os.environ.get("STEPS", "2"))):
    t = time.perf_counter(); r = g.run_adaptive(1); torch.cuda.synchronize()
    ph = g.phase_times(reset=True)
    its = r[0]["gmres_its"]
    print(f"step {k}: {time.perf_counter()-t:.2f} s newton {r[0]['newton_its']} gmres {its} dt {r[0]['dt']:.3f} retries {r[0]['retries']}")
    print("   per launch ms:", {k2: round(v["ms"] / max(v["count"], 1), 4) for k2, v in ph.items() if v["count"]})
    print("   totals ms:", {k2: round(v["ms"], 1) for k2, v in ph.items() if v["count"]})
