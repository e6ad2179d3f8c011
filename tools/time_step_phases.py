"""Per-phase device times of one Delta-t-forced NKS step (library per-launch profiling), for a config.

    CFG=3 DT=0.5 python tools/time_step_phases.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import nks_inputs as ni  # noqa: E402
from paper_2209_08001_b200 import Solver  # noqa: E402

cfg = ni.CONFIGS[int(os.environ.get("CFG", "3"))]
shape = cfg["shape"]
sol = ni.solver_default()
sol["gmres_stall_cycles"] = 3
g = Solver(shape, ni.model_default(), sol, nsub=cfg["nsub"], overlap=cfg["overlap"])
c, eta = ni.initial_fields(shape, 0)
g.set_fields(c, eta, None)
dt = float(os.environ.get("DT", "0.5"))
torch.cuda.synchronize()
g.set_profiling(True)
g.phase_times(reset=True)
info = g.step(dt, raise_on_fail=False)
torch.cuda.synchronize()
ph = g.phase_times(reset=True)
tot = sum(v["ms"] for v in ph.values())
print(json.dumps({"config": cfg["name"], "dt": dt, "newton_its": info.get("newton_its"), "gmres_its": info.get("gmres_its"),
                  "status": info.get("status"), "total_ms": tot,
                  "phases": {k: {"ms": round(v["ms"], 3), "count": v["count"], "ms_per": round(v["ms"] / max(1, v["count"]), 4)}
                             for k, v in sorted(ph.items(), key=lambda kv: -kv[1]["ms"])}}))
