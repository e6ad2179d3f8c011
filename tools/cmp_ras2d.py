"""Compare the 2D RAS apply designs (one lane per row / 4 lanes per row / level-synchronous) on the GPU:
outputs must agree to roundoff, and each is timed with CUDA events (20 launches after warm-up)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import nks_inputs as ni
from paper_2209_08001_b200 import Solver

CASES = [((512, 512), (4, 4), 2), ((96, 80), (3, 2), 2), ((64, 64), (1, 1), 2), ((130, 70), (2, 1), 1)]
if "SHAPE" in os.environ:
    CASES = [(tuple(int(v) for v in os.environ["SHAPE"].split(",")), tuple(int(v) for v in os.environ["NSUB"].split(",")), 2)]
MODES = {"rows": {}, "quad": {"NKS_RAS2D_OLD": "1"}, "level": {"NKS_RAS_LEVEL": "1"}}
for shape, nsub, ov in CASES:
    nf = 4
    c, eta = ni.initial_fields(shape, 0)
    r = torch.from_numpy(ni.random_direction(nf, shape, 11)).cuda()
    out = {}
    for name, env in MODES.items():
        for k in ("NKS_RAS2D_OLD", "NKS_RAS_LEVEL"):
            os.environ.pop(k, None)
        os.environ.update(env)
        sol = ni.solver_default()
        sol["factor_fp32"] = int(os.environ.get("FP32", "0"))
        g = Solver(shape, ni.model_default(), sol, nsub=nsub, overlap=ov)
        g.set_fields(c, eta, None)
        X = g.get_state()
        g.pc_setup(X, 0.3)
        z = g.pc_apply(r)
        torch.cuda.synchronize()
        g.set_profiling(True); g.phase_times(reset=True)
        for _ in range(20):
            g.pc_apply(r)
        ph = g.phase_times(reset=True)
        out[name] = (z.cpu().numpy(), ph["ras_apply"]["ms"] / max(1, ph["ras_apply"]["count"]))
        del g
    ref = out["level"][0]
    msg = [f"{shape} nsub {nsub} ov {ov}:"]
    for name, (z, ms) in out.items():
        err = np.abs(z - ref).max() / np.abs(ref).max()
        msg.append(f"{name} {ms:.4f} ms relerr {err:.2e}")
    print(" | ".join(msg), flush=True)
