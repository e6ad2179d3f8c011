"""Microbenchmark of the residual F (K1) and matrix-free J.v (K2) kernels.

For each grid: X^n from the common seeded init (u^0 = 0 is enough: kernel cost is value independent),
X^b = X^n + U(-1e-3, 1e-3) on c and eta, v ~ U(-1, 1); dt = 0.01.  Kernel time = the library's
CUDA events around the launch on its own stream (nks_phase_times), mean over REPS launches after
warm-up.  Algorithmic bytes per point: F reads X^b (nf), c^a, eta^a, T^n and
writes F (nf); J.v reads v (nf), the 4 cached pointwise partials, c^a and writes nf.

    python tools/micro_fjv.py [2d512] [3d128] [3d256] [3d512]
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import nks_inputs as ni
from paper_2209_08001_b200 import PC_NONE, Solver

GRIDS = {"2d512": (512, 512), "3d128": (128, 128, 128), "3d256": (256, 256, 256), "3d512": (512, 512, 512)}
REPS = int(os.environ.get("REPS", "20"))


def run(name, shape, hbm):
    d = len(shape)
    nf = 2 + d
    N = int(np.prod(shape))
    sol = dict(ni.solver_default())
    sol["gmres_restart"] = 1            # no Krylov basis needed (512^3 would not fit with 31 vectors)
    g = Solver(shape, ni.model_default(), sol, pc_type=PC_NONE)
    gen = torch.Generator(device="cuda").manual_seed(0)
    c = 0.1622 + (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.01
    eta = 0.1 + (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 0.02
    u = torch.zeros((d,) + tuple(shape), device="cuda", dtype=torch.float64)
    g.set_fields(c, eta, u)
    xb = torch.cat([c[None], eta[None], u]).contiguous()
    xb[0] += (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2e-3
    xb[1] += (torch.rand(shape, device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2e-3
    v = (torch.rand((nf,) + tuple(shape), device="cuda", dtype=torch.float64, generator=gen) - 0.5) * 2
    for _ in range(3):
        g.eval_residual(xb, 0.01)
        g.eval_jv(xb, v, 0.01)
    torch.cuda.synchronize()
    g.set_profiling(True)
    g.phase_times(reset=True)
    for _ in range(REPS):
        g.eval_residual(xb, 0.01)
        g.eval_jv(xb, v, 0.01)
    ph = g.phase_times(reset=True)
    out = {}
    for key, per_pt in (("residual", 2 * nf + 3), ("jv", 2 * nf + 5)):
        ms = ph[key]["ms"] / ph[key]["count"]
        gbs = per_pt * 8 * N / (ms * 1e-3) / 1e9
        out[key] = {"ms": ms, "GDOF_s": nf * N / (ms * 1e-3) / 1e9, "alg_GB_s": gbs, "frac_hbm": gbs / hbm,
                    "alg_bytes": per_pt * 8 * N}
    del g
    torch.cuda.empty_cache()
    return out


if __name__ == "__main__":
    peaks = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                        "MEASURED_PEAKS.json")))
    hbm = float(peaks["hbm_gbs"])
    names = sys.argv[1:] or ["2d512", "3d128", "3d256"]
    res = {n: run(n, GRIDS[n], hbm) for n in names}
    print(json.dumps({"hbm_gbs_measured": hbm, "kernels": res}, indent=1))
