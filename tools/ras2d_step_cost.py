#!/usr/bin/env python
"""Per-wavefront-step cost of the 2D RAS apply (ras2d_rows.cu) for several box geometries on 512^2.

The apply is a chain of 2 (ex + 2 (ey - 1)) dependent wavefront steps per box (reading R21); a box is
split into a cluster of stripes whose boundary rows travel through distributed shared memory every step.
With the ablation build (NKS_BUILD_TAG=abl NKS_BUILD_DEFS=-DNKS_R2_ABLATE, loaded with NKS_LIB) and
NKS_RAS2D_CSMAX=1, boxes of <= 32 rows run as ONE CTA (no DSMEM hand-off): comparing ns per wavefront step
across geometries and stripe caps separates the in-CTA step latency from the stripe hand-off.

    python tools/ras2d_step_cost.py
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import nks_inputs as ni  # noqa: E402
from paper_2209_08001_b200 import Solver  # noqa: E402
from paper_2209_08001_b200.build import build  # noqa: E402


def main():
    build()
    shape = (512, 512)
    c, eta = ni.initial_fields(shape, 0)
    grid = ((4, 4), (8, 8), (16, 16), (32, 4), (32, 8), (4, 32), (2, 2))
    if os.environ.get("NSUBS"):                  # e.g. NSUBS="4,4;32,4"
        grid = tuple(tuple(int(v) for v in t.split(",")) for t in os.environ["NSUBS"].split(";"))
    for nsub in grid:
        delta = 2
        g = Solver(shape, ni.model_default(), ni.solver_default(), nsub=nsub, overlap=delta)
        g.set_fields(c, eta, None)
        X = g.get_state()
        g.pc_setup(X, 0.5)
        r = torch.rand((4,) + shape, dtype=torch.float64, device="cuda")
        for _ in range(3):
            g.pc_apply(r)
        torch.cuda.synchronize()
        g.set_profiling(True)
        g.phase_times(reset=True)
        for _ in range(20):
            g.pc_apply(r)
        ph = g.phase_times(reset=True)
        g.set_profiling(False)
        ms = ph["ras_apply"]["ms"] / ph["ras_apply"]["count"]
        ey = shape[0] // nsub[0] + 2 * delta
        ex = shape[1] // nsub[1] + 2 * delta
        steps = 2 * (ex + 2 * (ey - 1))
        print(json.dumps({"nsub_yx": nsub, "box_rows": ey, "box_cols": ex, "boxes": nsub[0] * nsub[1],
                          "csmax": os.environ.get("NKS_RAS2D_CSMAX", "8"), "apply_ms": ms, "wavefront_steps": steps,
                          "ns_per_step": ms * 1e6 / steps}), flush=True)
        del g
        torch.cuda.empty_cache()


if __name__ == "__main__":
    main()
