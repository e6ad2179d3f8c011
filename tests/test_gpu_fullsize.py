"""Full-size step parity (BASELINE configs 2 and 3) -- GPU through the C ABI vs the oracle.

The GPU runs the configuration exactly as bench.py does (config 2: 512^2, RAS 4x4 boxes, delta = 2,
BILU(0), GMRES(30); config 3: 128^3, RAS 8x8x8 boxes); the oracle takes the same steps in
"dt-forced" mode (SURVEY 8(c) "Parity criteria": parity per step on the accepted dt sequence) with
its large-grid Krylov path (oracle/krylov.py: matrix-free J v + spectral-preconditioned GMRES(30),
pinned against the exact gauge-pinned direct-LU Newton in tests/test_oracle_krylov.py).  Both sides
stop at Newton rtol 1e-11 (reading R16) from identical seeded inputs.

Bar (BASELINE.json north_star): relative L2 <= 1e-8 per field (u in the canonical gauge, R14),
energy relative <= 1e-10, mass drift <= 1e-12 relative.
"""
import time

import numpy as np
import pytest

import nks_inputs as ni
from oracle import krylov, scheme, solver

pytestmark = pytest.mark.gpu

MODEL = ni.model_default()


def rel_l2(a, b):
    return [float(np.linalg.norm(a[f] - b[f]) / max(np.linalg.norm(b[f]), 1e-300)) for f in range(a.shape[0])]


def _gpu(cfg, sol):
    from paper_2209_08001_b200 import Solver
    return Solver(cfg["shape"], MODEL, sol, h=cfg["h"], nsub=cfg["nsub"], overlap=cfg["overlap"], pc_reuse=1)


def _oracle_init(cfg):
    shape = cfg["shape"]
    m = scheme.Model.from_dict(len(shape), cfg["h"], MODEL)
    c, eta = ni.initial_fields(shape, 0)
    cbar = c.mean()
    u = solver.init_displacement_fft(m, c, cbar)
    X = solver.gauge_project(np.concatenate([c[None], eta[None], u]))
    return m, X, cbar


def _compare(Xg, Xo, m, cbar, Xprev, tag):
    errs = rel_l2(Xg, Xo)
    assert max(errs) <= 1e-8, (tag, errs)
    eg, eo = scheme.energy(m, Xg, cbar), scheme.energy(m, Xo, cbar)
    assert abs(eg - eo) <= 1e-10 * abs(eo), (tag, eg, eo)
    m0 = scheme.mass(m, Xprev)
    assert abs(scheme.mass(m, Xg) - m0) <= 1e-12 * abs(m0), tag
    return errs


def test_config2_two_steps_of_the_bench_trajectory():
    """Config 2 (2D 512^2): the first two accepted steps of bench.py's trajectory (adaptive controller,
    the bench's gmres_stall_cycles = 3), replayed dt-forced by the oracle.  Also records how the free
    running controllers compare: both predict the same dt from the same X'_d (Eq. sencondt); the GPU's
    BILU(0)-RAS GMRES may stagnate at that dt and retry where the exact oracle does not."""
    cfg = ni.CONFIGS[2]
    sol = dict(ni.solver_default(), gmres_stall_cycles=3)
    m, X, cbar = _oracle_init(cfg)
    g = _gpu(cfg, sol)
    g.set_fields(*ni.initial_fields(cfg["shape"], 0), None)
    Xg0 = g.get_state()
    assert max(rel_l2(Xg0, X)) <= 1e-10          # u^0: GPU cuFFT vs oracle numpy FFT, same gauge
    Xprev = None
    for k in range(2):
        rec = g.run_adaptive(1)[0]
        Xg = g.get_state()
        if k == 1:
            # the oracle's own controller, same history: the predicted dt must be the GPU's first attempt
            xd = solver.change_rate(X, Xprev, dt_prev, "rms")
            pred = solver.predict_dt(xd, sol["zeta"], sol["dt_min"], sol["dt_max"])
            assert rec["xd"] == pytest.approx(xd, rel=1e-9)
            assert rec["dt"] == pytest.approx(pred / np.sqrt(2) ** rec["retries"], rel=1e-9)
        t0 = time.perf_counter()
        Xo, info = solver.newton_step(m, X, rec["dt"], cbar, sol, linsolve=krylov.make_linsolve())
        assert info["converged"]
        errs = _compare(Xg, Xo, m, cbar, X, f"config 2 step {k}")
        print(f"config2 step {k}: dt {rec['dt']:.6g} retries {rec['retries']} newton gpu {rec['newton_its']} "
              f"oracle {info['newton_its']} gmres gpu {rec['gmres_its']}; rel L2 {['%.1e' % e for e in errs]}; "
              f"oracle {time.perf_counter() - t0:.1f} s")
        Xprev, X, dt_prev = X, Xo, rec["dt"]


def test_config3_first_step():
    """Config 3 (3D 128^3, RAS 8x8x8 boxes of 16^3, delta = 2): the trajectory's first step (dt_init =
    0.01) on the GPU against the oracle's Newton step on the same seeded state."""
    cfg = ni.CONFIGS[3]
    sol = dict(ni.solver_default(), gmres_stall_cycles=3)
    m, X, cbar = _oracle_init(cfg)
    g = _gpu(cfg, sol)
    g.set_fields(*ni.initial_fields(cfg["shape"], 0), None)
    assert max(rel_l2(g.get_state(), X)) <= 1e-10
    rec = g.run_adaptive(1)[0]
    Xg = g.get_state()
    del g
    Xo, info = solver.newton_step(m, X, rec["dt"], cbar, sol, linsolve=krylov.make_linsolve())
    assert info["converged"] and rec["dt"] == sol["dt_init"]
    errs = _compare(Xg, Xo, m, cbar, X, "config 3 step 0")
    print(f"config3 step 0: dt {rec['dt']} newton gpu {rec['newton_its']} oracle {info['newton_its']}; "
          f"rel L2 {['%.1e' % e for e in errs]}")
