"""Pins of the oracle's Krylov path (oracle/krylov.py) and of the controller's retry and the Newton
line-search branches (oracle/solver.py) -- no GPU.

What pins what:
  * matrix-free J v  = the assembled sparse J (jacobian.assemble) and the complex-step directional
    derivative of F (an independent definition, exact to rounding);
  * SpectralPC       = the exact inverse of J at a uniform state (constant coefficients), checked by
    applying it to J v -- ties the hand-written Fourier symbol to the operator;
  * gmres            = numpy's dense solve on small nonsymmetric systems (textbook special case);
  * Newton with the Krylov path = Newton with the gauge-pinned direct LU (the exact oracle);
  * run_adaptive retry rule: two forced failures -> dt/2, zeta*4;
  * line search (reading R17): a rejected lambda = 1 followed by an accepted lambda < 1, each decision
    re-checked here against the admissibility and Armijo conditions.
"""
import math

import numpy as np
import pytest

import nks_inputs as ni
from oracle import jacobian, krylov, scheme, solver

SOL = ni.solver_default()


def model(d):
    return scheme.Model.from_dict(d, 0.25, ni.model_default())


def init_state(shape, seed=0):
    d = len(shape)
    m = model(d)
    c, eta = ni.initial_fields(shape, seed)
    cbar = c.mean()
    X = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
    return m, X, cbar


@pytest.mark.parametrize("shape", [(8, 10), (5, 6, 7)])
def test_matfree_jv_matches_assembled_and_complex_step(shape):
    m, Xa, cbar = init_state(shape)
    d = len(shape)
    Xb = Xa.copy()
    Xb[:2] += np.stack(ni.perturbed_state(Xa[0], Xa[1], 3, 2e-3)) - Xa[:2]
    Xb[2:] += ni.random_displacement(d, shape, 4, 1e-4)
    v = ni.random_direction(2 + d, shape, 5)
    jm = krylov.Linearisation(m, Xa, Xb, 0.07).jv(v)
    ja = jacobian.jv(m, Xa, Xb, 0.07, v)
    jc = jacobian.jv_complex_step(m, Xa, Xb, 0.07, cbar, v)
    s = np.linalg.norm(jc)
    assert np.linalg.norm(jm - ja) <= 1e-13 * s
    assert np.linalg.norm(jm - jc) <= 1e-13 * s


@pytest.mark.parametrize("shape,dt", [((12, 10), 0.01), ((12, 10), 2.0), ((6, 5, 4), 0.3), ((7, 9), 0.5)])
def test_spectral_pc_inverts_the_uniform_state_jacobian(shape, dt):
    """At a uniform state every coefficient of J is constant, so the per-wave-number inverse is exact:
    PC(J v) = v for every v without a gauge component (odd axes included: no parity null modes)."""
    d = len(shape)
    m = model(d)
    X = np.zeros((2 + d,) + shape)
    X[0], X[1] = 0.1622, 0.13
    Xb = X.copy()
    Xb[0], Xb[1] = 0.1630, 0.128          # level b differs from a: a_kl of the DVD quotients, still uniform
    lin = krylov.Linearisation(m, X, Xb, dt)
    pcd = krylov.SpectralPC(lin)
    v = solver.gauge_project(ni.random_direction(2 + d, shape, 7))
    back = pcd.apply(lin.jv(v))
    assert np.linalg.norm(back - v) <= 1e-11 * np.linalg.norm(v)


@pytest.mark.parametrize("n,restart", [(40, 30), (60, 7)])
def test_gmres_solves_small_systems(n, restart):
    rng = np.random.default_rng(n)
    A = np.eye(n) * 4 + rng.uniform(-1, 1, (n, n)) / math.sqrt(n)
    b = rng.uniform(-1, 1, n)
    Minv = np.linalg.inv(np.diag(np.diag(A)))
    x, its, res, ok = krylov.gmres(lambda v: A @ v, b, 1e-12 * np.linalg.norm(b), restart, 1000,
                                   lambda v: Minv @ v)
    assert ok and res <= 1e-12 * np.linalg.norm(b)
    np.testing.assert_allclose(x, np.linalg.solve(A, b), rtol=0, atol=1e-10)
    assert np.linalg.norm(b - A @ x) == pytest.approx(res, rel=1e-6, abs=1e-14)


@pytest.mark.parametrize("shape,dt", [((16, 16), 0.01), ((16, 16), 2.0), ((12, 14), 0.5), ((6, 8, 8), 0.01),
                                      ((6, 8, 8), 1.0)])
def test_krylov_newton_equals_direct_newton(shape, dt):
    """The large-grid oracle path (spectral-preconditioned GMRES(30), xi_r = 1e-10) reaches the same
    root as exact Newton with the gauge-pinned direct LU, with the same Newton count."""
    m, X, cbar = init_state(shape)
    Xd, i_d = solver.newton_step(m, X, dt, cbar, SOL)
    stats = []
    Xk, i_k = solver.newton_step(m, X, dt, cbar, SOL, linsolve=krylov.make_linsolve(stats=stats))
    assert i_d["converged"] and i_k["converged"]
    assert i_d["newton_its"] == i_k["newton_its"]
    assert all(s["converged"] for s in stats)
    for f in range(X.shape[0]):
        assert np.linalg.norm(Xk[f] - Xd[f]) <= 1e-12 * max(np.linalg.norm(Xd[f]), 1e-300)
    assert scheme.energy(m, Xk, cbar) == pytest.approx(scheme.energy(m, Xd, cbar), rel=1e-13)


def test_controller_retry_rule_two_forced_failures(monkeypatch):
    """a diverged attempt is retried with dt/sqrt(2) and zeta*2.  Two forced failures at the
    second step must give dt = predicted/2 and zeta = 4 zeta_0, and zeta stays doubled afterwards."""
    shape = (12, 12)
    m, X, cbar = init_state(shape)
    real = solver.newton_step
    calls = {"n": 0, "dts": []}

    def flaky(m_, Xa, dt, cbar0, sol, X0=None, linsolve=None):
        calls["n"] += 1
        calls["dts"].append(dt)
        if calls["n"] in (2, 3):                 # the first two attempts of step 1 fail
            return Xa.copy(), {"converged": False, "reason": "forced", "newton_its": 0, "lambdas": []}
        return real(m_, Xa, dt, cbar0, sol, X0=X0, linsolve=linsolve)

    monkeypatch.setattr(solver, "newton_step", flaky)
    sol = dict(SOL)
    _, recs = solver.run_adaptive(m, X, cbar, sol, 3)
    predicted = calls["dts"][1]
    assert predicted > sol["dt_min"]
    assert calls["dts"][2] == pytest.approx(predicted / math.sqrt(2), rel=1e-15)
    assert recs[1]["dt"] == pytest.approx(predicted / 2, rel=1e-15)
    assert recs[1]["retries"] == 2 and recs[1]["zeta"] == 4 * sol["zeta"]
    assert recs[0]["retries"] == 0 and recs[0]["zeta"] == sol["zeta"]
    assert recs[2]["zeta"] == 4 * sol["zeta"]                       # zeta is never reset


def test_controller_dt_floor_aborts(monkeypatch):
    """Every attempt failing drives dt below dt_min/1024 (reading R24): the run aborts."""
    shape = (8, 8)
    m, X, cbar = init_state(shape)

    def always_fail(m_, Xa, dt, cbar0, sol, X0=None, linsolve=None):
        return Xa.copy(), {"converged": False, "reason": "forced", "newton_its": 0, "lambdas": []}

    monkeypatch.setattr(solver, "newton_step", always_fail)
    with pytest.raises(RuntimeError, match="floor"):
        solver.run_adaptive(m, X, cbar, dict(SOL), 1)


def _check_line_search(m, Xa, dt, cbar, scale):
    """Newton with the direction scaled by `scale`: the first iterate's lambda must be the first of
    1, 1/2, ... whose trial state is admissible and satisfies ||F(X + l S)|| <= (1 - 1e-4 l) ||F(X)||."""
    def scaled(m_, Xa_, X, dt_, cbar0, b, fnorm):
        return scale * solver.direct_linsolve(m_, Xa_, X, dt_, cbar0, b, fnorm)

    Xs, info = solver.newton_step(m, Xa, dt, cbar, SOL, linsolve=scaled)
    assert info["converged"]
    lam = info["lambdas"][0]
    assert lam < 1.0
    # re-derive the first iterate's decisions independently
    F0 = scheme.residual(m, Xa, Xa, dt, cbar)
    f0 = np.linalg.norm(F0)
    S = scale * solver.direct_linsolve(m, Xa, Xa, dt, cbar, solver.gauge_project(-F0), f0)
    reasons = []
    l = 1.0
    while l > lam:
        Xt = Xa + l * S
        if not scheme.admissible(Xt):
            reasons.append("inadmissible")
        else:
            ft = np.linalg.norm(scheme.residual(m, Xa, Xt, dt, cbar))
            assert not ft <= (1 - SOL["ls_alpha"] * l) * f0
            reasons.append("armijo")
        l /= 2
    assert l == lam
    Xt = Xa + lam * S
    assert scheme.admissible(Xt)
    assert np.linalg.norm(scheme.residual(m, Xa, Xt, dt, cbar)) <= (1 - SOL["ls_alpha"] * lam) * f0
    # the iteration still reaches the root of the unmodified Newton iteration
    Xd, _ = solver.newton_step(m, Xa, dt, cbar, SOL)
    for f in range(Xa.shape[0]):
        assert np.linalg.norm(Xs[f] - Xd[f]) <= 1e-10 * np.linalg.norm(Xd[f])
    return lam, reasons


def test_line_search_rejects_full_step_by_armijo():
    m, X, cbar = init_state((10, 12))
    lam, reasons = _check_line_search(m, X, 0.05, cbar, 3.0)     # lambda = 1 overshoots: F -> ~ -2F
    assert lam == 0.5 and reasons == ["armijo"]


def test_line_search_rejects_inadmissible_trial_states():
    m, X, cbar = init_state((10, 12))
    lam, reasons = _check_line_search(m, X, 0.05, cbar, 600.0)
    assert "inadmissible" in reasons and lam <= 2.0 ** -9
