"""Pins of oracle/scheme.py against what the paper and mathematics fix (no GPU).

Each test names the passage it pins.  None of them re-types the oracle's formula:
they check closed forms, high-precision values (mpmath), exact discrete identities
(DVD, summation by parts), symmetries and special cases.
"""
import json
import math
import os

import mpmath as mp
import numpy as np
import pytest

import nks_inputs as ni
from oracle import scheme, solver

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "paper_constants.json")))
mp.mp.dps = 50


def model(d=2, **over):
    p = ni.model_default()
    p.update(over)
    return scheme.Model.from_dict(d, 0.25, p)


# ----------------------------------------------------------------------------- Psi and derivatives

def test_psi_closed_forms():
    assert scheme.psi(0.5) == pytest.approx(GOLD["psi_half"]["value"], rel=1e-15)
    z = np.linspace(0.01, 0.99, 97)
    np.testing.assert_allclose(scheme.psi(z), scheme.psi(1 - z), rtol=1e-14, atol=1e-16)
    ref = mp.mpf("0.25") * mp.log(mp.mpf("0.25")) + mp.mpf("0.75") * mp.log(mp.mpf("0.75"))
    assert scheme.psi(0.25) == pytest.approx(float(ref), rel=1e-15)


@pytest.mark.parametrize("s", [1, 2, 3, 4, 5, 6, 9])
def test_psi_derivatives_vs_mpmath(s):
    f = lambda z: z * mp.log(z) + (1 - z) * mp.log(1 - z)
    for z in [0.05, 0.3, 0.5, 0.77]:
        ref = mp.diff(f, mp.mpf(z), s)
        assert scheme.psi_deriv(z, s) == pytest.approx(float(ref), rel=1e-12)


# ----------------------------------------------------------------------------- Psi_S quotient

def _psiS_literal_mp(y1, y2, S):
    """Literal P:452-456 in 50-digit arithmetic: [Psi_S(ybar, d) - Psi_S(ybar, -d)]/(2d)."""
    f = lambda z: z * mp.log(z) + (1 - z) * mp.log(1 - z)
    yb = (mp.mpf(y1) + mp.mpf(y2)) / 2
    dl = (mp.mpf(y2) - mp.mpf(y1)) / 2
    ders = [mp.diff(f, yb, s) for s in range(0, 2 * S + 1)]

    def PS(x):
        return ders[0] + sum(x ** s * ders[s] / mp.factorial(s) for s in range(1, 2 * S + 1))
    return (PS(dl) - PS(-dl)) / (2 * dl)


@pytest.mark.parametrize("y1,y2", [(0.2, 0.21), (0.1, 0.13), (0.5, 0.6), (0.016, 0.02), (0.6, 0.61)])
def test_psiS_equals_literal_definition(y1, y2):
    assert scheme.psiS_quotient(y1, y2, 10) == pytest.approx(float(_psiS_literal_mp(y1, y2, 10)), rel=1e-13)


def test_psiS_special_cases():
    # delta = 0 -> Psi'(ybar) (the quotient's limit)
    for y in [0.01, 0.2, 0.5, 0.9]:
        assert scheme.psiS_quotient(y, y, 10) == pytest.approx(math.log(y / (1 - y)), rel=1e-15, abs=1e-15)
    # symmetric in its arguments
    assert scheme.psiS_quotient(0.2, 0.3, 10) == scheme.psiS_quotient(0.3, 0.2, 10)


@pytest.mark.parametrize("y1,y2", [(0.2, 0.24), (0.1, 0.15), (0.016, 0.02), (0.4, 0.7)])
def test_psiS_truncation_bound(y1, y2):
    """|Psi_S - Psi[y1,y2]| <= (|delta|/min(ybar,1-ybar))^(2S) (Taylor remainder)."""
    f = lambda z: z * mp.log(z) + (1 - z) * mp.log(1 - z)
    exact = (f(mp.mpf(y1)) - f(mp.mpf(y2))) / (mp.mpf(y1) - mp.mpf(y2))
    yb, dl = (y1 + y2) / 2, abs(y2 - y1) / 2
    r = dl / min(yb, 1 - yb)
    err = abs(scheme.psiS_quotient(y1, y2, 10) - float(exact))
    assert err <= r ** 20 + 1e-14 * abs(float(exact))
    # and the truncation error decreases with S (R^S -> 0)
    errs = [abs(scheme.psiS_quotient(y1, y2, S) - float(exact)) for S in (2, 4, 6)]
    assert errs[0] >= errs[1] >= errs[2] or errs[0] < 1e-14


# ----------------------------------------------------------------------------- App. A vs App. B

def _complex_step(f, x, *args):
    return np.imag(f(x + 1e-30j, *args)) / 1e-30


def test_appB_coefficients_are_gradients_of_appA_polynomial():
    """dPhi/dc = M0 + M1 c + M2 c^2 + M3 c^3 + M4 c^4 and dPhi/deta = M5 phi + M6 phi^2 (P:1102-1103,
    P:1113-1121) where Phi is App. A's polynomial part -- verifies the printed M's."""
    m = model()
    rng = np.random.default_rng(3)
    c = rng.uniform(0.05, 0.25, 200)
    eta = rng.uniform(0.0, 1.2, 200)
    phi = 1 - eta
    dc = np.imag(scheme.E1(m, c + 1e-30j, eta + 0j)) / 1e-30
    de = np.imag(scheme.E1(m, c + 0j, eta + 1e-30j)) / 1e-30
    ref_c = m.M0() + m.M1(phi) * c + m.M2(phi) * c ** 2 + m.M3() * c ** 3 + m.M4() * c ** 4
    ref_e = m.M5(c) * phi + m.M6(c) * phi ** 2
    np.testing.assert_allclose(dc, ref_c, rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(de, ref_e, rtol=1e-12, atol=1e-10)


def test_model_default_has_printed_wells():
    """Model-default coefficients (reading R6): the two printed equilibria have a
    common chemical potential and eta-stationarity of the ordered well."""
    m = model()
    (c1, e1), (c2, e2) = GOLD["wells"]["value"]
    f = lambda c, e: scheme.E1(m, c, e) + scheme.E2(m, c, e)
    mu1 = np.imag(f(c1 + 1e-30j, e1 - 1e-9 + 0j)) / 1e-30
    mu2 = np.imag(f(c2 + 1e-30j, e2 + 0j)) / 1e-30
    assert mu1 == pytest.approx(mu2, rel=1e-4)
    de2 = np.imag(f(c2 + 0j, e2 + 1e-30j)) / 1e-30
    assert abs(de2) < 1e-3 * abs(mu2)


# ----------------------------------------------------------------------------- DVD identities

def _pairs(n=400, seed=4):
    rng = np.random.default_rng(seed)
    ca = rng.uniform(0.05, 0.24, n)
    ea = rng.uniform(0.02, 1.0, n)
    cb = ca + rng.uniform(-0.03, 0.03, n)
    eb = ea + rng.uniform(-0.2, 0.2, n)
    eb = np.clip(eb, 0.01, 1.1)
    return ca, ea, cb, eb


def test_G1_exact_discrete_gradient():
    """G^1 . (V^b - V^a) = E1(b) - E1(a) exactly (App. B)."""
    m = model()
    ca, ea, cb, eb = _pairs()
    gc, ge = scheme.G1(m, ca, cb, ea, eb)
    lhs = gc * (cb - ca) + ge * (eb - ea)
    rhs = scheme.E1(m, cb, eb) - scheme.E1(m, ca, ea)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-11, atol=1e-12)


def test_G1_collapses_to_gradient():
    m = model()
    ca, ea, _, _ = _pairs()
    gc, ge = scheme.G1(m, ca, ca, ea, ea)
    dc = np.imag(scheme.E1(m, ca + 1e-30j, ea + 0j)) / 1e-30
    de = np.imag(scheme.E1(m, ca + 0j, ea + 1e-30j)) / 1e-30
    np.testing.assert_allclose(gc, dc, rtol=1e-12, atol=1e-10)
    np.testing.assert_allclose(ge, de, rtol=1e-12, atol=1e-10)


def test_G2_exact_quotient_is_exact_dvd_and_G2S_approximates_it():
    """Eq. (D2): G^2.(dV) = E2(b) - E2(a); G^{2,S} -> G^2."""
    m = model()
    ca, ea, cb, eb = _pairs()
    keep = (np.abs(cb - ca) > 1e-3) & (np.abs(cb * eb - ca * ea) > 1e-3) & \
           (np.abs(cb * (4 - 3 * eb) - ca * (4 - 3 * ea)) > 1e-3)
    ca, ea, cb, eb = ca[keep], ea[keep], cb[keep], eb[keep]
    gc, ge = scheme.G2_exact(m, ca, cb, ea, eb)
    lhs = gc * (cb - ca) + ge * (eb - ea)
    rhs = scheme.E2(m, cb, eb) - scheme.E2(m, ca, ea)
    np.testing.assert_allclose(lhs, rhs, rtol=1e-9, atol=1e-11)
    # small steps: Psi_S quotient agrees with the exact one to the Taylor bound
    cb2 = ca * (1 + 1e-2)
    eb2 = ea * (1 + 1e-2)
    g2s = scheme.G2S(m, ca, cb2, ea, eb2)
    g2e = scheme.G2_exact(m, ca, cb2, ea, eb2)
    np.testing.assert_allclose(g2s[0], g2e[0], rtol=1e-8, atol=1e-8)


def test_G2S_collapses_to_log_gradient():
    """a = b: G^{2,S} = (dE2/dc, dE2/deta) (P:1102-1104 log parts)."""
    m = model()
    ca, ea, _, _ = _pairs()
    gc, ge = scheme.G2S(m, ca, ca, ea, ea)
    dc = np.imag(scheme.E2(m, ca + 1e-30j, ea + 0j)) / 1e-30
    de = np.imag(scheme.E2(m, ca + 0j, ea + 1e-30j)) / 1e-30
    np.testing.assert_allclose(gc, dc, rtol=1e-12, atol=1e-12)
    np.testing.assert_allclose(ge, de, rtol=1e-12, atol=1e-12)
    # theta = 0 -> 0
    m0 = model(theta=0.0)
    assert np.all(scheme.G2S(m0, ca, ca * 1.01, ea, ea)[0] == 0)


@pytest.mark.parametrize("d,shape", [(2, (8, 10)), (3, (6, 4, 6))])
def test_G3_dvd_with_equilibrium_at_both_levels(d, shape):
    """<G^3 . dV> = E~3(b) - E~3(a) when [D^ sigma^el] = 0 at both levels (reading R12/R13)."""
    m = model(d)
    ca, ea = ni.initial_fields(shape, 1)
    cb, eb = ni.initial_fields(shape, 2)
    cbar = ca.mean()
    cb = cb - cb.mean() + cbar          # same mass
    ua = solver.init_displacement(m, ca, cbar)
    ub = solver.init_displacement(m, cb, cbar)
    Xa = np.concatenate([ca[None], ea[None], ua])
    Xb = np.concatenate([cb[None], eb[None], ub])
    g3c, _ = scheme.G3(m, Xa, Xb, cbar)
    vol = m.h ** d
    lhs = vol * np.sum(g3c * (cb - ca))
    rhs = scheme.energy_parts(m, Xb, cbar)[2] - scheme.energy_parts(m, Xa, cbar)[2]
    assert lhs == pytest.approx(rhs, rel=1e-10, abs=1e-14)


@pytest.mark.parametrize("d,shape", [(2, (8, 10)), (3, (5, 4, 6))])
def test_G4_dvd(d, shape):
    """<G^4 . dV> = E~4(b) - E~4(a)."""
    m = model(d)
    ca, ea = ni.initial_fields(shape, 1)
    cb, eb = ni.initial_fields(shape, 2, c_amp=0.02, eta_amp=0.05)
    X = lambda c, e: np.concatenate([c[None], e[None], np.zeros((d,) + shape)])
    Xa, Xb = X(ca, ea), X(cb, eb)
    g4c, g4e = scheme.G4(m, Xa, Xb)
    lhs = m.h ** d * np.sum(g4c * (cb - ca) + g4e * (eb - ea))
    rhs = scheme.energy_parts(m, Xb, 0.0)[3] - scheme.energy_parts(m, Xa, 0.0)[3]
    assert lhs == pytest.approx(rhs, rel=1e-11)


def test_G4_fourier_symbol():
    """D^2 of a single Fourier mode = -sum_j (2 - 2 cos k_j h)/h^2 times the mode."""
    m = model(2)
    ny, nx = 8, 12
    y, x = np.meshgrid(np.arange(ny), np.arange(nx), indexing="ij")
    kx, ky = 2 * np.pi * 3 / nx, 2 * np.pi * 1 / ny
    f = np.cos(kx * x + ky * y)
    lap = scheme.laplacian(f, m.h, 2)
    sym = -((2 - 2 * np.cos(kx)) + (2 - 2 * np.cos(ky))) / m.h ** 2
    np.testing.assert_allclose(lap, sym * f, atol=1e-12)


# ----------------------------------------------------------------------------- summation by parts / A11

def test_summation_by_parts_prefactor_one():
    """-sum phi D(M~ D psi) = sum_faces M~ D^+phi D^+psi (Eq. summation; reading R15: prefactor 1)."""
    m = model(2)
    shape = (9, 12)
    rng = np.random.default_rng(7)
    phi, psi_, ca = rng.normal(size=shape), rng.normal(size=shape), rng.uniform(0.1, 0.2, shape)
    lhs = -np.sum(phi * scheme.div_M_grad(psi_, ca, m.kappa, m.h, 2))
    rhs = sum(np.sum(scheme.mobility_face(ca, m.kappa, j, 2) * scheme.D_plus(phi, j, m.h, 2)
                     * scheme.D_plus(psi_, j, m.h, 2)) for j in range(2))
    assert lhs == pytest.approx(rhs, rel=1e-12)


def test_A11_semipositive_symmetric_cauchy_schwarz():
    """Eq. (neq:02)."""
    m = model(3)
    shape = (4, 5, 6)
    rng = np.random.default_rng(8)
    ca = rng.uniform(0.1, 0.2, shape)
    A = lambda f: -scheme.div_M_grad(f, ca, m.kappa, m.h, 3)
    for _ in range(5):
        a, b = rng.normal(size=shape), rng.normal(size=shape)
        aa, bb, ab, ba = np.sum(a * A(a)), np.sum(b * A(b)), np.sum(a * A(b)), np.sum(b * A(a))
        assert aa >= 0 and bb >= 0
        assert ab == pytest.approx(ba, rel=1e-12)
        assert abs(ab) <= math.sqrt(aa * bb) * (1 + 1e-12)


# ----------------------------------------------------------------------------- residual F

def test_residual_uniform_state():
    """Uniform c, eta, u = 0: F_c = F_u = 0 identically; F_eta = 0 where eta^b solves the scalar
    equation (eta - eta0)/dt + G^1_eta + G^{2,S}_eta = 0 found by a bracketing root finder."""
    from scipy.optimize import brentq
    m = model(2)
    shape = (6, 8)
    c0, e0, dt = 0.1622, 0.1, 0.05
    Xa = np.zeros((4,) + shape)
    Xa[0], Xa[1] = c0, e0
    g = lambda eb: (eb - e0) / dt + (scheme.G1(m, c0, c0, e0, eb)[1] + scheme.G2S(m, c0, c0, e0, eb)[1])
    eb = brentq(g, 0.01, 0.9, xtol=1e-15)
    Xb = Xa.copy()
    Xb[1] = eb
    F = scheme.residual(m, Xa, Xb, dt, c0)
    assert np.abs(F).max() < 1e-11
    # and the oracle Newton reaches the same uniform root
    Xn, info = solver.newton_step(m, Xa, dt, c0, ni.solver_default())
    assert info["converged"]
    np.testing.assert_allclose(Xn[1], eb, rtol=1e-12)
    np.testing.assert_allclose(Xn[0], c0, rtol=1e-14)


def _rand_state(d, shape, seed=0):
    ca, ea = ni.initial_fields(shape, seed)
    cb, eb = ni.perturbed_state(ca, ea, seed + 1, 1e-2)
    ua = ni.random_displacement(d, shape, seed + 2)
    ub = ni.random_displacement(d, shape, seed + 3)
    Xa = np.concatenate([ca[None], ea[None], ua])
    Xb = np.concatenate([cb[None], eb[None], ub])
    return Xa, Xb, ca.mean()


def test_residual_translation_equivariance():
    m = model(3)
    Xa, Xb, cb = _rand_state(3, (5, 6, 7))
    F = scheme.residual(m, Xa, Xb, 0.1, cb)
    roll = lambda X: np.roll(np.roll(X, 2, axis=1), -3, axis=3)
    F2 = scheme.residual(m, roll(Xa), roll(Xb), 0.1, cb)
    np.testing.assert_allclose(F2, roll(F), rtol=1e-13, atol=1e-12)


def test_residual_axis_permutation_symmetry():
    """Cubic C is symmetric under swapping x and y (with u_x <-> u_y)."""
    m = model(3)
    Xa, Xb, cb = _rand_state(3, (6, 6, 5))

    def swap(X):
        Y = np.swapaxes(X, 2, 3).copy()       # array axes (z, y, x): swap y and x
        Y[[2, 3]] = Y[[3, 2]]
        return Y
    F = scheme.residual(m, Xa, Xb, 0.1, cb)
    F2 = scheme.residual(m, swap(Xa), swap(Xb), 0.1, cb)
    np.testing.assert_allclose(F2, swap(F), rtol=1e-12, atol=1e-11)


def test_residual_reflection_symmetry():
    """Reflection i_x -> -i_x (about a cell) with u_x -> -u_x maps F to the reflected F (F_ux negated)."""
    m = model(2)
    Xa, Xb, cb = _rand_state(2, (6, 8))

    def refl(X, flip_u=True):
        Y = np.roll(X[..., ::-1], 1, axis=-1).copy()
        if flip_u:
            Y[2] = -Y[2]
        return Y
    F = scheme.residual(m, Xa, Xb, 0.1, cb)
    F2 = scheme.residual(m, refl(Xa), refl(Xb), 0.1, cb)
    np.testing.assert_allclose(F2, refl(F), rtol=1e-12, atol=1e-11)


def test_residual_mass_rows_telescope():
    """sum_i (D M~ D G)_i = 0, so sum F_c = sum (c^b - c^a)/dt (mass law P:389)."""
    m = model(2)
    Xa, Xb, cb = _rand_state(2, (7, 9))
    F = scheme.residual(m, Xa, Xb, 0.3, cb)
    assert np.sum(F[0]) == pytest.approx(np.sum(Xb[0] - Xa[0]) / 0.3, rel=1e-10, abs=1e-9)


def test_residual_reductions_theta_L_gamma_zero():
    """theta = Lscale = gamma = 0: F_c, F_eta involve only G^1; F_u = 0 (P:634 L = 0 case)."""
    m = model(2, theta=0.0, Lscale=0.0, gamma_c=0.0, gamma_eta=0.0)
    Xa, Xb, cb = _rand_state(2, (6, 6))
    F = scheme.residual(m, Xa, Xb, 0.1, cb)
    g1 = scheme.G1(m, Xa[0], Xb[0], Xa[1], Xb[1])
    assert np.abs(F[2:]).max() == 0.0
    np.testing.assert_allclose(F[1], (Xb[1] - Xa[1]) / 0.1 + g1[1], rtol=1e-14)


def test_elastic_energy_nonnegative_and_quadratic():
    m = model(3)
    Xa, _, cb = _rand_state(3, (4, 5, 6))
    e3 = scheme.E3(m, Xa[2:], Xa[0], cb)
    assert np.all(e3 >= 0)
    e3b = scheme.E3(m, 2 * Xa[2:], 2 * (Xa[0] - cb) + cb, cb)
    np.testing.assert_allclose(e3b, 4 * e3, rtol=1e-12)


def test_gauge_invariance_of_residual():
    """Adding a constant on each parity sub-lattice to u leaves F unchanged (reading R14)."""
    m = model(2)
    Xa, Xb, cb = _rand_state(2, (6, 8))
    ids, ncls = solver.sublattice_ids((6, 8))
    Y = Xb.copy()
    for k in range(ncls):
        Y[2][ids == k] += 0.3 * (k + 1)
        Y[3][ids == k] -= 0.2 * (k + 2)
    np.testing.assert_allclose(scheme.residual(m, Xa, Y, 0.1, cb), scheme.residual(m, Xa, Xb, 0.1, cb),
                               rtol=1e-11, atol=1e-9)
