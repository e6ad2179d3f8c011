"""Pins of the oracle's homogeneous Neumann boundary conditions (Eq. (boundaryequ); reading
R38: cell-centred mirror ghosts, even for c, eta, u, odd stress ghosts in the outer derivative of the u
rows) -- no GPU.

What pins what:
  * the u rows are minus the gradient of the discrete elastic energy (complex-step derivative of E~3, an
    independent definition): the traction-free condition is the natural one of E~3 (n.sigma = 0);
  * G^4 at a = b is the gradient of the discrete interfacial energy E~4 (complex step): the mirror ghosts
    make the boundary differences vanish (n.grad c = n.grad eta = 0);
  * the flux form conserves mass exactly (n.M grad mu = 0; Thm. 2.1);
  * summation by parts without boundary terms (the B_1, B_2 of P:160 vanish);
  * the elastic operator is symmetric with the translations as its only null space (the gauge, R38);
  * J v = complex-step derivative of F; the Newton step conserves mass, decreases the energy and obeys the
    per-step dissipation identity; the Krylov path reaches the direct-LU root.
"""
import numpy as np
import pytest

import nks_inputs as ni
from oracle import jacobian, krylov, scheme, solver

SOL = ni.solver_default()
H = 0.25


def model(d):
    return scheme.Model.from_dict(d, H, ni.model_default(), bc="neumann")


def state(shape, seed=0):
    d = len(shape)
    m = model(d)
    c, eta = ni.initial_fields(shape, seed)
    cbar = c.mean()
    u = solver.init_displacement(m, c, cbar)
    return m, np.concatenate([c[None], eta[None], u]), cbar


def _grad_cs(fun, x, eps=1e-30):
    g = np.zeros(x.size)
    flat = x.ravel()
    for k in range(x.size):
        xc = flat.astype(complex)
        xc[k] += 1j * eps
        g[k] = np.imag(fun(xc.reshape(x.shape))) / eps
    return g.reshape(x.shape)


@pytest.mark.parametrize("shape", [(5, 6), (3, 4, 3)])
def test_u_rows_are_minus_the_elastic_energy_gradient(shape):
    d = len(shape)
    m = model(d)
    rng = np.random.default_rng(1)
    c = 0.16 + 0.01 * rng.uniform(-1, 1, shape)
    u = 1e-3 * rng.uniform(-1, 1, (d,) + shape)
    X = np.concatenate([c[None], 0.1 + 0 * c[None], u])
    cbar = 0.158
    F = scheme.residual(m, X, X, 1.0, cbar)
    vol = H ** d
    g = _grad_cs(lambda uu: vol * np.sum(scheme.E3(m, uu, c.astype(complex), cbar)), u)
    np.testing.assert_allclose(F[2:], -g / vol, rtol=0, atol=1e-12 * np.abs(g / vol).max())


@pytest.mark.parametrize("shape", [(5, 6), (4, 3, 5)])
def test_G4_is_the_interfacial_energy_gradient(shape):
    d = len(shape)
    m = model(d)
    rng = np.random.default_rng(2)
    c = 0.16 + 0.01 * rng.uniform(-1, 1, shape)
    eta = 0.1 + 0.01 * rng.uniform(-1, 1, shape)
    X = np.concatenate([c[None], eta[None], np.zeros((d,) + shape)])
    g4c, g4e = scheme.G4(m, X, X)
    vol = H ** d
    gc = _grad_cs(lambda cc: vol * np.sum(scheme.E4(m, cc, eta.astype(complex))), c)
    ge = _grad_cs(lambda ee: vol * np.sum(scheme.E4(m, c.astype(complex), ee)), eta)
    np.testing.assert_allclose(g4c, gc / vol, rtol=0, atol=1e-11 * np.abs(gc / vol).max())
    np.testing.assert_allclose(g4e, ge / vol, rtol=0, atol=1e-11 * np.abs(ge / vol).max())


def test_flux_form_conserves_mass_and_sums_by_parts():
    shape = (7, 9)
    rng = np.random.default_rng(3)
    ca = 0.16 + 0.01 * rng.uniform(-1, 1, shape)
    g, f = rng.normal(size=shape), rng.normal(size=shape)
    assert abs(np.sum(scheme.div_M_grad(g, ca, 0.008, H, 2, "neumann"))) < 1e-13 * np.abs(g).sum() / H ** 2
    # -sum f Lap g = sum over the INTERIOR faces of D+f D+g (no boundary term), brute force
    lhs = -np.sum(f * scheme.laplacian(g, H, 2, "neumann"))
    rhs = 0.0
    ny, nx = shape
    for y in range(ny):
        for x in range(nx):
            if x + 1 < nx:
                rhs += (f[y, x + 1] - f[y, x]) * (g[y, x + 1] - g[y, x]) / H ** 2
            if y + 1 < ny:
                rhs += (f[y + 1, x] - f[y, x]) * (g[y + 1, x] - g[y, x]) / H ** 2
    assert lhs == pytest.approx(rhs, rel=1e-12)


@pytest.mark.parametrize("shape,expect", [((6, 7), 2), ((6, 6), 3), ((5, 5), 2), ((8, 8), 3), ((4, 4, 4), 6),
                                          ((4, 5, 4), 4)])
def test_elastic_null_space_is_rigid_motions(shape, expect):
    """Nullity = the d translations + one discrete rotation per pair of even extents (reading R38); the
    rotation modes of solver.neumann_rotations are in the null space; the pinned matrix is nonsingular."""
    d = len(shape)
    m = model(d)
    Auu, _ = solver.elastic_block(m, shape)
    A = Auu.toarray()
    np.testing.assert_allclose(A, A.T, atol=1e-9 * np.abs(A).max())
    s = np.linalg.svd(A, compute_uv=False)
    assert int(np.sum(s < 1e-9 * s[0])) == expect
    n = int(np.prod(shape))
    for I in range(d):                    # every constant component is in the null space
        v = np.zeros(d * n)
        v[I * n:(I + 1) * n] = 1.0
        assert np.abs(A @ v).max() < 1e-9 * np.abs(A).max()
    rots = solver.neumann_rotations(shape)
    assert len(rots) == expect - d
    for r in rots:
        assert np.abs(A @ r.ravel()).max() < 1e-9 * np.abs(A).max()
    rows = [r - 2 * n for r in solver.pinned_rows(shape, d, "neumann")]
    Ap, _ = solver.pin(Auu, np.zeros(d * n), rows)
    s2 = np.linalg.svd(Ap.toarray(), compute_uv=False)
    assert s2[-1] > 1e-10 * s2[0]


@pytest.mark.parametrize("shape", [(8, 10), (5, 6, 5)])
def test_neumann_jv_matches_complex_step(shape):
    m, Xa, cbar = state(shape)
    d = len(shape)
    Xb = Xa.copy()
    Xb[:2] += np.stack(ni.perturbed_state(Xa[0], Xa[1], 3, 2e-3)) - Xa[:2]
    v = ni.random_direction(2 + d, shape, 4)
    jc = jacobian.jv_complex_step(m, Xa, Xb, 0.1, cbar, v)
    ja = jacobian.jv(m, Xa, Xb, 0.1, v)
    jm = krylov.Linearisation(m, Xa, Xb, 0.1).jv(v)
    s = np.linalg.norm(jc)
    assert np.linalg.norm(ja - jc) <= 1e-13 * s and np.linalg.norm(jm - jc) <= 1e-13 * s


@pytest.mark.parametrize("dt", [0.01, 0.5, 2.0])
def test_neumann_step_laws(dt):
    """Newton step with Neumann boundaries: quadratic convergence, mass conservation, energy decay and the
    per-step dissipation identity E^b - E^a = -dt h^d [sum_faces M~ (D+ G_c)^2 + sum G_eta^2] + <R^S.dV>,
    the boundary faces carrying no flux."""
    shape = (10, 12)
    m, Xa, cbar = state(shape)
    Xb, info = solver.newton_step(m, Xa, dt, cbar, SOL)
    assert info["converged"]
    assert abs(scheme.mass(m, Xb) - scheme.mass(m, Xa)) <= 1e-12 * abs(scheme.mass(m, Xa))
    assert scheme.energy(m, Xb, cbar) <= scheme.energy(m, Xa, cbar) + 1e-10
    assert np.abs(scheme.residual(m, Xb, Xb, 1.0, cbar)[2:]).max() < 1e-9    # equilibrium at the new level
    gc, ge = scheme.G_S(m, Xa, Xb, cbar)
    vol = H ** 2
    diss = np.sum(ge ** 2)
    for j in range(2):
        mp = scheme.mobility_face(Xa[0], m.kappa, j, 2, "neumann")
        dg = scheme.D_plus(gc, j, H, 2, "neumann")           # 0 across the boundary faces
        diss += np.sum(mp * dg ** 2)
    g2e = scheme.G2_exact(m, Xa[0], Xb[0], Xa[1], Xb[1])
    g2s = scheme.G2S(m, Xa[0], Xb[0], Xa[1], Xb[1])
    rs = vol * np.sum((g2e[0] - g2s[0]) * (Xb[0] - Xa[0]) + (g2e[1] - g2s[1]) * (Xb[1] - Xa[1]))
    lhs = scheme.energy(m, Xb, cbar) - scheme.energy(m, Xa, cbar)
    assert lhs == pytest.approx(-dt * vol * diss + rs, rel=1e-7, abs=1e-9)
    h = info["hist"]
    for k in range(1, len(h) - 1):
        if h[k] > 1e-8 * h[0]:
            assert h[k + 1] <= 50.0 * h[k] ** 2 / h[0] + 1e-12 * h[0]


def test_neumann_translation_gauge_and_krylov_path():
    """F is invariant under a constant displacement (the gauge); the Krylov Newton path reaches the
    direct-LU root."""
    shape = (12, 10)
    m, X, cbar = state(shape)
    Y = X.copy()
    Y[2] += 0.3
    Y[3] -= 0.1
    np.testing.assert_allclose(scheme.residual(m, X, Y, 0.1, cbar), scheme.residual(m, X, X, 0.1, cbar),
                               rtol=0, atol=1e-10)
    Xd, i_d = solver.newton_step(m, X, 0.3, cbar, SOL)
    Xk, i_k = solver.newton_step(m, X, 0.3, cbar, SOL, linsolve=krylov.make_linsolve())
    assert i_d["converged"] and i_k["converged"] and i_d["newton_its"] == i_k["newton_its"]
    for f in range(X.shape[0]):
        assert np.linalg.norm(Xk[f] - Xd[f]) <= 1e-11 * np.linalg.norm(Xd[f])
    for I in (2, 3):
        assert abs(Xd[I].mean()) < 1e-15
    for r in solver.neumann_rotations(shape):
        assert abs(np.sum(Xd[2:] * r)) < 1e-14


def test_neumann_boxes_stop_at_the_walls():
    """Neumann Schwarz boxes (R38): extended by delta inside the domain only; owned points tile the grid."""
    from oracle import pc
    shape = (10, 12)
    owned = np.zeros(120, dtype=int)
    for b in pc.boxes(shape, (3, 2), 2, "neumann"):
        for j in range(2):
            assert b["s0"][j] >= 0 and b["s0"][j] + b["ext"][j] <= b["n"][j]
            assert b["ext"][j] <= b["own"][j] + 4
        for l in pc.local_points(b):
            if pc.is_owned(b, l):
                owned[pc.global_index(b, l)] += 1
    assert np.all(owned == 1)
