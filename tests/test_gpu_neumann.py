"""Homogeneous Neumann boundaries (Eq. (boundaryequ); reading R38) on the GPU
against the oracle (oracle/ with Model(bc="neumann"), pinned in tests/test_oracle_neumann.py): F and J.v
element by element, energy, the gauge (translations + discrete rotations), and whole steps at the
BASELINE bar (fields rel. L2 <= 1e-8, energy rel. <= 1e-10, mass drift <= 1e-12)."""
import numpy as np
import pytest

import nks_inputs as ni
from oracle import jacobian, scheme, solver

pytestmark = pytest.mark.gpu

MODEL = ni.model_default()
SOL = ni.solver_default()


def gpu(shape, pc_type=0):
    from paper_2209_08001_b200 import Solver
    return Solver(shape, MODEL, SOL, h=0.25, nsub=(1,) * len(shape), overlap=2, pc_type=pc_type, bc=1)


def omodel(d):
    return scheme.Model.from_dict(d, 0.25, MODEL, bc="neumann")


def states(shape, seed=0):
    d = len(shape)
    ca, ea = ni.initial_fields(shape, seed)
    ua = ni.random_displacement(d, shape, seed + 2, 1e-3)
    Xa = solver.gauge_project(np.concatenate([ca[None], ea[None], ua]), "neumann")
    cb, eb = ni.perturbed_state(ca, ea, seed + 1, 2e-3)
    Xb = np.concatenate([cb[None], eb[None], Xa[2:] + ni.random_displacement(d, shape, seed + 3, 1e-4)])
    return Xa, Xb


def rel(a, b):
    return [float(np.abs(a[f] - b[f]).max() / max(np.abs(b[f]).max(), 1e-300)) for f in range(a.shape[0])]


@pytest.mark.parametrize("shape", [(14, 18), (9, 7, 11), (6, 8, 8)])
def test_neumann_residual_jv_energy_parity(shape):
    d = len(shape)
    m = omodel(d)
    Xa, Xb = states(shape)
    g = gpu(shape)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    cbar = Xa[0].mean()
    for dt in (0.01, 1.3):
        Fg = g.eval_residual(Xb, dt).cpu().numpy()
        Fo = scheme.residual(m, Xa, Xb, dt, cbar)
        assert max(rel(Fg, Fo)) < 1e-12, rel(Fg, Fo)
        v = ni.random_direction(2 + d, shape, 7)
        Jg = g.eval_jv(Xb, v, dt).cpu().numpy()
        Jo = jacobian.jv(m, Xa, Xb, dt, v)
        assert max(rel(Jg, Jo)) < 1e-12, rel(Jg, Jo)
    parts, mass = g.energy()
    po = scheme.energy_parts(m, Xa, cbar)
    for a, b in zip(parts, po):
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12)
    assert mass == pytest.approx(scheme.mass(m, Xa), rel=1e-13)


@pytest.mark.parametrize("shape", [(12, 16), (11, 16), (6, 8, 6)])
def test_neumann_gauge(shape):
    """set_fields projects u onto the Neumann gauge exactly like the oracle: zero mean per component and
    no component along the discrete rotations of even-extent axis pairs."""
    d = len(shape)
    c, eta = ni.initial_fields(shape, 1)
    u = ni.random_displacement(d, shape, 4, 1e-2) + 0.3
    g = gpu(shape)
    g.set_fields(c, eta, u)
    Xg = g.get_state()
    Xo = solver.gauge_project(np.concatenate([c[None], eta[None], u]), "neumann")
    np.testing.assert_allclose(Xg[2:], Xo[2:], rtol=0, atol=1e-14)


@pytest.mark.parametrize("shape,pc,dts", [((8, 10), 0, [0.01]), ((16, 20), 5, [0.01, 0.5]),
                                          ((12, 14), 5, [0.01, 2.0]), ((6, 8, 8), 5, [0.01, 0.3])])
def test_neumann_step_parity(shape, pc, dts):
    """Whole NKS steps with Neumann boundaries (pc NONE or the spectral preconditioner) against the oracle's
    exact Newton with the gauge-pinned direct LU; u^0 from the oracle's pinned equilibrium solve.  (An odd
    extent leaves a near-null staircase mode under the mirror closure -- a direct solve is indifferent, an
    unpreconditioned Krylov solve stalls on it, in the oracle's GMRES as well -- so the Krylov cases here are
    the spectral preconditioner or tiny grids.)"""
    d = len(shape)
    m = omodel(d)
    c, eta = ni.initial_fields(shape, 0)
    cbar = c.mean()
    Xo = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
    g = gpu(shape, pc)
    g.set_fields(c, eta, Xo[2:])
    mass0 = scheme.mass(m, Xo)
    for dt in dts:
        Xo, info_o = solver.newton_step(m, Xo, dt, cbar, SOL)
        assert info_o["converged"]
        info_g = g.step(dt)
        Xg = g.get_state()
        r = [float(np.linalg.norm(Xg[f] - Xo[f]) / np.linalg.norm(Xo[f])) for f in range(2 + d)]
        assert max(r) <= 1e-8, (dt, r)
        assert info_g["energy"] == pytest.approx(scheme.energy(m, Xo, cbar), rel=1e-10)
        assert abs(info_g["mass"] - mass0) <= 1e-12 * abs(mass0)
        assert info_g["newton_its"] == info_o["newton_its"]


@pytest.mark.parametrize("shape", [(16, 20), (15, 12), (6, 8, 7)])
def test_neumann_u0_by_conjugate_gradients(shape):
    """Without u, a Neumann state solves u^0 by CG on its elastic block; it equals the oracle's gauge-pinned
    direct solve (R13, R38)."""
    d = len(shape)
    m = omodel(d)
    c, eta = ni.initial_fields(shape, 3)
    uo = solver.init_displacement(m, c, c.mean())
    g = gpu(shape)
    g.set_fields(c, eta, None)
    ug = g.get_state()[2:]
    for I in range(d):
        assert np.linalg.norm(ug[I] - uo[I]) <= 1e-10 * np.linalg.norm(uo[I])


@pytest.mark.parametrize("shape,nsub,delta,pc_type,variant", [((40, 36), (3, 2), 2, 2, "ras"), ((20, 24), (1, 1), 2, 2, "ras"),
                                                           ((9, 10, 11), (2, 1, 2), 1, 2, "ras"),
                                                           ((16, 18), (2, 2), 2, 3, "as")])
def test_neumann_schwarz_apply_parity(shape, nsub, delta, pc_type, variant):
    """Schwarz preconditioners on a Neumann grid: boxes stop at the walls, the box blocks come from probing J
    with 5^d colours (precond.cu), the 2D boxes run the pipelined apply -- against the oracle's Schwarz
    apply on the same clipped boxes."""
    from oracle import pc
    from paper_2209_08001_b200 import Solver
    d = len(shape)
    nf = 2 + d
    m = omodel(d)
    Xa, Xb = states(shape)
    dt = 0.3
    g = Solver(shape, MODEL, SOL, h=0.25, nsub=nsub, overlap=delta, pc_type=pc_type, bc=1)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = ni.random_direction(nf, shape, 14)
    zg = g.pc_apply(r).cpu().numpy()
    J = jacobian.assemble(m, Xa, Xb, dt)
    zo = pc.RAS(J, shape, nf, tuple(reversed(nsub)), delta, variant=variant, bc="neumann").apply(r)
    assert max(rel(zg, zo)) < 1e-10, rel(zg, zo)


@pytest.mark.parametrize("shape,nsub,dts", [((24, 20), (2, 2), [0.01, 0.5]), ((8, 8, 10), (1, 2, 2), [0.01, 0.2])])
def test_neumann_step_parity_with_ras(shape, nsub, dts):
    """Whole Neumann steps with the paper's preconditioner (left-RAS, BILU(0) boxes clipped at the walls)."""
    from paper_2209_08001_b200 import Solver
    d = len(shape)
    m = omodel(d)
    c, eta = ni.initial_fields(shape, 0)
    cbar = c.mean()
    Xo = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
    g = Solver(shape, MODEL, SOL, h=0.25, nsub=nsub, overlap=2, pc_type=2, bc=1)
    g.set_fields(c, eta, None)                   # u^0 by CG on the elastic block
    for dt in dts:
        Xo, info_o = solver.newton_step(m, Xo, dt, cbar, SOL)
        info_g = g.step(dt)
        Xg = g.get_state()
        r = [float(np.linalg.norm(Xg[f] - Xo[f]) / np.linalg.norm(Xo[f])) for f in range(2 + d)]
        assert max(r) <= 1e-8, (dt, r)
        assert info_g["energy"] == pytest.approx(scheme.energy(m, Xo, cbar), rel=1e-10)
