"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element.

Tolerances: pointwise operators (F, J.v, energy) are the same fp64
arithmetic in a different order -> 1e-12 relative to the field's max magnitude; solves are
compared at BASELINE.json's bar (fields rel. L2 <= 1e-8, energy rel. <= 1e-10, mass drift
<= 1e-12).
"""
import numpy as np
import pytest

import nks_inputs as ni
from oracle import jacobian, pc, scheme, solver

pytestmark = pytest.mark.gpu

MODEL = ni.model_default()
SOL = ni.solver_default()


def gpu_solver(shape, nsub=None, overlap=2, pc_type=2, **kw):
    from paper_2209_08001_b200 import Solver
    sol = dict(SOL)
    sol.update(kw.pop("sol", {}))
    return Solver(shape, MODEL, sol, h=0.25, nsub=nsub or (1,) * len(shape), overlap=overlap, pc_type=pc_type, **kw)


def oracle_model(d):
    return scheme.Model.from_dict(d, 0.25, MODEL)


def states(shape, seed=0, amp=2e-3):
    d = len(shape)
    ca, ea = ni.initial_fields(shape, seed)
    ua = ni.random_displacement(d, shape, seed + 2, 1e-3)
    Xa = np.concatenate([ca[None], ea[None], ua])
    cb, eb = ni.perturbed_state(ca, ea, seed + 1, amp)
    Xb = np.concatenate([cb[None], eb[None], ua + ni.random_displacement(d, shape, seed + 3, 1e-4)])
    return Xa, Xb


def field_rel_err(a, b):
    """max |a-b| / max |b| per field."""
    return [float(np.abs(a[f] - b[f]).max() / max(np.abs(b[f]).max(), 1e-300)) for f in range(a.shape[0])]


SHAPES = [(40, 36), (12, 20, 36), (64, 64), (9, 7, 11)]
# F / J.v only: 136 planes march in z chunks of 9 (launch heuristic for a one-tile plane), the last chunk a
# single plane -- the chunk prologue, the two-barrier pipeline and its tail on a ragged split
STENCIL_SHAPES = SHAPES + [(20, 12, 136)]


@pytest.mark.parametrize("shape", STENCIL_SHAPES)
def test_residual_parity(shape):
    d = len(shape)
    Xa, Xb = states(shape)
    g = gpu_solver(shape)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    cbar = Xa[0].mean()
    for dt in (0.01, 1.7):
        Fg = g.eval_residual(Xb, dt).cpu().numpy()
        Fo = scheme.residual(oracle_model(d), Xa, Xb, dt, cbar)
        errs = field_rel_err(Fg, Fo)
        assert max(errs) < 1e-12, errs


@pytest.mark.parametrize("shape", STENCIL_SHAPES)
def test_jv_parity(shape):
    d = len(shape)
    Xa, Xb = states(shape)
    v = ni.random_direction(2 + d, shape, 7)
    g = gpu_solver(shape)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    for dt in (0.01, 2.0):
        Jg = g.eval_jv(Xb, v, dt).cpu().numpy()
        Jo = jacobian.jv(oracle_model(d), Xa, Xb, dt, v)
        errs = field_rel_err(Jg, Jo)
        assert max(errs) < 1e-12, errs


@pytest.mark.parametrize("shape", [(40, 36), (12, 20, 36)])
def test_energy_and_mass_parity(shape):
    d = len(shape)
    Xa, _ = states(shape)
    g = gpu_solver(shape)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    parts, mass = g.energy()
    # the library projects u onto the canonical gauge; E3 is gauge invariant
    ref = scheme.energy_parts(oracle_model(d), Xa, Xa[0].mean())
    for a, b in zip(parts, ref):
        assert a == pytest.approx(b, rel=1e-12, abs=1e-12)
    assert mass == pytest.approx(scheme.mass(oracle_model(d), Xa), rel=1e-14)


@pytest.mark.parametrize("shape", [(64, 64), (36, 40), (8, 12, 10), (7, 9)])
def test_initial_displacement_and_gauge(shape):
    d = len(shape)
    c, eta = ni.initial_fields(shape, 3)
    g = gpu_solver(shape)
    g.set_fields(c, eta, None)
    X = g.get_state()
    uo = solver.init_displacement(oracle_model(d), c, c.mean())
    scale = np.abs(uo).max()
    assert np.abs(X[2:] - uo).max() <= 1e-10 * scale
    np.testing.assert_array_equal(X[0], c)


def test_set_fields_host_path_and_errors():
    from paper_2209_08001_b200 import NKSError
    shape = (16, 16)
    c, eta = ni.initial_fields(shape, 0)
    g = gpu_solver(shape)
    g.set_fields_host(c, eta)
    X = g.get_state()
    np.testing.assert_array_equal(X[1], eta)
    bad = eta.copy()
    bad[3, 4] = -0.2          # p = c*eta < 0: outside the domain of Psi
    with pytest.raises(NKSError):
        g.set_fields(c, bad)


# ---------------------------------------------------------------------------------------- preconditioner

PC_CASES = [((16, 16), (2, 2), 2), ((12, 14), (1, 1), 2), ((10, 13), (3, 2), 1), ((6, 7, 6), (1, 1, 2), 1),
            ((16, 16), (4, 4), 0)]


@pytest.mark.parametrize("shape,nsub,delta", PC_CASES)
def test_ras_bilu0_apply_parity(shape, nsub, delta):
    d = len(shape)
    nf = 2 + d
    Xa, Xb = states(shape)
    dt = 0.3
    g = gpu_solver(shape, nsub=nsub, overlap=delta)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = ni.random_direction(nf, shape, 11)
    zg = g.pc_apply(r).cpu().numpy()
    J = jacobian.assemble(oracle_model(d), Xa, Xb, dt)
    ras = pc.RAS(J, shape, nf, tuple(reversed(nsub)), delta)
    zo = ras.apply(r)
    errs = field_rel_err(zg, zo)
    assert max(errs) < 1e-10, errs


@pytest.mark.parametrize("variant", ["ras", "as"])
def test_ras3d_cluster_apply_parity(variant):
    """The 3D level-synchronous apply split over a cluster of 2 or 4 CTAs per box (precond.cu k_ras_apply_cl;
    nks_params.ras_cta_per_box forces it, auto picks it only for a strong-scaled rank's few boxes): against the
    oracle, and bit for bit equal to one CTA per box (same per-point summation order)."""
    from paper_2209_08001_b200 import PC_AS_BILU0, PC_RAS_BILU0
    shape, nsub, delta = (8, 10, 12), (1, 2, 2), 2
    nf = 5
    Xa, Xb = states(shape)
    dt = 0.3
    r = ni.random_direction(nf, shape, 13)
    pc_type = PC_RAS_BILU0 if variant == "ras" else PC_AS_BILU0
    out = {}
    for cta in (1, 2, 4):
        g = gpu_solver(shape, nsub=nsub, overlap=delta, pc_type=pc_type, sol={"ras_cta_per_box": cta})
        g.set_fields(Xa[0], Xa[1], Xa[2:])
        g.pc_setup(Xb, dt)
        out[cta] = g.pc_apply(r).cpu().numpy()
    J = jacobian.assemble(oracle_model(3), Xa, Xb, dt)
    zo = pc.RAS(J, shape, nf, tuple(reversed(nsub)), delta, variant=variant).apply(r)
    for cta in (1, 2, 4):
        assert max(field_rel_err(out[cta], zo)) < 1e-10, cta
    np.testing.assert_array_equal(out[2], out[1])
    np.testing.assert_array_equal(out[4], out[1])


@pytest.mark.parametrize("shape,nsub,delta", [((96, 80), (3, 2), 2), ((70, 130), (1, 2), 1), ((256, 40), (2, 1), 2)])
def test_ras2d_apply_parity(shape, nsub, delta):
    """The 2D RAS apply (ras2d_rows.cu: one lane per row, four component warps, a cluster of stripes per
    box) against the oracle's left-RAS on boxes of several stripes with ragged stripe heights, including
    132-row boxes (the config-2 box height) split over a full cluster."""
    nf = 4
    Xa, Xb = states(shape)
    dt = 0.3
    g = gpu_solver(shape, nsub=nsub, overlap=delta)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = ni.random_direction(nf, shape, 12)
    zg = g.pc_apply(r).cpu().numpy()
    J = jacobian.assemble(oracle_model(2), Xa, Xb, dt)
    zo = pc.RAS(J, shape, nf, tuple(reversed(nsub)), delta).apply(r)
    errs = field_rel_err(zg, zo)
    assert max(errs) < 1e-10, errs


SCHWARZ_CASES = [((16, 16), (2, 2), 2, "as"), ((16, 16), (2, 2), 2, "rras"), ((12, 14), (1, 1), 2, "as"),
                 ((10, 13), (3, 2), 1, "rras"), ((6, 7, 6), (1, 1, 2), 1, "as"), ((6, 7, 6), (2, 1, 1), 1, "rras")]


@pytest.mark.parametrize("shape,nsub,delta,variant", SCHWARZ_CASES)
def test_schwarz_variant_apply_parity(shape, nsub, delta, variant):
    """Classical AS and right-restricted AS against the oracle's Schwarz apply; the
    overlapping boxes' sums include a periodic self-overlapping box (nsub = 1 along an axis)."""
    from paper_2209_08001_b200 import PC_AS_BILU0, PC_RRAS_BILU0
    d = len(shape)
    nf = 2 + d
    Xa, Xb = states(shape)
    dt = 0.3
    g = gpu_solver(shape, nsub=nsub, overlap=delta, pc_type=PC_AS_BILU0 if variant == "as" else PC_RRAS_BILU0)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = ni.random_direction(nf, shape, 11)
    zg = g.pc_apply(r).cpu().numpy()
    J = jacobian.assemble(oracle_model(d), Xa, Xb, dt)
    zo = pc.RAS(J, shape, nf, tuple(reversed(nsub)), delta, variant=variant).apply(r)
    errs = field_rel_err(zg, zo)
    assert max(errs) < 1e-10, errs


@pytest.mark.parametrize("variant", ["as", "rras"])
def test_schwarz_variant_step_parity(variant):
    """A whole NKS step preconditioned by AS / RRAS: the same converged step as the oracle."""
    from paper_2209_08001_b200 import PC_AS_BILU0, PC_RRAS_BILU0
    _run_parity((16, 16), [0.5], (2, 2), 2, pc_type=PC_AS_BILU0 if variant == "as" else PC_RRAS_BILU0)


@pytest.mark.parametrize("shape,nsub", [((24, 24), (2, 2)), ((8, 8, 8), (2, 1, 1))])
def test_gmres_solves_the_newton_system(shape, nsub):
    d = len(shape)
    Xa, Xb = states(shape)
    dt = 0.5
    m = oracle_model(d)
    Fo = scheme.residual(m, Xa, Xb, dt, Xa[0].mean())
    g = gpu_solver(shape, nsub=nsub, sol={"gmres_rtol": 1e-12})
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    s, its = g.gmres_solve(Xb, -Fo, dt)
    s = s.cpu().numpy()
    J = jacobian.assemble(m, Xa, Xb, dt)
    res = J @ s.ravel() + Fo.ravel()
    assert np.linalg.norm(res) <= 1e-11 * np.linalg.norm(Fo)
    # the same Newton direction as the oracle's pinned direct solve (up to the gauge null space)
    import scipy.sparse.linalg as spla
    A, b = solver.pin(J, -Fo.ravel(), solver.pinned_rows(shape, d))
    so = spla.spsolve(A, b).reshape(s.shape)
    sg = solver.gauge_project(s)
    so = solver.gauge_project(so)
    for f in range(2 + d):
        assert np.linalg.norm(sg[f] - so[f]) <= 1e-8 * np.linalg.norm(so[f]) + 1e-14
    assert its < 200


# ---------------------------------------------------------------------------------------- time steps

def _run_parity(shape, dts, nsub, delta, seed=0, pc_type=2, fp32=False, sol=None):
    d = len(shape)
    m = oracle_model(d)
    c, eta = ni.initial_fields(shape, seed)
    cbar = c.mean()
    u0 = solver.init_displacement(m, c, cbar)
    Xo = np.concatenate([c[None], eta[None], u0])
    g = gpu_solver(shape, nsub=nsub, overlap=delta, pc_type=pc_type, sol=dict({"factor_fp32": int(fp32)}, **(sol or {})))
    g.set_fields(c, eta, None)          # the library solves its own u^0 (FFT)
    mass0 = scheme.mass(m, Xo)
    out = []
    for dt in dts:
        Xo, info_o = solver.newton_step(m, Xo, dt, cbar, SOL)
        assert info_o["converged"]
        info_g = g.step(dt)
        Xg = g.get_state()
        rel = [float(np.linalg.norm(Xg[f] - Xo[f]) / np.linalg.norm(Xo[f])) for f in range(2 + d)]
        e_o = scheme.energy(m, Xo, cbar)
        assert max(rel) <= 1e-8, (dt, rel)
        assert info_g["energy"] == pytest.approx(e_o, rel=1e-10)
        assert abs(info_g["mass"] - mass0) <= 1e-12 * abs(mass0)
        out.append((info_g, info_o, rel))
    return out


def test_step_parity_config1():
    """BASELINE config 1: 2D 64x64, fixed dt = 0.01, 10 steps, one self-overlapping subdomain, delta = 2."""
    cfg = ni.CONFIGS[1]
    out = _run_parity(cfg["shape"], [cfg["dt"]] * cfg["steps"], cfg["nsub"], cfg["overlap"])
    e = [o[0]["energy"] for o in out]
    assert all(e[k + 1] <= e[k] + 1e-10 for k in range(len(e) - 1))


@pytest.mark.parametrize("dts", [[0.5, 0.5], [2.0]])
def test_step_parity_large_dt(dts):
    _run_parity((32, 32), dts, (2, 2), 2)


def test_bilu0_breakdown_is_reported_as_divergence():
    """At dt = 2 after one dt = 2 step (eta ~ 0.3) J is indefinite and BILU(0)-RAS is unstable: GMRES
    stagnates (the oracle's own RAS/BILU(0) + GMRES(30) stalls at 0.97 relative residual on the same
    matrix, while exact subdomain LU converges in 48 iterations).  The library must stop early
    (stagnation rule, R18), report DIVERGED and leave X^n unchanged -- the adaptive
    controller then retries with dt/sqrt(2)."""
    shape = (32, 32)
    c, eta = ni.initial_fields(shape, 0)
    g = gpu_solver(shape, nsub=(2, 2), sol={"gmres_stall_cycles": 3})
    g.set_fields(c, eta, None)
    assert g.step(2.0)["converged"]
    X0 = g.get_state()
    info = g.step(2.0, raise_on_fail=False)
    assert info["status"] == "DIVERGED" and info["reason"] in ("gmres_stagnation", "gmres_projected"), info
    assert info["gmres_its"] < 1000
    np.testing.assert_array_equal(g.get_state(), X0)


def test_early_divergence_rule_keeps_the_controllers_decisions():
    """The opt-in early-divergence rule (gmres_stall_cycles = 3, R18) must only cut work: from the
    state after three adaptive steps at 128^2 (4x4 boxes, BILU(0)), every forced attempt has the same outcome
    as with the rule off (the paper's solver, which fails only at gmres_maxit): the accepted ones bit for bit
    (same GMRES count, same fields), the rejected ones earlier than at gmres_maxit."""
    shape = (128, 128)
    c, eta = ni.initial_fields(shape, 0)
    on = gpu_solver(shape, nsub=(4, 4), sol={"gmres_stall_cycles": 3})
    off = gpu_solver(shape, nsub=(4, 4), sol={"gmres_stall_cycles": 0})
    on.set_fields(c, eta, None)
    off.set_fields(c, eta, None)          # same cbar0; nks_set_state needs fields set once
    on.run_adaptive(3)
    X = on.get_state()
    outcomes = []
    for dt in (0.986, 1.414, 2.0):
        res = []
        for g in (on, off):
            g.set_state(X[0], X[1], X[2:])
            info = g.step(dt, raise_on_fail=False)
            res.append((info, g.get_state()))
        (i_on, X_on), (i_off, X_off) = res
        assert i_on["status"] == i_off["status"], (dt, i_on, i_off)
        if i_off["status"] == "OK":
            assert i_on["gmres_its"] == i_off["gmres_its"]
            np.testing.assert_array_equal(X_on, X_off)
        else:
            assert i_off["reason"] == "gmres_maxit" and i_on["reason"] in ("gmres_stagnation", "gmres_projected")
            assert i_on["gmres_its"] < i_off["gmres_its"]
        outcomes.append(i_off["status"])
    assert "OK" in outcomes and "DIVERGED" in outcomes, outcomes     # both branches exercised


def test_step_parity_3d():
    _run_parity((10, 12, 12), [0.01, 0.3], (1, 2, 2), 2)


def test_step_parity_no_preconditioner():
    _run_parity((16, 16), [0.01], (1, 1), 0, pc_type=0)


def test_adaptive_run_parity():
    """nks_run_adaptive vs the oracle controller on a 2D 32x32 grid."""
    shape = (32, 32)
    d = 2
    m = oracle_model(d)
    c, eta = ni.initial_fields(shape, 1)
    cbar = c.mean()
    Xo = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
    Xo, recs_o = solver.run_adaptive(m, Xo, cbar, SOL, 6)
    g = gpu_solver(shape, nsub=(2, 2))
    g.set_fields(c, eta, None)
    recs_g = g.run_adaptive(6)
    assert len(recs_g) == 6
    for rg, ro in zip(recs_g, recs_o):
        assert rg["dt"] == pytest.approx(ro["dt"], rel=1e-9)
        assert rg["energy"] == pytest.approx(ro["energy"], rel=1e-10)
        assert rg["retries"] == ro["retries"]
    Xg = g.get_state()
    for f in range(4):
        assert np.linalg.norm(Xg[f] - Xo[f]) <= 1e-8 * np.linalg.norm(Xo[f])


def test_step_failure_is_transactional():
    """A step that cannot converge (newton_maxit = 0) leaves X^n unchanged and reports DIVERGED."""
    shape = (16, 16)
    c, eta = ni.initial_fields(shape, 0)
    g = gpu_solver(shape, sol={"newton_maxit": 0})
    g.set_fields(c, eta, None)
    X0 = g.get_state()
    info = g.step(0.5, raise_on_fail=False)
    assert info["status"] == "DIVERGED" and info["reason"] == "newton_maxit"
    np.testing.assert_array_equal(g.get_state(), X0)


# ---------------------------------------------------------------------------------------- full-size sampled parity

def _window(X, centre, r):
    """Periodic window of radius r around centre (C-order index tuple), shape (nf, 2r+1, ...)."""
    idx = [np.arange(c - r, c + r + 1) % n for c, n in zip(centre, X.shape[1:])]
    return X[(slice(None),) + np.ix_(*idx)]


@pytest.mark.parametrize("cfg_id", [2, 3])
def test_full_size_sampled_residual_and_jv(cfg_id):
    """At BASELINE sizes: F and J.v are radius-2 stencils, so the oracle evaluated on a periodic
    9^d window reproduces the exact value at the window centre; compare 64 sampled points."""
    shape = ni.CONFIGS[cfg_id]["shape"]
    d = len(shape)
    m = oracle_model(d)
    c, eta = ni.initial_fields(shape, 0)
    cbar = c.mean()
    u0 = solver.init_displacement_fft(m, c, cbar)          # oracle-side u^0 (inputs never come from the GPU)
    Xa = np.concatenate([c[None], eta[None], u0])
    g = gpu_solver(shape, pc_type=0)
    g.set_fields(c, eta, u0)
    cb, eb = ni.perturbed_state(c, eta, 1, 1e-3)
    Xb = Xa.copy()
    Xb[0], Xb[1] = cb, eb
    v = ni.random_direction(2 + d, shape, 5)
    dt = 0.01
    F = g.eval_residual(Xb, dt).cpu().numpy()
    Jv = g.eval_jv(Xb, v, dt).cpu().numpy()
    rng = np.random.default_rng(9)
    r = 4
    for _ in range(64):
        ctr = tuple(int(rng.integers(0, n)) for n in shape)
        wa, wb, wv = _window(Xa, ctr, r), _window(Xb, ctr, r), _window(v, ctr, r)
        Fo = scheme.residual(m, wa, wb, dt, cbar)[(slice(None),) + (r,) * d]
        Jo = jacobian.jv(m, wa, wb, dt, wv)[(slice(None),) + (r,) * d]
        Fg = F[(slice(None),) + ctr]
        Jg = Jv[(slice(None),) + ctr]
        np.testing.assert_allclose(Fg, Fo, rtol=1e-11, atol=1e-11 * np.abs(F).max(axis=tuple(range(1, d + 1))).max())
        np.testing.assert_allclose(Jg, Jo, rtol=1e-11, atol=1e-11 * np.abs(Jv).max())


# ---------------------------------------------------------------------------------------- second workload

@pytest.mark.parametrize("Lscale", [3.0])
def test_single_particle_workload_parity(Lscale):
    """the paper's single-particle initial state (a sphere with c = 0.238,
    eta = 0.01 inside and c = 0.1375, eta = 0.99 outside), here r = 1 on a 3D 10^3 grid, with the
    paper's elastic multiplier script-L = 3 (the 80^3 run with script-L = 1 is tools/single_particle.py); two adaptive steps, GPU vs
    oracle.  (script-L = 0 leaves u undetermined -- all u rows vanish -- so it is not a case of the
    coupled system as formulated here.)"""
    shape = (10, 10, 10)
    d = 3
    model = dict(MODEL)
    model["Lscale"] = Lscale
    m = scheme.Model.from_dict(d, 0.25, model)
    c, eta = ni.sphere_fields(shape, 0.25, 1.0, 0.238, 0.01, 0.1375, 0.99)
    cbar = c.mean()
    Xo = np.concatenate([c[None], eta[None], solver.init_displacement(m, c, cbar)])
    Xo, recs_o = solver.run_adaptive(m, Xo, cbar, SOL, 2)
    from paper_2209_08001_b200 import Solver
    g = Solver(shape, model, SOL, h=0.25, nsub=(1, 2, 2), overlap=2)
    g.set_fields(c, eta, None)
    recs_g = g.run_adaptive(2)
    for rg, ro in zip(recs_g, recs_o):
        assert rg["dt"] == pytest.approx(ro["dt"], rel=1e-9)
        assert rg["energy"] == pytest.approx(ro["energy"], rel=1e-10)
    Xg = g.get_state()
    for f in range(2 + d):
        nrm = np.linalg.norm(Xo[f])
        if nrm > 0:
            assert np.linalg.norm(Xg[f] - Xo[f]) <= 1e-8 * nrm, f
        else:
            assert np.abs(Xg[f]).max() == 0.0


def test_fp32_factors_change_iterations_not_the_step():
    """factor_fp32: the level-synchronous subdomain solves read fp32 copies of the
    BILU(0) factors.  The preconditioner only steers GMRES, so the accepted step still matches the
    oracle at BASELINE's bar, and the apply itself stays within fp32 rounding of the fp64 apply."""
    shape = (10, 12, 12)
    out = _run_parity(shape, [0.01, 0.3], (1, 2, 2), 2, fp32=True)
    assert len(out) == 2
    Xa, Xb = states(shape)
    r = ni.random_direction(5, shape, 11)
    z = []
    for f32 in (0, 1):
        g = gpu_solver(shape, nsub=(1, 2, 2), overlap=2, sol={"factor_fp32": f32})
        g.set_fields(Xa[0], Xa[1], Xa[2:])
        g.pc_setup(Xb, 0.3)
        z.append(g.pc_apply(r).cpu().numpy())
    rel = np.abs(z[1] - z[0]).max() / np.abs(z[0]).max()
    assert 0 < rel < 1e-4, rel


PCI_CASES = [((1, 1), 2, 1, 0), ((4, 4), 2, 1, 0), ((4, 4), 0, 1, 0), ((4, 4), 2, 0, 0), ((4, 4), 2, 2, 0),
             ((4, 4), 2, 1, 1), ((2, 4), 1, 2, 1)]


@pytest.mark.parametrize("nsub,overlap,reuse,fp32", PCI_CASES)
def test_preconditioner_independence(nsub, overlap, reuse, fp32):
    """SURVEY 8(c).3 'preconditioner independence' (the Newton solve is insensitive to the
    subdomain solver): two steps of the same dt (so pc_reuse = 2 keeps the factors across steps) with
    different box counts, overlaps, factorisation reuse and factor precision reach the same X^{n+1}
    as the single-box reference to 1e-10 relative, with the same Newton counts (+-1 at the tolerance)."""
    shape = (32, 32)
    c, eta = ni.initial_fields(shape, 0)
    dts = [0.3, 0.3]

    def run(nsub_, ov_, reuse_, f32_):
        g = gpu_solver(shape, nsub=nsub_, overlap=ov_, pc_reuse=reuse_,
                       sol={"factor_fp32": f32_, "gmres_maxit": 6000})
        g.set_fields(c, eta)
        infos = [g.step(dt) for dt in dts]
        return g.get_state(), infos

    X0, i0 = run((1, 1), 2, 1, 0)
    X1, i1 = run(nsub, overlap, reuse, fp32)
    for f in range(X0.shape[0]):
        rel = np.linalg.norm(X1[f] - X0[f]) / np.linalg.norm(X0[f])
        assert rel <= 1e-10, (f, rel)
    for a, b in zip(i0, i1):
        assert abs(a["newton_its"] - b["newton_its"]) <= 1, (a["newton_its"], b["newton_its"])
        assert abs(a["energy"] - b["energy"]) <= 1e-10 * abs(a["energy"])


# ---------------------------------------------------------------------------------------- ILU(k) / LU
ILUK_CASES = [((16, 16), (2, 2), 2, 1), ((16, 16), (2, 2), 2, 2), ((12, 14), (2, 1), 1, -1), ((14, 12), (1, 1), 2, 1),
              ((6, 7, 6), (1, 1, 2), 1, 1), ((6, 6, 6), (2, 1, 1), 1, -1)]


@pytest.mark.parametrize("shape,nsub,delta,level", ILUK_CASES)
def test_iluk_apply_parity(shape, nsub, delta, level):
    """RAS with ILU(1), ILU(2) and exact block LU box solves (ilu_level = k, -1) against the oracle's
    level-of-fill ILU(k) (oracle/pc.py: biluk, pinned by the fill-path theorem and L U = A)."""
    d = len(shape)
    nf = 2 + d
    Xa, Xb = states(shape)
    dt = 0.3
    g = gpu_solver(shape, nsub=nsub, overlap=delta, sol={"ilu_level": level})
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = ni.random_direction(nf, shape, 13)
    zg = g.pc_apply(r).cpu().numpy()
    J = jacobian.assemble(oracle_model(d), Xa, Xb, dt)
    zo = pc.RAS(J, shape, nf, tuple(reversed(nsub)), delta, fill=None if level < 0 else level).apply(r)
    errs = field_rel_err(zg, zo)
    assert max(errs) < 1e-10, errs


@pytest.mark.parametrize("level", [1, 2, -1])
def test_iluk_step_parity_and_fewer_iterations(level):
    """A step with ILU(k) / LU subdomain solves reaches the oracle's root; more fill never needs more GMRES
    iterations than ILU(0) here (Table 1 trend)."""
    shape, dts = (24, 24), [0.5]
    its = {}
    for lv in (0, level):
        out = _run_parity(shape, dts, (2, 2), 2, sol={"ilu_level": lv})
        its[lv] = out[0][0]["gmres_its"]
    assert its[level] <= its[0], its


def test_one_reduction_per_gmres_iteration():
    """DCGS2 Arnoldi (north_star item 5): one global reduction per GMRES iteration, plus one per restart
    cycle closing and per true-residual check (nks_counters)."""
    shape = (32, 32)
    Xa, Xb = states(shape)
    g = gpu_solver(shape, nsub=(2, 2), sol={"gmres_restart": 10})
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    rhs = solver.gauge_project(ni.random_direction(4, shape, 5))     # consistent: no left-null-space part
    r0 = g.counters()["reductions"]
    s, its = g.gmres_solve(Xb, rhs, 0.3)
    red = g.counters()["reductions"] - r0
    cycles = (its + 9) // 10
    assert its > 10
    assert its <= red <= its + 2 * cycles + 2, (its, red, cycles)


# ---------------------------------------------------------------------------------------- spectral preconditioner
@pytest.mark.parametrize("shape,dt", [((32, 24), 0.3), ((8, 10, 12), 0.05), ((33, 17), 2.0)])
def test_spectral_pc_apply_parity(shape, dt):
    """NKS_PC_SPECTRAL (cuFFT + per-wave-number inverse of the mean-coefficient Jacobian) against the
    oracle's SpectralPC (numpy FFT; pinned as the exact inverse of J at a uniform state)."""
    from oracle import krylov
    d = len(shape)
    nf = 2 + d
    Xa, Xb = states(shape)
    g = gpu_solver(shape, pc_type=5)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = solver.gauge_project(ni.random_direction(nf, shape, 21))
    zg = g.pc_apply(r).cpu().numpy()
    zo = krylov.SpectralPC(krylov.Linearisation(oracle_model(d), Xa, Xb, dt)).apply(r)
    errs = field_rel_err(zg, zo)
    assert max(errs) < 1e-11, errs


@pytest.mark.parametrize("shape,dts", [((48, 40), [0.01, 0.5, 2.0]), ((10, 12, 8), [0.01, 0.3])])
def test_spectral_pc_step_parity(shape, dts):
    """Full steps with the spectral preconditioner reach the oracle's root (the preconditioner only steers
    GMRES), with far fewer GMRES iterations than the one-level Schwarz method."""
    out = _run_parity(shape, dts, (1,) * len(shape), 2, pc_type=5)
    for info_g, _, _ in out:
        assert info_g["gmres_its"] <= 30 * info_g["newton_its"], info_g


@pytest.mark.parametrize("shape,nsub,dt", [((32, 24), (2, 2), 0.3), ((8, 10, 12), (2, 1, 2), 0.05)])
def test_two_level_pc_apply_parity(shape, nsub, dt):
    """NKS_PC_RAS_SPECTRAL: z = S r + RAS(r - J S r), the spectral global correction followed by left-RAS /
    BILU(0) on the remaining residual, against the same composition of the oracle's pieces."""
    from oracle import krylov
    d = len(shape)
    nf = 2 + d
    Xa, Xb = states(shape)
    g = gpu_solver(shape, nsub=nsub, overlap=2, pc_type=6)
    g.set_fields(Xa[0], Xa[1], Xa[2:])
    g.pc_setup(Xb, dt)
    r = solver.gauge_project(ni.random_direction(nf, shape, 23))
    zg = g.pc_apply(r).cpu().numpy()
    m = oracle_model(d)
    lin = krylov.Linearisation(m, Xa, Xb, dt)
    z1 = krylov.SpectralPC(lin).apply(r)
    J = jacobian.assemble(m, Xa, Xb, dt)
    z2 = pc.RAS(J, shape, nf, tuple(reversed(nsub)), 2).apply(r - lin.jv(z1))
    errs = field_rel_err(zg, z1 + z2)
    assert max(errs) < 1e-10, errs


def test_two_level_pc_step_parity():
    out = _run_parity((48, 40), [0.01, 0.5], (2, 2), 2, pc_type=6)
    for info_g, _, _ in out:
        assert info_g["gmres_its"] <= 40 * info_g["newton_its"], info_g


@pytest.mark.parametrize("shape", [(64, 48), (16, 12, 20), (11, 13)])
def test_u0_conjugate_gradients_match_fft(shape):
    """u^0 by conjugate gradients on the elastic block (the z-slab / Neumann path, forced here with
    u0_cg = 1) equals the FFT equilibrium in the canonical gauge (reading R13/R14)."""
    c, eta = ni.initial_fields(shape, 2)
    g1 = gpu_solver(shape, pc_type=0)
    g1.set_fields(c, eta, None)
    g2 = gpu_solver(shape, pc_type=0, sol={"u0_cg": 1})
    g2.set_fields(c, eta, None)
    u1, u2 = g1.get_state()[2:], g2.get_state()[2:]
    for I in range(len(shape)):
        assert np.linalg.norm(u2[I] - u1[I]) <= 1e-10 * np.linalg.norm(u1[I])
