"""Pins of oracle/jacobian.py, oracle/solver.py and oracle/pc.py (no GPU)."""
import math

import numpy as np
import pytest
import scipy.sparse.linalg as spla

import nks_inputs as ni
from oracle import jacobian, pc, scheme, solver

SOL = ni.solver_default()


def model(d=2, **over):
    p = ni.model_default()
    p.update(over)
    return scheme.Model.from_dict(d, 0.25, p)


def state(d, shape, seed=0, amp=1e-2, equilibrium=True):
    m = model(d)
    ca, ea = ni.initial_fields(shape, seed)
    cbar = ca.mean()
    ua = solver.init_displacement(m, ca, cbar) if equilibrium else ni.random_displacement(d, shape, seed + 2)
    Xa = np.concatenate([ca[None], ea[None], ua])
    cb, eb = ni.perturbed_state(ca, ea, seed + 1, amp)
    Xb = np.concatenate([cb[None], eb[None], ua + ni.random_displacement(d, shape, seed + 3, 1e-4)])
    return m, Xa, Xb, cbar


# ----------------------------------------------------------------------------- Jacobian

@pytest.mark.parametrize("d,shape", [(2, (8, 10)), (3, (5, 6, 5))])
def test_jacobian_vs_complex_step_and_fd(d, shape):
    m, Xa, Xb, cbar = state(d, shape)
    v = ni.random_direction(2 + d, shape, 9)
    ja = jacobian.jv(m, Xa, Xb, 0.05, v)
    jc = jacobian.jv_complex_step(m, Xa, Xb, 0.05, cbar, v)
    jf = jacobian.jv_central_fd(m, Xa, Xb, 0.05, cbar, v)
    scale = np.linalg.norm(jc)
    assert np.linalg.norm(ja - jc) <= 1e-13 * scale
    assert np.linalg.norm(jf - jc) <= 1e-6 * scale          # BASELINE: FD agreement 1e-6


@pytest.mark.parametrize("shape,expect", [((6, 6), 8), ((5, 5), 2), ((6, 5), 4)])
def test_elastic_operator_null_space(shape, expect):
    """Central-difference elasticity on a periodic grid: nullity d*2^(#even axes) (reading R14)."""
    m = model(2)
    Auu, _ = solver.elastic_block(m, shape)
    s = np.linalg.svd(Auu.toarray(), compute_uv=False)
    assert int(np.sum(s < 1e-9 * s[0])) == expect
    np.testing.assert_allclose(Auu.toarray(), Auu.toarray().T, atol=1e-9)


def test_elastic_null_space_3d():
    m = model(3)
    Auu, _ = solver.elastic_block(m, (4, 4, 4))
    s = np.linalg.svd(Auu.toarray(), compute_uv=False)
    assert int(np.sum(s < 1e-9 * s[0])) == 24


def test_full_jacobian_nullity_2d():
    m, Xa, Xb, cbar = state(2, (8, 8))
    J = jacobian.assemble(m, Xa, Xb, 0.01).toarray()
    s = np.linalg.svd(J, compute_uv=False)
    assert int(np.sum(s < 1e-10 * s[0])) == 8          # d * 2^d
    # pinned matrix is nonsingular
    A, _ = solver.pin(jacobian.assemble(m, Xa, Xb, 0.01), np.zeros(J.shape[0]), solver.pinned_rows((8, 8), 2))
    s2 = np.linalg.svd(A.toarray(), compute_uv=False)
    assert s2[-1] > 1e-10 * s2[0]


# ----------------------------------------------------------------------------- u^0 (reading R13)

@pytest.mark.parametrize("d,shape", [(2, (10, 12)), (3, (6, 4, 6)), (2, (7, 8))])
def test_init_displacement_lu_equals_fft(d, shape):
    m = model(d)
    c, _ = ni.initial_fields(shape, 3)
    u1 = solver.init_displacement(m, c, c.mean())
    u2 = solver.init_displacement_fft(m, c, c.mean())
    if all(n % 2 == 0 for n in shape):
        np.testing.assert_allclose(u1, u2, atol=1e-14 + 1e-10 * np.abs(u1).max())
    X = np.concatenate([c[None], c[None] * 0 + 0.1, u1])
    F = scheme.residual(m, X, X, 1.0, c.mean())
    assert np.abs(F[2:]).max() < 1e-9 * m.C11 * m.eps0


# ----------------------------------------------------------------------------- Newton

def test_newton_quadratic_convergence():
    m, Xa, _, cbar = state(2, (12, 12))
    Xn, info = solver.newton_step(m, Xa, 0.5, cbar, SOL)
    assert info["converged"]
    h = info["hist"]
    for k in range(1, len(h) - 1):
        if h[k] > 1e-8 * h[0]:
            assert h[k + 1] <= 50.0 * h[k] ** 2 / h[0] + 1e-12 * h[0]


def test_newton_dense_lu_agrees_with_sparse():
    """A dense LU on the pinned matrix (2D 8x8, 256 unknowns) gives the same step."""
    m, Xa, _, cbar = state(2, (8, 8))
    J = jacobian.assemble(m, Xa, Xa, 0.1)
    F = scheme.residual(m, Xa, Xa, 0.1, cbar).ravel()
    A, b = solver.pin(J, -F, solver.pinned_rows((8, 8), 2))
    s_sparse = spla.spsolve(A, b)
    s_dense = np.linalg.solve(A.toarray(), b)
    np.testing.assert_allclose(s_sparse, s_dense, rtol=1e-10, atol=1e-13 * np.abs(s_dense).max())
    # the dropped (pinned) equations are redundant: the full system holds
    assert np.linalg.norm(J @ s_dense + F) <= 1e-10 * np.linalg.norm(F)


@pytest.mark.parametrize("dt", [0.01, 0.5, 2.0])
def test_newton_mass_and_energy_laws(dt):
    """Thm 3.2: mass conserved; energy non-increasing (within the R^S term)."""
    m, Xa, _, cbar = state(2, (12, 12))
    Xn, info = solver.newton_step(m, Xa, dt, cbar, SOL)
    assert info["converged"]
    ma, mb = scheme.mass(m, Xa), scheme.mass(m, Xn)
    assert abs(mb - ma) <= 1e-12 * abs(ma)
    assert scheme.energy(m, Xn, cbar) <= scheme.energy(m, Xa, cbar) + 1e-10


def test_dissipation_identity():
    """E^b - E^a = -dt h^d [sum_faces M~ (D^+ G^S_c)^2 + sum (G^S_eta)^2] + <(G - G^S).dV>."""
    m, Xa, _, cbar = state(2, (10, 10))
    dt = 0.2
    Xb, info = solver.newton_step(m, Xa, dt, cbar, SOL)
    assert info["converged"]
    gc, ge = scheme.G_S(m, Xa, Xb, cbar)
    vol = m.h ** 2
    diss = sum(np.sum(scheme.mobility_face(Xa[0], m.kappa, j, 2) * scheme.D_plus(gc, j, m.h, 2) ** 2)
               for j in range(2)) + np.sum(ge ** 2)
    g2e = scheme.G2_exact(m, Xa[0], Xb[0], Xa[1], Xb[1])
    g2s = scheme.G2S(m, Xa[0], Xb[0], Xa[1], Xb[1])
    rs = vol * np.sum((g2e[0] - g2s[0]) * (Xb[0] - Xa[0]) + (g2e[1] - g2s[1]) * (Xb[1] - Xa[1]))
    lhs = scheme.energy(m, Xb, cbar) - scheme.energy(m, Xa, cbar)
    rhs = -dt * vol * diss + rs
    assert lhs == pytest.approx(rhs, rel=1e-7, abs=1e-9)


def test_gauge_projection():
    X = np.random.default_rng(0).normal(size=(4, 6, 8))
    Y = solver.gauge_project(X)
    ids, ncls = solver.sublattice_ids((6, 8))
    assert ncls == 4
    for I in (2, 3):
        for k in range(ncls):
            assert abs(Y[I][ids == k].mean()) < 1e-15
    np.testing.assert_array_equal(Y[:2], X[:2])


# ----------------------------------------------------------------------------- controller

def test_controller_closed_forms():
    assert solver.predict_dt(0.0, 100, 0.01, 2.0) == 2.0
    assert solver.predict_dt(10.0, 100, 0.01, 2.0) == pytest.approx(2 / math.sqrt(10001), rel=1e-15)
    assert solver.predict_dt(1e6, 100, 0.01, 2.0) == 0.01
    Xn = np.ones((4, 2, 2))
    Xp = np.zeros((4, 2, 2))
    assert solver.change_rate(Xn, Xp, 0.5, "rms") == pytest.approx(2.0)
    assert solver.change_rate(Xn, Xp, 0.5, "l2") == pytest.approx(math.sqrt(16) / 0.5)


def test_run_adaptive_small():
    m, Xa, _, cbar = state(2, (8, 8))
    X, recs = solver.run_adaptive(m, Xa, cbar, SOL, 4)
    assert recs[0]["dt"] == SOL["dt_init"]
    for r in recs:
        assert r["converged"]
        assert r["mass"] == pytest.approx(recs[0]["mass"], rel=1e-12)
    e = [r["energy"] for r in recs]
    assert all(e[i + 1] <= e[i] + 1e-10 for i in range(len(e) - 1))
    assert recs[1]["dt"] >= SOL["dt_min"]


# ----------------------------------------------------------------------------- RAS / BILU(0)

def test_footprint_sizes():
    assert len(pc.footprint(2)) == 13 and len(pc.footprint(3)) == 25


def test_boxes_partition_of_unity():
    shape = (10, 12)
    bx = pc.boxes(shape, (3, 2), 2)
    owned = np.zeros(120, dtype=int)
    for b in bx:
        for l in pc.local_points(b):
            if pc.is_owned(b, l):
                owned[pc.global_index(b, l)] += 1
    assert np.all(owned == 1)


def test_bilu0_defining_property():
    """(L U)_pq = A_pq for every (p, q) on the block pattern (definition of ILU(0))."""
    m, Xa, Xb, cbar = state(2, (8, 8))
    J = jacobian.assemble(m, Xa, Xb, 0.1)
    b = pc.boxes((8, 8), (2, 2), 1)[0]
    A, pts = pc.box_blocks(J, b, 4, 64)
    L, U = pc.bilu0(A, len(pts))
    n = len(pts)
    for (p, q), blk in A.items():
        acc = np.zeros((4, 4))
        for k in range(min(p, q) + 1):
            lpk = np.eye(4) if k == p else L.get((p, k))
            ukq = U.get((k, q))
            if lpk is not None and ukq is not None:
                acc += lpk @ ukq
        np.testing.assert_allclose(acc, blk, rtol=1e-10, atol=1e-10 * np.abs(blk).max() + 1e-12)
    assert n == 36


def test_bilu0_is_exact_on_a_line():
    """A one-row box: the 13-point pattern is banded with no fill, so ILU(0) = exact LU."""
    m, Xa, Xb, cbar = state(2, (8, 16))
    J = jacobian.assemble(m, Xa, Xb, 0.1)
    b = {"start": [3, 2], "own": [6, 1], "ext": [6, 1], "delta": 0, "n": [16, 8]}
    A, pts = pc.box_blocks(J, b, 4, 128)
    L, U = pc.bilu0(A, len(pts))
    r = np.random.default_rng(1).normal(size=(len(pts), 4))
    x = pc.lu_solve(L, U, r, len(pts))
    M = np.zeros((len(pts) * 4,) * 2)
    for (p, q), blk in A.items():
        M[p * 4:(p + 1) * 4, q * 4:(q + 1) * 4] = blk
    np.testing.assert_allclose(x.ravel(), np.linalg.solve(M, r.ravel()), rtol=1e-10, atol=1e-12)


def test_ras_exact_matches_textbook_formula():
    """z = sum_i R_i^{0T} (R_i J R_i^T)^{-1} R_i^delta r with explicit 0/1 restriction matrices
    (Cai-Sarkis left-RAS) when no box wraps the periodic seam."""
    d, shape, nf = 2, (16, 16), 4
    m, Xa, Xb, cbar = state(d, shape)
    J = jacobian.assemble(m, Xa, Xb, 0.1).toarray()
    n = 256
    ras = pc.RAS(jacobian.assemble(m, Xa, Xb, 0.1), shape, nf, (2, 2), 2, exact=True)
    r = np.random.default_rng(2).normal(size=(nf,) + shape)
    z = ras.apply(r)
    zref = np.zeros(nf * n)
    for b in ras.boxes:
        pts = pc.local_points(b)
        g = [pc.global_index(b, l) for l in pts]
        cols = [f * n + gi for gi in g for f in range(nf)]      # point-major local ordering
        R = np.zeros((len(cols), nf * n))
        R[np.arange(len(cols)), cols] = 1
        Ai = R @ J @ R.T
        xi = np.linalg.solve(Ai, R @ r.ravel())
        own = np.array([pc.is_owned(b, l) for l in pts for f in range(nf)])
        R0 = R * own[:, None]
        zref += R0.T @ xi
    np.testing.assert_allclose(z.ravel(), zref, rtol=1e-10, atol=1e-12)


@pytest.mark.parametrize("variant", ["as", "rras"])
def test_schwarz_variants_match_textbook_formulas(variant):
    """Classical AS: z = sum_i R_i^T A_i^{-1} R_i r; right-restricted: z = sum_i R_i^T A_i^{-1} R_i^0 r, with
    explicit 0/1 restriction matrices and exact subdomain solves (Cai-Sarkis)."""
    d, shape, nf = 2, (16, 16), 4
    m, Xa, Xb, cbar = state(d, shape)
    Jsp = jacobian.assemble(m, Xa, Xb, 0.1)
    J = Jsp.toarray()
    n = 256
    pre = pc.RAS(Jsp, shape, nf, (2, 2), 2, exact=True, variant=variant)
    r = np.random.default_rng(3).normal(size=(nf,) + shape)
    z = pre.apply(r)
    zref = np.zeros(nf * n)
    for b in pre.boxes:
        pts = pc.local_points(b)
        g = [pc.global_index(b, l) for l in pts]
        cols = [f * n + gi for gi in g for f in range(nf)]
        R = np.zeros((len(cols), nf * n))
        R[np.arange(len(cols)), cols] = 1
        own = np.array([pc.is_owned(b, l) for l in pts for f in range(nf)])
        Rin = R * own[:, None] if variant == "rras" else R
        zref += R.T @ np.linalg.solve(R @ J @ R.T, Rin @ r.ravel())
    np.testing.assert_allclose(z.ravel(), zref, rtol=1e-10, atol=1e-12)


def test_schwarz_variants_coincide_without_overlap():
    """delta = 0: the boxes tile the grid, R_i^0 = R_i^delta, so RAS = AS = RRAS (block Jacobi over boxes)."""
    d, shape, nf = 2, (12, 12), 4
    m, Xa, Xb, cbar = state(d, shape)
    Jsp = jacobian.assemble(m, Xa, Xb, 0.2)
    r = np.random.default_rng(4).normal(size=(nf,) + shape)
    zs = [pc.RAS(Jsp, shape, nf, (3, 2), 0, variant=v).apply(r) for v in ("ras", "as", "rras")]
    np.testing.assert_array_equal(zs[0], zs[1])
    np.testing.assert_array_equal(zs[0], zs[2])


def test_ras_block_diagonal_reduces_to_block_jacobi():
    """With a block-diagonal J, BILU(0)-RAS = point-block Jacobi: z_p = J_pp^{-1} r_p."""
    import scipy.sparse as sp
    shape, nf = (8, 8), 4
    rng = np.random.default_rng(5)
    blocks = rng.normal(size=(64, nf, nf)) + 4 * np.eye(nf)
    # field-major block diagonal
    rows, cols, vals = [], [], []
    for p in range(64):
        for a in range(nf):
            for b in range(nf):
                rows.append(a * 64 + p)
                cols.append(b * 64 + p)
                vals.append(blocks[p, a, b])
    J = sp.csr_matrix((vals, (rows, cols)), shape=(256, 256))
    ras = pc.RAS(J, shape, nf, (2, 2), 2)
    r = rng.normal(size=(nf,) + shape)
    z = ras.apply(r).reshape(nf, 64)
    zref = np.stack([np.linalg.solve(blocks[p], r.reshape(nf, 64)[:, p]) for p in range(64)], axis=1)
    np.testing.assert_allclose(z, zref, rtol=1e-12)


# ----------------------------------------------------------------------------- ILU(k) subdomain solvers

def _box_matrix(shape=(8, 8), nsub=(2, 2), delta=1, dt=0.1):
    m, Xa, Xb, cbar = state(2, shape)
    J = jacobian.assemble(m, Xa, Xb, dt)
    b = pc.boxes(shape, nsub, delta)[0]
    A, pts = pc.box_blocks(J, b, 4, int(np.prod(shape)))
    return A, len(pts)


def _fill_path_levels(A, n):
    """Level of fill by the fill-path theorem (Hysom & Pothen 2001): lev(i, j) = (edges of the shortest
    path i -> j in the graph of A whose interior vertices are all < min(i, j)) - 1; brute force BFS."""
    adj = {i: set() for i in range(n)}
    for (p, q) in A:
        if p != q:
            adj[p].add(q)
    lev = {}
    for i in range(n):
        for j in range(n):
            if i == j:
                continue
            lim = min(i, j)
            dist = {i: 0}
            frontier = [i]
            found = None
            while frontier and found is None:
                nxt = []
                for v in frontier:
                    for w in adj[v]:
                        if w == j:
                            found = dist[v] + 1
                            break
                        if w < lim and w not in dist:
                            dist[w] = dist[v] + 1
                            nxt.append(w)
                    if found is not None:
                        break
                frontier = nxt
            if found is not None:
                lev[(i, j)] = found - 1
    return lev


def test_fill_levels_match_the_fill_path_theorem():
    A, n = _box_matrix(shape=(6, 6), nsub=(1, 1), delta=0)        # 36 points, 13-point pattern
    ref = _fill_path_levels(A, n)
    for k in (0, 1, 2, 3):
        got = pc.fill_levels(A, n, k)
        want = {(i, j) for (i, j), lv in ref.items() if lv <= k}
        have = {(i, j) for i in range(n) for j, lv in got[i].items() if i != j}
        assert have == want, k
        for (i, j) in have:
            assert got[i][j] == ref[(i, j)]


def test_biluk_level0_is_bilu0():
    A, n = _box_matrix()
    L0, U0 = pc.bilu0(A, n)
    L, U = pc.biluk(A, n, 0)
    assert set(L) == set(L0) and set(U) == set(U0)
    for key in L0:
        np.testing.assert_allclose(L[key], L0[key], rtol=1e-14, atol=1e-14 * np.abs(L0[key]).max())


@pytest.mark.parametrize("k", [1, 2])
def test_biluk_defining_property(k):
    """(L U)_pq = A_pq on the level-k pattern (the definition of ILU(k)); the pattern grows with k."""
    A, n = _box_matrix()
    L, U = pc.biluk(A, n, k)
    pattern = set(L) | set(U)
    assert len(pattern) > len(A)
    nf = 4
    for (p, q) in pattern:
        acc = np.zeros((nf, nf))
        for kk in range(min(p, q) + 1):
            lpk = np.eye(nf) if kk == p else L.get((p, kk))
            ukq = U.get((kk, q))
            if lpk is not None and ukq is not None:
                acc += lpk @ ukq
        ref = A.get((p, q), np.zeros((nf, nf)))
        scale = max(np.abs(ref).max(), 1.0)
        np.testing.assert_allclose(acc, ref, rtol=0, atol=1e-10 * scale)


def test_biluk_unlimited_is_the_exact_lu():
    """No level limit: L U = A exactly, and the RAS apply equals the one with dense LAPACK box solves."""
    shape, nsub, delta = (8, 8), (2, 2), 1
    m, Xa, Xb, cbar = state(2, shape)
    J = jacobian.assemble(m, Xa, Xb, 0.1)
    r = ni.random_direction(4, shape, 3)
    z_lu = pc.RAS(J, shape, 4, nsub, delta, fill=None).apply(r)
    z_ex = pc.RAS(J, shape, 4, nsub, delta, exact=True).apply(r)
    np.testing.assert_allclose(z_lu, z_ex, rtol=0, atol=1e-10 * np.abs(z_ex).max())
    z0 = pc.RAS(J, shape, 4, nsub, delta).apply(r)
    assert np.abs(z0 - z_ex).max() > 1e-6 * np.abs(z_ex).max()   # ILU(0) is not exact on these boxes
