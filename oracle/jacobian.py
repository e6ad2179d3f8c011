"""Oracle: the Newton Jacobian J = dF/dX^b of scheme NSOA-1, assembled as a SciPy CSR matrix
(TEST INFRASTRUCTURE ONLY).

J_m := grad F(X_m).  The matrix is composed from sparse grid operators
(shift, central difference, Laplacian, D M~ D) exactly mirroring the residual of
``scheme.residual``; the only pointwise non-linear derivatives,
a_kl = d(G^1 + G^{2,S})_k / d(c^b, eta^b)_l, are taken by complex-step
differentiation of ``scheme.G1 + scheme.G2S`` (exact to rounding for analytic
functions; no subtractive cancellation).

Unknown ordering of the assembled matrix: field-major (all c, all eta, all u_1, ...),
each field in C order.  (The paper orders unknowns by points; an ordering is
a permutation and does not change the solution.)
"""
from __future__ import annotations

import numpy as np
import scipy.sparse as sp

from . import scheme

CSTEP = 1e-30


def _shift_matrix(shape, j: int, s: int, bc: str = "periodic", parity: int = 1):
    """Sparse S with (S f)_i = f_{i + s e_j} for C-order grids of ``shape``: exactly scheme.shift applied to
    the unit vectors (periodic wrap, or the Neumann mirror ghost, odd with parity -1)."""
    d = len(shape)
    n = int(np.prod(shape))
    idx = np.arange(n, dtype=float).reshape(shape)
    src = scheme.shift(idx, j, s, d, bc).ravel().astype(np.int64)
    val = np.ones(n)
    if bc != "periodic" and parity == -1:
        val = scheme.shift(np.ones(shape), j, s, d, bc, -1).ravel()
    return sp.csr_matrix((val, (np.arange(n), src)), shape=(n, n))


def grid_operators(shape, h, bc="periodic"):
    """Dictionary of sparse operators: I, Dhat[j] (even ghosts), Dhat_o[j] (the outer derivative of the u
    rows: odd stress ghosts for Neumann, = Dhat for periodic), Lap, Splus[j], Sminus[j]."""
    d = len(shape)
    n = int(np.prod(shape))
    I = sp.identity(n, format="csr")
    Sp = [_shift_matrix(shape, j, 1, bc) for j in range(d)]
    Sm = [_shift_matrix(shape, j, -1, bc) for j in range(d)]
    Dhat = [(Sp[j] - Sm[j]) / (2 * h) for j in range(d)]
    if bc == "periodic":
        Dhat_o = Dhat
    else:
        Dhat_o = [(_shift_matrix(shape, j, 1, bc, -1) - _shift_matrix(shape, j, -1, bc, -1)) / (2 * h) for j in range(d)]
    Lap = sum((Sp[j] - 2 * I + Sm[j]) / h ** 2 for j in range(d))
    return {"I": I, "Sp": Sp, "Sm": Sm, "Dhat": Dhat, "Dhat_o": Dhat_o, "Lap": Lap, "n": n, "d": d, "bc": bc}


def div_M_grad_matrix(ops, ca, kappa, h):
    """W with W g = D M~ D g, mobility at level n."""
    d, bc = ops["d"], ops["bc"]
    W = 0 * ops["I"]
    for j in range(d):
        mp = scheme.mobility_face(ca, kappa, j, d, bc).ravel()
        mm = scheme.shift(scheme.mobility_face(ca, kappa, j, d, bc), j, -1, d, bc).ravel()
        W = W + (sp.diags(mp) @ (ops["Sp"][j] - ops["I"]) - sp.diags(mm) @ (ops["I"] - ops["Sm"][j])) / h ** 2
    return W.tocsr()


def pointwise_partials(m: scheme.Model, Xa, Xb):
    """a_kl = d(G1+G2S)_k/d(c^b, eta^b)_l at each point, by complex step (k, l in {c, eta})."""
    ca, ea, cb, eb = Xa[0], Xa[1], Xb[0], Xb[1]

    def g(cb_, eb_):
        g1 = scheme.G1(m, ca, cb_, ea, eb_)
        g2 = scheme.G2S(m, ca, cb_, ea, eb_)
        return g1[0] + g2[0], g1[1] + g2[1]
    gc_dc, ge_dc = g(cb + 1j * CSTEP, eb + 0j)
    gc_de, ge_de = g(cb + 0j, eb + 1j * CSTEP)
    return (np.imag(gc_dc) / CSTEP, np.imag(gc_de) / CSTEP,
            np.imag(ge_dc) / CSTEP, np.imag(ge_de) / CSTEP)


def stress_operators(m: scheme.Model, ops):
    """sig[I][J] = (list of d sparse ops acting on u_1..u_d, coefficient op acting on c) such that
    sigma^el_IJ(u, c) = sum_M sig_u[M] u_M + sig_c c + const."""
    d, L = m.d, m.Lscale
    D = ops["Dhat"]
    Z = 0 * ops["I"]
    K = m.C11 + (d - 1) * m.C12
    sig = [[None] * d for _ in range(d)]
    for I in range(d):
        for J in range(d):
            if I == J:
                su = [L * m.C12 * D[M] + (L * (m.C11 - m.C12) * D[I] if M == I else Z) for M in range(d)]
                sc = -L * K * m.eps0 * ops["I"]
            else:
                # sigma_IJ = 2 L C44 eps_IJ = L C44 (D_J u_I + D_I u_J)
                su = [(L * m.C44 * D[J] if M == I else Z) + (L * m.C44 * D[I] if M == J else Z)
                      for M in range(d)]
                sc = Z
            sig[I][J] = (su, sc)
    return sig


def assemble(m: scheme.Model, Xa, Xb, dt):
    """Analytic J = dF/dX^b (field-major ordering) as CSR."""
    d, h = m.d, m.h
    shape = Xb.shape[1:]
    ops = grid_operators(shape, h, m.bc)
    I = ops["I"]
    D = ops["Dhat"]
    Lap = ops["Lap"]
    a11, a12, a21, a22 = [a.ravel() for a in pointwise_partials(m, Xa, Xb)]
    W = div_M_grad_matrix(ops, Xa[0], m.kappa, h)
    K = m.Lscale * (m.C11 + (d - 1) * m.C12)
    # dG_c/dX^b: pointwise a11, a12; G3_c = -(eps0/2)(T^a + T^b), T^b = K(sum_J D_J u_J - d eps0 (c^b - cbar0));
    # G4_c = -gamma_c Lap (c^a + c^b)/2.
    dGc_dc = sp.diags(a11) + (m.eps0 / 2) * K * d * m.eps0 * I - (m.gamma_c / 2) * Lap
    dGc_de = sp.diags(a12)
    dGc_du = [-(m.eps0 / 2) * K * D[J] for J in range(d)]
    dGe_dc = sp.diags(a21)
    dGe_de = sp.diags(a22) - (3 * m.gamma_eta / 2) * Lap
    blocks = [[None] * (2 + d) for _ in range(2 + d)]
    blocks[0][0] = I / dt - W @ dGc_dc
    blocks[0][1] = -W @ dGc_de
    for J in range(d):
        blocks[0][2 + J] = -W @ dGc_du[J]
    blocks[1][0] = dGe_dc
    blocks[1][1] = I / dt + dGe_de
    sig = stress_operators(m, ops)
    Do = ops["Dhat_o"]
    for Irow in range(d):
        blocks[2 + Irow][0] = sum(Do[J] @ sig[Irow][J][1] for J in range(d))
        for M in range(d):
            blocks[2 + Irow][2 + M] = sum(Do[J] @ sig[Irow][J][0][M] for J in range(d))
    return sp.bmat(blocks, format="csr")


def jv_complex_step(m: scheme.Model, Xa, Xb, dt, cbar0, v):
    """J v = Im F(X^b + i eps v)/eps (exact directional derivative; independent of ``assemble``)."""
    Fc = scheme.residual(m, Xa.astype(complex), Xb + 1j * CSTEP * v, dt, cbar0)
    return np.imag(Fc) / CSTEP


def jv_central_fd(m: scheme.Model, Xa, Xb, dt, cbar0, v, eps=1e-6):
    """[F(X + eps v) - F(X - eps v)]/(2 eps) (BASELINE.json J.v check)."""
    return (scheme.residual(m, Xa, Xb + eps * v, dt, cbar0)
            - scheme.residual(m, Xa, Xb - eps * v, dt, cbar0)) / (2 * eps)


def jv(m: scheme.Model, Xa, Xb, dt, v):
    """J v with the assembled matrix (field-major flatten)."""
    J = assemble(m, Xa, Xb, dt)
    return (J @ v.ravel()).reshape(v.shape)
