"""Oracle: a Krylov path for the Newton systems of large grids (TEST INFRASTRUCTURE ONLY).

The exact-Newton oracle (``solver.newton_step``) solves J S = -F with a gauge-pinned sparse
direct LU.  That is exact but its fill makes it impractical beyond ~10^5 unknowns, so for the
full-size parity cases (512^2: 1.0 M unknowns, 128^3: 10.5 M) the same Newton iteration
(readings R16/R17/R29) is run with this linear solver instead:

* J v matrix-free, written out from SURVEY 8(c).1 step 8 (the linearisation of the residual of
  ``scheme.residual``):
      w_c = a11 v_c + a12 v_eta + (eps0 K/2)(d eps0 v_c - sum_J D^_J v_uJ) - (gamma_c/2) Lap v_c
      w_e = a21 v_c + a22 v_eta - (3 gamma_eta/2) Lap v_eta
      (J v)_c = v_c/dt - D M~ D w_c,   (J v)_eta = v_eta/dt + w_e,
      (J v)_uI = sum_J D^_J sigma_IJ(v_u, v_c)  with the eigenstrain -eps0 v_c delta_IJ inside eps^el,
  K = Lscale (C11 + (d-1) C12); a_kl = d(G1 + G2S)_k / d(c^b, eta^b)_l are the complex-step
  partials of ``jacobian.pointwise_partials``.  Pinned against the assembled J and against the
  complex-step directional derivative of F (tests/test_oracle_krylov.py).
* restarted right-preconditioned GMRES(m) (Saad, Iterative Methods, Alg. 6.10 + 9.5: modified
  Gram-Schmidt Arnoldi, Givens rotations, x0 = 0), stopping on the TRUE residual
  ||b - J s|| <= tol checked at every restart (reading R18);
* a spectral preconditioner: J with every coefficient replaced by its grid mean (a_kl, the face
  mobility M~) is translation invariant, so the discrete Fourier transform diagonalises it into one
  (2+d) x (2+d) matrix per wave number (D^_J -> i sin(k_J h)/h, Lap -> -sum_J (2 - 2 cos k_J h)/h^2).
  Its inverse is applied per wave number; on the gauge modes (every sin(k_J h) = 0, reading R14) the
  u block is singular and the preconditioned u is set to 0 there.  The preconditioner only changes
  how many GMRES iterations are needed, never the solution GMRES converges to.

Nothing here is shared with the CUDA library.
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft as sfft

from . import jacobian, scheme

_WORKERS = os.cpu_count() or 1


# ----------------------------------------------------------------------------- J v, matrix-free

class Linearisation:
    """J = dF/dX^b at (X^a, X^b, dt): the pointwise partials are taken once per Newton iterate."""

    def __init__(self, m: scheme.Model, Xa, Xb, dt):
        self.m, self.Xa, self.dt = m, Xa, dt
        self.a11, self.a12, self.a21, self.a22 = jacobian.pointwise_partials(m, Xa, Xb)
        self.K = m.Lscale * (m.C11 + (m.d - 1) * m.C12)

    def jv(self, v):
        """J v for v of shape (2+d, *grid)."""
        m, d, h, bc = self.m, self.m.d, self.m.h, self.m.bc
        vc, ve, vu = v[0], v[1], v[2:]
        div_u = sum(scheme.D_hat(vu[J], J, h, d, bc) for J in range(d))
        wc = (self.a11 * vc + self.a12 * ve + (m.eps0 * self.K / 2) * (d * m.eps0 * vc - div_u)
              - (m.gamma_c / 2) * scheme.laplacian(vc, h, d, bc))
        we = self.a21 * vc + self.a22 * ve - (3 * m.gamma_eta / 2) * scheme.laplacian(ve, h, d, bc)
        out = np.empty_like(v)
        out[0] = vc / self.dt - scheme.div_M_grad(wc, self.Xa[0], m.kappa, h, d, bc)
        out[1] = ve / self.dt + we
        # sigma(v_u, v_c): the stress of eps(v_u) - eps0 v_c I (cbar0 is a constant and drops out)
        sig = scheme.stress(m, scheme.elastic_strain(m, vu, vc, 0.0))
        for I in range(d):
            out[2 + I] = sum(scheme.D_hat(sig[I][J], J, h, d, bc, -1) for J in range(d))
        return out


# ----------------------------------------------------------------------------- spectral preconditioner

class SpectralPC:
    """Inverse of the mean-coefficient Jacobian, per wave number (real-to-complex FFT over the grid)."""

    def __init__(self, lin: Linearisation):
        m, d, h, dt = lin.m, lin.m.d, lin.m.h, lin.dt
        shape = lin.Xa.shape[1:]
        self.shape, self.d, self.nf = shape, d, 2 + d
        # wave numbers: axis j (0 = x) is array axis d-1-j; the last array axis (x) is half-spectrum
        ks = []
        for ax, n in enumerate(shape):
            f = np.fft.rfftfreq(n) if ax == d - 1 else np.fft.fftfreq(n)
            ks.append(2 * np.pi * f)
        grids = np.meshgrid(*ks, indexing="ij")
        s = [np.sin(grids[d - 1 - J]) / h for J in range(d)]                 # D^_J -> i s_J
        lam = sum((2 - 2 * np.cos(grids[d - 1 - J])) / h ** 2 for J in range(d))   # -Lap -> lam
        Mbar = float(np.mean([np.mean(scheme.mobility_face(lin.Xa[0], m.kappa, J, d)) for J in range(d)]))
        a11, a12, a21, a22 = (float(np.mean(a)) for a in (lin.a11, lin.a12, lin.a21, lin.a22))
        K = lin.K
        L = m.Lscale
        kshape = lam.shape
        P = np.zeros(kshape + (self.nf, self.nf), dtype=complex)
        # c row: v_c/dt + Mbar lam w_c
        wc_c = a11 + (m.eps0 * K / 2) * d * m.eps0 + (m.gamma_c / 2) * lam
        P[..., 0, 0] = 1 / dt + Mbar * lam * wc_c
        P[..., 0, 1] = Mbar * lam * a12
        for J in range(d):
            P[..., 0, 2 + J] = Mbar * lam * (-(m.eps0 * K / 2) * 1j * s[J])
        # eta row
        P[..., 1, 0] = a21
        P[..., 1, 1] = 1 / dt + a22 + (3 * m.gamma_eta / 2) * lam
        # u rows: sum_J i s_J sigma_IJ,  sigma_II = L[C12 tr + (C11-C12) eps_II] - K eps0 v_c
        for I in range(d):
            P[..., 2 + I, 0] = 1j * s[I] * (-K * m.eps0)
            for M in range(d):
                if I == M:
                    P[..., 2 + I, 2 + M] = -L * (m.C11 * s[I] ** 2 + m.C44 * sum(s[J] ** 2 for J in range(d) if J != I))
                else:
                    P[..., 2 + I, 2 + M] = -L * (m.C12 + m.C44) * s[I] * s[M]
        null = np.all(np.stack([np.abs(sj) < 1e-12 for sj in s]), axis=0)
        if m.bc == "periodic":
            for I in range(d):
                P[null, 2 + I, 2 + I] = 1.0      # gauge modes: u block replaced by I (then zeroed below)
        else:
            # Neumann (R38): the Fourier modes are not its eigenvectors and its gauge is not the parity
            # classes, so the singular u block gets a regular stand-in of the elastic diagonal's scale
            for I in range(d):
                P[null, 2 + I, 2 + I] = -L * m.C11 / h ** 2
        Pinv = np.linalg.inv(P)
        if m.bc == "periodic":
            Pinv[null, 2:, :] = 0.0
            Pinv[null, :, 2:] = 0.0
        self.Pinv = np.ascontiguousarray(np.moveaxis(Pinv, (-2, -1), (0, 1)))   # (nf, nf, *kshape)

    def apply(self, r):
        rh = sfft.rfftn(r, axes=tuple(range(1, self.d + 1)), workers=_WORKERS)
        zh = np.einsum("ij...,j...->i...", self.Pinv, rh)
        return sfft.irfftn(zh, s=self.shape, axes=tuple(range(1, self.d + 1)), workers=_WORKERS)


# ----------------------------------------------------------------------------- GMRES(m)

def gmres(matvec, b, tol, restart=30, maxit=10000, precond=None):
    """Right-preconditioned restarted GMRES, x0 = 0 (Saad Alg. 6.10 with MGS, Alg. 9.5 for the right
    preconditioner).  Returns (x, iterations, true residual norm, converged)."""
    M = precond if precond is not None else (lambda v: v)
    x = np.zeros_like(b)
    r = b.copy()
    beta = float(np.linalg.norm(r))
    its = 0
    while True:
        if beta <= tol:
            return x, its, beta, True
        if its >= maxit:
            return x, its, beta, False
        V = [r / beta]
        H = np.zeros((restart + 1, restart))
        g = np.zeros(restart + 1)
        g[0] = beta
        cs, sn = np.zeros(restart), np.zeros(restart)
        Zs = []
        j = 0
        while j < restart and its < maxit:
            z = M(V[j])
            Zs.append(z)
            w = matvec(z)
            for i in range(j + 1):                       # modified Gram-Schmidt
                H[i, j] = float(np.vdot(V[i], w))
                w = w - H[i, j] * V[i]
            hnext = float(np.linalg.norm(w))
            H[j + 1, j] = hnext
            for i in range(j):                           # previous rotations
                a, c2 = H[i, j], H[i + 1, j]
                H[i, j], H[i + 1, j] = cs[i] * a + sn[i] * c2, -sn[i] * a + cs[i] * c2
            rr = np.hypot(H[j, j], H[j + 1, j])
            cs[j], sn[j] = (H[j, j] / rr, H[j + 1, j] / rr) if rr > 0 else (1.0, 0.0)
            H[j, j], H[j + 1, j] = rr, 0.0
            g[j + 1], g[j] = -sn[j] * g[j], cs[j] * g[j]
            its += 1
            j += 1
            if abs(g[j]) <= tol or hnext == 0.0:         # converged estimate, or lucky breakdown
                break
            V.append(w / hnext)
        y = np.zeros(j)
        for k in range(j - 1, -1, -1):
            y[k] = (g[k] - H[k, k + 1:j] @ y[k + 1:j]) / H[k, k]
        x = x + sum(y[k] * Zs[k] for k in range(j))
        r = b - matvec(x)
        beta = float(np.linalg.norm(r))


def make_linsolve(restart=30, rtol=1e-10, atol=0.0, maxit=10000, stats=None):
    """A linear solver for ``solver.newton_step(linsolve=...)``: solves J S = b (b = -F, gauge-
    projected by the caller) by spectral-preconditioned GMRES(restart) to
    ||J S - b|| <= max(rtol ||F||, atol) (reading R16)."""
    def linsolve(m, Xa, X, dt, cbar0, b, fnorm):
        lin = Linearisation(m, Xa, X, dt)
        pcd = SpectralPC(lin)
        S, its, res, ok = gmres(lin.jv, b, max(rtol * fnorm, atol), restart, maxit, pcd.apply)
        if stats is not None:
            stats.append({"gmres_its": its, "residual": res, "converged": ok})
        if not ok:
            return None
        return S
    return linsolve
