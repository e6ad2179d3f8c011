"""Oracle: gauge, initial mechanical equilibrium, exact Newton with line search, and the adaptive
time-step controller (TEST INFRASTRUCTURE ONLY).

* gauge (reading R14): the central-difference elastic operator on a periodic grid annihilates
  displacements that are constant on each parity sub-lattice of the even-length axes; u is
  reported with zero mean per (component, sub-lattice).
* u^0 (reading R13): [D^ sigma^el]^0 = 0 solved at t_0 (needed by the proof P:403-417).
* Newton: X_{m+1} = X_m + lambda_m S_m with J_m S_m = -F(X_m) solved EXACTLY by a
  sparse direct LU in which one redundant u-row per (component, sub-lattice) is replaced by an
  identity row (reading R14); line search of reading R17; stop at ||F|| <= max(eps_r ||F_0||, eps_a).
* controller: Eq. (sencondt) P:596-607 with the RMS norm of reading R23 and the retry rule P:605-607.
"""
from __future__ import annotations

import math

import numpy as np
import scipy.sparse as sp
import scipy.sparse.linalg as spla

from . import jacobian, scheme


# ----------------------------------------------------------------------------- gauge

def sublattice_ids(shape, bc="periodic"):
    """Class id of each point: bits = parity of the coordinate along each EVEN-length axis.  Neumann
    (reading R38): the elastic null space is the translations only -- one class."""
    d = len(shape)
    ids = np.zeros(shape, dtype=np.int64)
    if bc != "periodic":
        return ids, 1
    coords = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    bit = 0
    for j in range(d):                       # j = 0 is x (array axis d-1)
        ax = d - 1 - j
        if shape[ax] % 2 == 0:
            ids += (coords[ax] % 2) << bit
            bit += 1
    return ids, 1 << bit


def neumann_rotations(shape):
    """Discrete rigid rotations of a Neumann grid (reading R38): for every axis pair (I, J) whose extents are
    both even, u_I = s(x_J), u_J = -s(x_I) with the staircase s(k) = floor((k + 1)/2) has D^ s = 1/(2h)
    everywhere under the mirror ghosts, so its strain vanishes.  Returned orthonormalised against the
    translations and each other, as (d, *shape) arrays."""
    d = len(shape)
    coords = np.meshgrid(*[np.arange(n) for n in shape], indexing="ij")
    modes = []
    for I in range(d):
        for J in range(I + 1, d):
            aI, aJ = d - 1 - I, d - 1 - J          # array axes of coordinate axes I, J
            if shape[aI] % 2 or shape[aJ] % 2:
                continue
            r = np.zeros((d,) + tuple(shape))
            r[I] = (coords[aJ] + 1) // 2
            r[J] = -((coords[aI] + 1) // 2)
            for K in range(d):
                r[K] -= r[K].mean()                # orthogonal to the translations
            for q in modes:
                r -= np.sum(r * q) * q
            modes.append(r / np.sqrt(np.sum(r * r)))
    return modes


def gauge_project(X, bc="periodic"):
    """Subtract, for every u component, its mean on each parity sub-lattice (reading R14).  Neumann
    (reading R38): the mean of every component (translations) and the discrete rotation modes."""
    d = X.ndim - 1
    shape = X.shape[1:]
    if bc != "periodic":
        Y = X.copy()
        for I in range(d):
            Y[2 + I] -= Y[2 + I].mean()
        for r in neumann_rotations(shape):
            Y[2:] -= np.sum(Y[2:] * r) * r
        return Y
    ids, ncls = sublattice_ids(shape, bc)
    Y = X.copy()
    for I in range(d):
        u = Y[2 + I]
        for k in range(ncls):
            mask = ids == k
            u[mask] -= u[mask].mean()
    return Y


def pinned_rows(shape, d, bc="periodic"):
    """Row indices (field-major) of one u_I row per (component, sub-lattice): the first point of the class.
    Neumann: u_I at the first point per component, and per rotation mode (I, J) u_J at x_I = 1 (the mode's
    u_J differs there from the first point, so the pins fix it)."""
    if bc != "periodic":
        n = int(np.prod(shape))
        rows = [(2 + I) * n for I in range(d)]
        for I in range(d):
            for J in range(I + 1, d):
                if shape[d - 1 - I] % 2 or shape[d - 1 - J] % 2:
                    continue
                idx = [0] * d
                idx[d - 1 - I] = 1
                rows.append((2 + J) * n + int(np.ravel_multi_index(tuple(idx), shape)))
        return rows
    ids, ncls = sublattice_ids(shape, bc)
    n = int(np.prod(shape))
    flat = ids.ravel()
    rows = []
    for I in range(d):
        for k in range(ncls):
            rows.append((2 + I) * n + int(np.argmax(flat == k)))
    return rows


def pin(A, b, rows):
    """Replace the given rows of A by identity rows and the matching entries of b by 0."""
    A = A.tolil(copy=True)
    b = b.copy()
    for r in rows:
        A.rows[r] = [r]
        A.data[r] = [1.0]
        b[r] = 0.0
    return A.tocsc(), b


# ----------------------------------------------------------------------------- initial elastic equilibrium

def elastic_block(m: scheme.Model, shape):
    """Sparse operator A_uu (u rows, u cols) and A_uc with F_u = A_uu u + A_uc (c - cbar0)."""
    ops = jacobian.grid_operators(shape, m.h, m.bc)
    sig = jacobian.stress_operators(m, ops)
    D = ops["Dhat_o"]
    d = m.d
    Auu = sp.bmat([[sum(D[J] @ sig[I][J][0][M] for J in range(d)) for M in range(d)] for I in range(d)],
                  format="csr")
    Auc = sp.vstack([sum(D[J] @ sig[I][J][1] for J in range(d)) for I in range(d)], format="csr")
    return Auu, Auc


def init_displacement(m: scheme.Model, c, cbar0):
    """u^0 solving [D^ sigma^el(u, c^0)] = 0 in the canonical gauge (reading R13) by pinned sparse LU."""
    shape = c.shape
    d = m.d
    n = c.size
    Auu, Auc = elastic_block(m, shape)
    b = -(Auc @ (c - cbar0).ravel())
    rows = [r - 2 * n for r in pinned_rows(shape, d, m.bc)]
    A, b = pin(Auu, b, rows)
    u = spla.spsolve(A, b).reshape((d,) + shape)
    X = np.zeros((2 + d,) + shape)
    X[2:] = u
    return gauge_project(X, m.bc)[2:]


def init_displacement_fft(m: scheme.Model, c, cbar0):
    """Same u^0 via the discrete Fourier transform (for grids too large for the sparse LU).

    D^_J acting on exp(i k.x) is i s_J with s_J = sin(k_J h)/h; the d x d symbol of
    sum_J D^_J sigma_IJ is solved per wavenumber; modes with all s_J = 0 are the gauge (set to 0).
    """
    d, h = m.d, m.h
    shape = c.shape
    L = m.Lscale
    K = m.C11 + (d - 1) * m.C12
    rho = np.fft.fftn(c - cbar0)
    ks = np.meshgrid(*[2 * np.pi * np.fft.fftfreq(n) for n in shape], indexing="ij")
    s = [np.sin(ks[d - 1 - J]) / h for J in range(d)]   # s[J] along axis J
    # F_I = sum_J i s_J sigma_IJ ; sigma_II = L[C12 sum_M i s_M u_M + (C11-C12) i s_I u_I - K eps0 rho]
    #                              sigma_IJ = L C44 (i s_J u_I + i s_I u_J)
    A = np.zeros((d, d) + shape, dtype=complex)
    for I in range(d):
        for M in range(d):
            if I == M:
                A[I, M] = -L * (m.C11 * s[I] ** 2 + m.C44 * sum(s[J] ** 2 for J in range(d) if J != I))
            else:
                A[I, M] = -L * (m.C12 + m.C44) * s[I] * s[M]
    # F_I = sum_M A_IM u_M - i s_I L K eps0 rho = 0  =>  A u = i s_I L K eps0 rho
    rhs = np.stack([1j * s[I] * L * K * m.eps0 * rho for I in range(d)])
    A2 = np.moveaxis(A.reshape(d, d, -1), -1, 0)
    r2 = np.moveaxis(rhs.reshape(d, -1), -1, 0)
    null = np.all(np.stack([np.abs(si) < 1e-12 for si in s]), axis=0).ravel()
    A2[null] = np.eye(d)
    r2[null] = 0
    uh = np.linalg.solve(A2, r2[..., None])[..., 0]
    uh = np.moveaxis(uh, 0, -1).reshape((d,) + shape)
    return np.real(np.stack([np.fft.ifftn(uh[I]) for I in range(d)]))


# ----------------------------------------------------------------------------- Newton

def norm(F):
    """Unweighted Euclidean norm over all (2+d)N entries (reading R16)."""
    return float(np.sqrt(np.sum(F * F)))


def direct_linsolve(m: scheme.Model, Xa, X, dt, cbar0, b, fnorm):
    """J S = b by the gauge-pinned sparse direct LU (reading R14): exact up to rounding."""
    J = jacobian.assemble(m, Xa, X, dt)
    A, bb = pin(J, b.ravel(), pinned_rows(X.shape[1:], m.d, m.bc))
    return spla.spsolve(A, bb).reshape(X.shape)


def newton_step(m: scheme.Model, Xa, dt, cbar0, sol: dict, X0=None, linsolve=None):
    """One NSOA-1 time step by Newton.  Returns (X^b, info).

    linsolve(m, Xa, X, dt, cbar0, b, fnorm) -> S solves J(X) S = b with b = -F(X) whose u rows are
    projected onto range(J) (the u_I sub-lattice sums span the left null space, reading R14); the
    default is the exact gauge-pinned direct LU, ``krylov.make_linsolve`` the GMRES path of the
    large-grid parity cases.  A linsolve returning None is a linear-solver failure (DIVERGED)."""
    d = m.d
    shape = Xa.shape[1:]
    X = (Xa if X0 is None else X0).copy()          # X_0 = X^n (reading R29)
    F = scheme.residual(m, Xa, X, dt, cbar0)
    f0 = norm(F)
    hist = [f0]
    solve = linsolve if linsolve is not None else direct_linsolve
    info = {"converged": False, "reason": "", "newton_its": 0, "fnorm0": f0, "hist": hist,
            "lambdas": []}
    for it in range(sol["newton_maxit"] + 1):
        if hist[-1] <= max(sol["newton_rtol"] * f0, sol["newton_atol"]):
            info["converged"] = True
            break
        if it == sol["newton_maxit"]:
            info["reason"] = "newton_maxit"
            return Xa.copy(), info
        S = solve(m, Xa, X, dt, cbar0, gauge_project(-F, m.bc), hist[-1])
        if S is None:
            info["reason"] = "linear_solver"
            return Xa.copy(), info
        lam, fn = 1.0, hist[-1]
        accepted = False
        for _ in range(sol["ls_max_halvings"] + 1):
            Xt = X + lam * S
            if scheme.admissible(Xt):
                Ft = scheme.residual(m, Xa, Xt, dt, cbar0)
                ft = norm(Ft)
                if np.isfinite(ft) and ft <= (1 - sol["ls_alpha"] * lam) * fn:
                    accepted = True
                    break
            lam /= 2
        if not accepted:
            info["reason"] = "line_search"
            return Xa.copy(), info
        info["lambdas"].append(lam)
        X = gauge_project(Xt, m.bc)
        F = Ft
        hist.append(ft)
        info["newton_its"] = it + 1
    info["fnorm"] = hist[-1]
    return X, info


def step_report(m: scheme.Model, X, cbar0):
    """Energy parts and mass after a step."""
    parts = scheme.energy_parts(m, X, cbar0)
    return {"energy": float(sum(parts)), "energy_parts": [float(p) for p in parts],
            "mass": float(scheme.mass(m, X))}


# ----------------------------------------------------------------------------- adaptive controller

def predict_dt(xd: float, zeta: float, dt_min: float, dt_max: float) -> float:
    """Eq. (sencondt): max(dt_min, dt_max / sqrt(1 + zeta X'_d^2))."""
    return max(dt_min, dt_max / math.sqrt(1 + zeta * xd * xd))


def change_rate(Xn, Xprev, dt_prev, kind: str = "rms") -> float:
    """X'_d = ||X^n - X^{n-1}|| / dt_{n-1}; norm per reading R23."""
    diff = Xn - Xprev
    if kind == "rms":
        nrm = math.sqrt(float(np.sum(diff * diff)) / diff.size)
    elif kind == "l2":
        nrm = math.sqrt(float(np.sum(diff * diff)))
    elif kind == "ceta_l2":
        nrm = math.sqrt(float(np.sum(diff[:2] * diff[:2])))
    else:
        raise ValueError(kind)
    return nrm / dt_prev


def run_adaptive(m: scheme.Model, X0, cbar0, sol: dict, nsteps: int, forced_dts=None, linsolve=None):
    """Adaptive time stepping.  forced_dts: optional list of accepted dt to replay."""
    X = X0.copy()
    Xprev = None
    dt_prev = None
    zeta = sol["zeta"]
    records = []
    for n in range(nsteps):
        if forced_dts is not None:
            dt = forced_dts[n]
        elif n == 0:
            dt = sol["dt_init"]
        else:
            dt = predict_dt(change_rate(X, Xprev, dt_prev, sol["xd_norm"]), zeta, sol["dt_min"], sol["dt_max"])
        retries = 0
        while True:
            Xb, info = newton_step(m, X, dt, cbar0, sol, linsolve=linsolve)
            if info["converged"] or forced_dts is not None:
                break
            dt /= math.sqrt(2)
            zeta *= 2
            retries += 1
            if dt < sol["dt_min"] * sol["dt_floor_factor"]:
                raise RuntimeError("adaptive controller: dt below floor")
        rec = step_report(m, Xb, cbar0)
        rec.update({"dt": dt, "retries": retries, "newton_its": info["newton_its"],
                    "converged": info["converged"], "zeta": zeta})
        records.append(rec)
        Xprev, X, dt_prev = X, Xb, dt
    return X, records
