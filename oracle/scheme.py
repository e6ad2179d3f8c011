"""Oracle: the DVD scheme NSOA-1 of arXiv 2209.08001, written out plainly (TEST INFRASTRUCTURE ONLY).

Fields are NumPy arrays in C order over the grid (z, y, x) with x fastest; axis
index ``j`` (0 = x, 1 = y, 2 = z) maps to array axis ``d-1-j``.  A state X is an
array of shape (2+d, *grid): X[0] = c, X[1] = eta, X[2+j] = u_{j+1} (displacement
along axis j).  Periodic boundary conditions.  Level "a" = t_n (known),
level "b" = t_{n+1} (unknown).

Everything here is fp64 and vectorised with ``np.roll``; functions also accept
complex arrays so that ``jacobian.py`` can take complex-step derivatives.
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np


# ----------------------------------------------------------------------------- parameters

@dataclass
class Model:
    """Dimensionless model parameters (App. A/B) + grid spacing.

    The CALPHAD-style inputs L0..L3, U1, U4, dE0 are in units of V_m*dE, so the
    1/(V_m dE) factors of App. B are 1.
    """
    d: int
    h: float
    theta: float
    gamma_c: float
    gamma_eta: float
    kappa: float
    eps0: float
    C11: float
    C12: float
    C44: float
    Lscale: float
    w_c: float
    L0: float
    L1: float
    L2: float
    L3: float
    U1: float
    U4: float
    dE0: float
    S: int = 10
    bc: str = "periodic"        # "periodic" or "neumann": Eq. (boundaryequ), reading R38

    @staticmethod
    def from_dict(d: int, h: float, p: dict, bc: str = "periodic") -> "Model":
        keys = ["theta", "gamma_c", "gamma_eta", "kappa", "eps0", "C11", "C12", "C44", "Lscale",
                "w_c", "L0", "L1", "L2", "L3", "U1", "U4", "dE0", "S"]
        return Model(d=d, h=h, bc=bc, **{k: p[k] for k in keys})

    # ---- App. B coefficients, literally -------------------------------------
    def M0(self):
        return self.dE0 + (self.L0 - self.L1 + self.L2 - self.L3)

    def M1(self, phi):
        return -(2 * self.L0 - 6 * self.L1 + 10 * self.L2 - 14 * self.L3) + 24 * self.U1 * phi ** 2 \
            + 72 * self.U4 * phi ** 2

    def M2(self, phi):
        return -(6 * self.L1 - 24 * self.L2 + 54 * self.L3) - 216 * self.U4 * phi ** 2 \
            - 144 * self.U4 * phi ** 3

    def M3(self):
        return -(16 * self.L2 - 80 * self.L3)

    def M4(self):
        return -40 * self.L3

    def M5(self, c):
        return -(24 * self.U1 * c ** 2 + 72 * self.U4 * (1 - 2 * c) * c ** 2)

    def M6(self, c):
        return 144 * self.U4 * c ** 3


# ----------------------------------------------------------------------------- grid operators
# P:224-233 per axis; multi-D = per-axis sums (reading R10).  Boundary conditions: periodic
# wrap, or -- homogeneous Neumann, reading R38 -- cell-centred mirror ghosts reflected about the boundary
# face (f_{-1-k} = f_k, f_{N+k} = f_{N-1-k}), even for c, eta, u and the mobility, ODD (sign
# flipped) for the stress in the outer derivative of the u rows (traction-free: n . sigma = 0 on the face).

def shift(f, j: int, s: int, d: int, bc: str = "periodic", parity: int = 1):
    """Value at i + s*e_j: periodic wrap, or the mirror ghost of a Neumann grid (parity -1: odd ghost)."""
    ax = d - 1 - j
    if bc == "periodic":
        return np.roll(f, -s, axis=ax)
    n = f.shape[ax]
    idx = np.arange(n) + s
    lo, hi = idx < 0, idx >= n
    src = np.where(lo, -1 - idx, np.where(hi, 2 * n - 1 - idx, idx))
    out = np.take(f, src, axis=ax)
    if parity == -1:
        shape = [1] * f.ndim
        shape[ax] = n
        out = out * np.where(lo | hi, -1.0, 1.0).reshape(shape)
    return out


def D_plus(f, j, h, d, bc="periodic"):
    """[D^+ f]_i = (f_{i+1} - f_i)/h."""
    return (shift(f, j, 1, d, bc) - f) / h


def D_minus(f, j, h, d, bc="periodic"):
    """[D^- f]_i = (f_i - f_{i-1})/h."""
    return (f - shift(f, j, -1, d, bc)) / h


def D_hat(f, j, h, d, bc="periodic", parity=1):
    """Central difference [D^ f]_i = (f_{i+1} - f_{i-1})/(2h)."""
    return (shift(f, j, 1, d, bc, parity) - shift(f, j, -1, d, bc, parity)) / (2 * h)


def laplacian(f, h, d, bc="periodic"):
    """[D^2 f]_i summed over axes: sum_j (f_{i+e_j} - 2 f_i + f_{i-e_j})/h^2 (R10)."""
    return sum((shift(f, j, 1, d, bc) - 2 * f + shift(f, j, -1, d, bc)) / h ** 2 for j in range(d))


def mobility_face(ca, kappa, j, d, bc="periodic"):
    """M~_{i+1/2 e_j} = kappa [c_i(1-c_i) + c_{i+1}(1-c_{i+1})]/2 at level n (reading R9)."""
    m = ca * (1 - ca)
    return kappa * (m + shift(m, j, 1, d, bc)) / 2


def div_M_grad(g, ca, kappa, h, d, bc="periodic"):
    """[D M~ D g]_i = sum_j [M~_{i+1/2}(g_{i+1}-g_i) - M~_{i-1/2}(g_i-g_{i-1})]/h^2.
    Neumann: the mirror ghost makes the flux through a boundary face vanish (n . M grad = 0)."""
    out = 0
    for j in range(d):
        mp = mobility_face(ca, kappa, j, d, bc)
        mm = shift(mp, j, -1, d, bc)
        out = out + (mp * (shift(g, j, 1, d, bc) - g) - mm * (g - shift(g, j, -1, d, bc))) / h ** 2
    return out


# ----------------------------------------------------------------------------- entropy Psi

def psi(z):
    """Psi(z) = z ln z + (1-z) ln(1-z)."""
    return z * np.log(z) + (1 - z) * np.log(1 - z)


def psi_deriv(z, s: int):
    """s-th derivative of Psi: Psi'(z) = ln(z/(1-z)); s>=2: (s-2)! [(-1)^s z^(1-s) + (1-z)^(1-s)].

    (Direct differentiation of P:68; needed by the Taylor polynomial Psi_S of P:452.)
    """
    if s == 1:
        return np.log(z) - np.log(1 - z)
    return math.factorial(s - 2) * ((-1) ** s * z ** (1 - s) + (1 - z) ** (1 - s))


def psiS_quotient(y1, y2, S: int):
    """Psi_S[y1, y2] of P:452-456, step by step.

    Psi_S(y, delta) = Psi(y) + sum_{s=1}^{2S} delta^s Psi^(s)(y)/s!
    Psi_S[y1,y2]   = [Psi_S(ybar, delta) - Psi_S(ybar, -delta)] / (2 delta), ybar = (y1+y2)/2,
                     delta = (y2 - y1)/2
    The numerator is a polynomial in delta whose s-th coefficient is a_s (1 - (-1)^s)
    (Psi(ybar) cancels); dividing it by 2*delta term by term ("a polynomial of the small
    parameter delta") gives sum_s a_s (1 - (-1)^s)/2 * delta^(s-1).
    """
    ybar = (y1 + y2) / 2
    delta = (y2 - y1) / 2
    total = 0
    for s in range(1, 2 * S + 1):
        if s % 2 == 0:          # (1 - (-1)^s)/2 = 0: the even terms vanish identically (skipping an
            continue            # exact zero leaves every bit of the sum unchanged)
        a_s = psi_deriv(ybar, s) / math.factorial(s)
        total = total + a_s * ((1 - (-1) ** s) // 2) * delta ** (s - 1)
    return total


def psi_exact_quotient(y1, y2):
    """Psi[y1,y2] = (Psi(y1) - Psi(y2))/(y1 - y2); unstable for y1 ~ y2."""
    return (psi(y1) - psi(y2)) / (y1 - y2)


# ----------------------------------------------------------------------------- free energies

def Q(k: int, x, y):
    """(x^k - y^k)/(x - y) written as the polynomial sum_{j<k} x^j y^(k-1-j)."""
    return sum(x ** j * y ** (k - 1 - j) for j in range(k))


def E1(m: Model, c, eta):
    """E1 = Phi(c, eta): the polynomial part of App. A's E_G with eta1=eta2=eta3=eta
    (P:1015-1017), phi_i = 1 - (eta_j+eta_k)/2 = 1 - eta (reading R3), E0_Ni := 0, and
    Phi = E^dis + E^ord(c,eta) - E^ord(c,1).
    """
    phi = 1 - eta
    e_dis = m.dE0 * c + c * (1 - c) * sum(Li * (2 * c - 1) ** i
                                         for i, Li in enumerate((m.L0, m.L1, m.L2, m.L3)))
    sum_phi2 = 3 * phi ** 2
    prod_phi = phi ** 3

    def e_ord(sp2, pp):
        return (6 * m.U1 * c ** 2 * sp2 - 2 * m.U1 * c ** 2 * sp2
                + 12 * m.U4 * (1 - 2 * c) * c ** 2 * sp2 - 48 * m.U4 * c ** 3 * pp)
    return e_dis + e_ord(sum_phi2, prod_phi) - e_ord(0.0 * sum_phi2, 0.0 * prod_phi)


def E2(m: Model, c, eta):
    """E2 = theta{ w_c Psi(c) + 3/4 Psi(c eta) + 1/4 Psi(c(4-3 eta)) } (w_c reading R2)."""
    return m.theta * (m.w_c * psi(c) + 0.75 * psi(c * eta) + 0.25 * psi(c * (4 - 3 * eta)))


def strain(m: Model, u):
    """eps_IJ = (D^_J u_I + D^_I u_J)/2 (reading R11 keeps I,J <= d)."""
    d = m.d
    du = [[D_hat(u[I], J, m.h, d, m.bc) for J in range(d)] for I in range(d)]   # du[I][J] = D^_J u_I
    return [[0.5 * (du[I][J] + du[J][I]) for J in range(d)] for I in range(d)]


def elastic_strain(m: Model, u, c, cbar0):
    """eps^el = eps(u) - eps0 (c - cbar0) I."""
    e = strain(m, u)
    for I in range(m.d):
        e[I][I] = e[I][I] - m.eps0 * (c - cbar0)
    return e


def stress(m: Model, eel):
    """sigma^el = Lscale C : eps^el for the cubic C of P:1069-1074 (Lscale: P:634)."""
    d = m.d
    tr = sum(eel[I][I] for I in range(d))
    sig = [[None] * d for _ in range(d)]
    for I in range(d):
        for J in range(d):
            if I == J:
                sig[I][J] = m.Lscale * (m.C12 * tr + (m.C11 - m.C12) * eel[I][I])
            else:
                sig[I][J] = m.Lscale * 2 * m.C44 * eel[I][J]
    return sig


def E3(m: Model, u, c, cbar0):
    """E3 = 1/2 eps^el : C : eps^el times Lscale."""
    e = elastic_strain(m, u, c, cbar0)
    d = m.d
    tr = sum(e[I][I] for I in range(d))
    sq = sum(e[I][I] ** 2 for I in range(d))
    off = sum(e[I][J] ** 2 for I in range(d) for J in range(I + 1, d))
    return 0.5 * m.Lscale * (m.C12 * tr ** 2 + (m.C11 - m.C12) * sq + 4 * m.C44 * off)


def E4(m: Model, c, eta):
    """E4 = gamma_c/2 [(D^+- c)^2] + 3 gamma_eta/2 [(D^+- eta)^2], summed over axes."""
    d, h = m.d, m.h
    out = 0
    for j in range(d):
        out = out + m.gamma_c / 2 * (D_plus(c, j, h, d, m.bc) ** 2 + D_minus(c, j, h, d, m.bc) ** 2) / 2
        out = out + 3 * m.gamma_eta / 2 * (D_plus(eta, j, h, d, m.bc) ** 2 + D_minus(eta, j, h, d, m.bc) ** 2) / 2
    return out


def energy_parts(m: Model, X, cbar0):
    """(E~1, E~2, E~3, E~4) summed with cell volume h^d (reading R35)."""
    c, eta, u = X[0], X[1], X[2:]
    vol = m.h ** m.d
    return (vol * np.sum(E1(m, c, eta)), vol * np.sum(E2(m, c, eta)),
            vol * np.sum(E3(m, u, c, cbar0)), vol * np.sum(E4(m, c, eta)))


def energy(m: Model, X, cbar0):
    """Total discrete free energy E~."""
    return sum(energy_parts(m, X, cbar0))


def mass(m: Model, X):
    """<c> = h^d sum c."""
    return m.h ** m.d * np.sum(X[0])


# ----------------------------------------------------------------------------- discrete variational derivatives

def G1(m: Model, ca, cb, ea, eb):
    """G~^1 of App. B."""
    pa, pb = 1 - ea, 1 - eb
    ch = (ca + cb) / 2
    phih = (pa + pb) / 2
    gc = ((m.M1(pa) + m.M1(pb)) / 2 * ch + (m.M2(pa) + m.M2(pb)) / 6 * Q(3, cb, ca)
          + m.M3() / 4 * Q(4, cb, ca) + m.M4() / 5 * Q(5, cb, ca) + m.M0())
    ge = (m.M5(ca) + m.M5(cb)) / 2 * phih + (m.M6(ca) + m.M6(cb)) / 6 * Q(3, pb, pa)
    return gc, ge


def G2S(m: Model, ca, cb, ea, eb):
    """G~^{2,S} of Eq. (D2-1), with the w_c weight of reading R2 on the Psi(c) term."""
    pa, pb = ca * ea, cb * eb                      # p = c eta
    qa, qb = ca * (4 - 3 * ea), cb * (4 - 3 * eb)  # q = c(4 - 3 eta)
    eh = (ea + eb) / 2
    ch = (ca + cb) / 2
    Pc = psiS_quotient(cb, ca, m.S)
    Pp = psiS_quotient(pb, pa, m.S)
    Pq = psiS_quotient(qb, qa, m.S)
    gc = m.theta / 4 * (4 * m.w_c * Pc + 3 * eh * Pp + (4 - 3 * eh) * Pq)
    ge = m.theta / 4 * (3 * ch * (Pp - Pq))
    return gc, ge


def G2_exact(m: Model, ca, cb, ea, eb):
    """G~^2 with exact quotients, Eq. (D2) -- used only by energy-law pins."""
    pa, pb = ca * ea, cb * eb
    qa, qb = ca * (4 - 3 * ea), cb * (4 - 3 * eb)
    eh = (ea + eb) / 2
    ch = (ca + cb) / 2
    Pc = psi_exact_quotient(cb, ca)
    Pp = psi_exact_quotient(pb, pa)
    Pq = psi_exact_quotient(qb, qa)
    gc = m.theta / 4 * (4 * m.w_c * Pc + 3 * eh * Pp + (4 - 3 * eh) * Pq)
    ge = m.theta / 4 * (3 * ch * (Pp - Pq))
    return gc, ge


def trace_stress(m: Model, u, c, cbar0):
    """T(u, c) = tr sigma^el(u, c)."""
    sig = stress(m, elastic_strain(m, u, c, cbar0))
    return sum(sig[I][I] for I in range(m.d))


def G3(m: Model, Xa, Xb, cbar0):
    """G~^3 = (-eps0 I:C:[eps^el]^{n+1/2}, 0) (multi-D via P:1105, reading R12)."""
    Ta = trace_stress(m, Xa[2:], Xa[0], cbar0)
    Tb = trace_stress(m, Xb[2:], Xb[0], cbar0)
    return -m.eps0 * (Ta + Tb) / 2, 0 * Ta


def G4(m: Model, Xa, Xb):
    """G~^4 = (-gamma_c D^2 c^{n+1/2}, -3 gamma_eta D^2 eta^{n+1/2})."""
    ch = (Xa[0] + Xb[0]) / 2
    eh = (Xa[1] + Xb[1]) / 2
    return -m.gamma_c * laplacian(ch, m.h, m.d, m.bc), -3 * m.gamma_eta * laplacian(eh, m.h, m.d, m.bc)


def G_S(m: Model, Xa, Xb, cbar0):
    """G~^S = G~^1 + G~^{2,S} + G~^3 + G~^4."""
    g1 = G1(m, Xa[0], Xb[0], Xa[1], Xb[1])
    g2 = G2S(m, Xa[0], Xb[0], Xa[1], Xb[1])
    g3 = G3(m, Xa, Xb, cbar0)
    g4 = G4(m, Xa, Xb)
    return g1[0] + g2[0] + g3[0] + g4[0], g1[1] + g2[1] + g3[1] + g4[1]


def residual(m: Model, Xa, Xb, dt, cbar0):
    """Nonlinear residual F(X^b) of scheme NSOA-1, rows as in reading R36:

    F_c   = (c^b - c^a)/dt - D M~ D G_c          (V_t = -A~ G, A~ = diag(-D M~ D, 1))
    F_eta = (eta^b - eta^a)/dt + G_eta
    F_u_I = sum_J D^_J sigma^el_IJ(u^b, c^b)     ([D^ sigma^el]^{n+1} = 0)
    """
    d = m.d
    gc, ge = G_S(m, Xa, Xb, cbar0)
    F = np.empty_like(Xb)
    F[0] = (Xb[0] - Xa[0]) / dt - div_M_grad(gc, Xa[0], m.kappa, m.h, d, m.bc)
    F[1] = (Xb[1] - Xa[1]) / dt + ge
    sig = stress(m, elastic_strain(m, Xb[2:], Xb[0], cbar0))
    for I in range(d):     # Neumann: odd stress ghosts across the J faces (traction-free, reading R38)
        F[2 + I] = sum(D_hat(sig[I][J], J, m.h, d, m.bc, -1) for J in range(d))
    return F


def admissible(X) -> bool:
    """0 < c, p = c eta, q = c(4 - 3 eta) < 1 and all finite (domain of Psi; reading R17)."""
    c, eta = np.real(X[0]), np.real(X[1])
    if not np.all(np.isfinite(np.real(X))):
        return False
    p, q = c * eta, c * (4 - 3 * eta)
    return bool(np.all((c > 0) & (c < 1) & (p > 0) & (p < 1) & (q > 0) & (q < 1)))
