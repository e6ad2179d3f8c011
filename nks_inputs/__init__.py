"""Seeded synthetic inputs and parameter presets shared by the oracle and the CUDA path.

This module holds NO arithmetic of the method (no free energy, no stencil, no
solver step).  It only supplies:

* ``model_default()``   -- the documented non-paper coefficient set (DESIGN.md
  "Readings" R6-R8) as plain numbers;
* ``solver_default()``  -- tolerances / controller constants (Z16-Z24);
* ``CONFIGS``           -- the five BASELINE.json configurations as dicts;
* ``initial_fields()``  -- the seeded random initial state (Z25/Z26);
* ``perturbed_state()`` / ``random_direction()`` -- microbenchmark inputs.

Both ``oracle/`` and ``paper_2209_08001_b200`` read these values; each side
derives everything else (M0..M6, K, strains, ...) on its own.
"""
from __future__ import annotations

import numpy as np

# --------------------------------------------------------------------------------------
# Model parameters (dimensionless).  Citations: P:n = /root/reference/PAPER.md line n.
# --------------------------------------------------------------------------------------

R_GAS = 8.314462618          # J/(mol K)
T_BODY = 1037.0              # K, P:1024 (body text); Z5
V_M = 1.48e-5                # m^3/mol
DELTA_E = 3.3e7              # J/m^3
LENGTH_SCALE = 1.5e-9        # m


def model_default() -> dict:
    """Model-default parameter set (NOT printed in the paper; R6/R7/R8).

    * theta = R T / (V_m dE) with T = 1037 K            -> 17.6538...
    * gamma_c, gamma_eta: P:962 nondimensionalised by dE * L^2   -> 33.670, 0.080808
    * kappa = 0.008; eps0 = 0.049; Lscale (the script-L of P:634) = 1
    * CALPHAD coefficients L0..L3, U1, U4 in units of V_m dE: not printed;
      fitted so that the reduced Gibbs energy has the printed wells (0.137, 1) and
      (0.229, 0.02) with a common tangent.
    * dE0 = (E0_Al - E0_Ni)/(V_m dE) chosen so that M0 = 0.
    * C11, C12, C44: not printed; invented cubic constants.
    * w_c = 1: the Psi(c) term of the main text is kept.
    """
    L = (-34.1306, 34.7869, -32.6177, 27.6058)
    theta = R_GAS * T_BODY / (V_M * DELTA_E)
    scale = DELTA_E * LENGTH_SCALE ** 2
    return {
        "theta": theta,
        "gamma_c": 2.5e-9 / scale,
        "gamma_eta": 6.0e-12 / scale,
        "kappa": 0.008,
        "eps0": 0.049,
        "C11": 7500.0,
        "C12": 4500.0,
        "C44": 3750.0,
        "Lscale": 1.0,
        "w_c": 1.0,
        "L0": L[0], "L1": L[1], "L2": L[2], "L3": L[3],
        "U1": -19.6708,
        "U4": 3.5,
        "dE0": -(L[0] - L[1] + L[2] - L[3]),
        "S": 10,
    }


def solver_default() -> dict:
    """Solver and controller constants."""
    return {
        "newton_rtol": 1e-11, "newton_atol": 0.0,      # Z16 (BASELINE Newton rtol 1e-11)
        "gmres_rtol": 1e-10, "gmres_atol": 0.0,        # Z16 (xi_r = 1e-10)
        "newton_maxit": 50, "gmres_restart": 30, "gmres_maxit": 10000,   # Z18, Z24
        "ls_alpha": 1e-4, "ls_max_halvings": 10,       # Z17
        "zeta": 100.0, "dt_min": 0.01, "dt_max": 2.0, "dt_init": 0.01,
        "dt_floor_factor": 1.0 / 1024.0,               # Z24
        "xd_norm": "rms",                              # Z23
    }


# --------------------------------------------------------------------------------------
# BASELINE.json configurations.  shape is C order (z, y, x), x fastest.
# --------------------------------------------------------------------------------------

CONFIGS = {
    1: {"name": "2d_64", "shape": (64, 64), "h": 0.25, "mode": "fixed", "dt": 0.01, "steps": 10,
        "nsub": (1, 1), "overlap": 2},
    2: {"name": "2d_512", "shape": (512, 512), "h": 0.25, "mode": "adaptive", "steps": 200,
        "nsub": (4, 4), "overlap": 2},
    3: {"name": "3d_128", "shape": (128, 128, 128), "h": 0.25, "mode": "adaptive", "steps": 50,
        "nsub": (8, 8, 8), "overlap": 2},
    4: {"name": "3d_256", "shape": (256, 256, 256), "h": 0.25, "mode": "adaptive", "steps": 20,
        "nsub": (8, 8, 8), "overlap": 2},
    5: {"name": "3d_512_micro", "shape": (512, 512, 512), "h": 0.25, "mode": "micro", "dt": 0.01},
}

CBAR = 0.1622          # V_f = 17.5 %
ETA_MEAN = 0.1


def initial_fields(shape, seed: int = 0, cbar: float = CBAR, c_amp: float = 0.005,
                   eta_mean: float = ETA_MEAN, eta_amp: float = 0.01):
    """Seeded initial (c0, eta0), C order over shape (x fastest).

    Draw order: first c noise U(-c_amp, c_amp), then eta noise U(-eta_amp, eta_amp),
    both from numpy PCG64 ``default_rng(seed)``.  c0 = cbar + noise, eta0 =
    eta_mean + noise (P:714 mean; BASELINE amplitude).
    """
    rng = np.random.default_rng(seed)
    n = int(np.prod(shape))
    c_noise = rng.uniform(-c_amp, c_amp, n)
    eta_noise = rng.uniform(-eta_amp, eta_amp, n)
    c0 = (cbar + c_noise).reshape(shape)
    eta0 = (eta_mean + eta_noise).reshape(shape)
    return c0, eta0


def perturbed_state(c, eta, seed: int = 1, amp: float = 1e-3):
    """X^b = X^n + U(-amp, amp) on c and eta: keeps delta != 0 in Psi_S."""
    rng = np.random.default_rng(seed)
    dc = rng.uniform(-amp, amp, c.size).reshape(c.shape)
    de = rng.uniform(-amp, amp, eta.size).reshape(eta.shape)
    return c + dc, eta + de


def random_direction(nfields: int, shape, seed: int = 1, amp: float = 1.0):
    """v ~ U(-amp, amp) on all 2+d components, shape (nfields, *shape)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-amp, amp, (nfields,) + tuple(shape))


def random_displacement(d: int, shape, seed: int = 2, amp: float = 1e-3):
    """A smooth-free random displacement field, used only as a test input (not an equilibrium)."""
    rng = np.random.default_rng(seed)
    return rng.uniform(-amp, amp, (d,) + tuple(shape))


def sphere_fields(shape, h: float, radius: float, c_in: float, eta_in: float,
                  c_out: float, eta_out: float):
    """Single embedded particle at the domain centre: a NEXT-row workload."""
    grids = np.meshgrid(*[(np.arange(n) + 0.5) * h for n in shape], indexing="ij")
    centre = [n * h / 2 for n in shape]
    r2 = sum((g - c0) ** 2 for g, c0 in zip(grids, centre))
    inside = r2 <= radius * radius
    c = np.where(inside, c_in, c_out).astype(np.float64)
    eta = np.where(inside, eta_in, eta_out).astype(np.float64)
    return c, eta


__all__ = ["model_default", "solver_default", "CONFIGS", "initial_fields", "perturbed_state",
           "random_direction", "random_displacement", "sphere_fields", "CBAR", "ETA_MEAN"]
