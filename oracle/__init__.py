"""CPU fp64 ORACLE for the NKS time step of arXiv 2209.08001 -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import anything under ``oracle/``.  The product
package ``paper_2209_08001_b200`` never imports it, and this package never
imports the product: the two share no code (only the seeded generators in
``nks_inputs``).

Plain, slow, obviously-correct NumPy/SciPy, fp64 throughout, each function
citing the PAPER.md passage (``P:n`` = line n of /root/reference/PAPER.md) it
follows.  Readings of silent/garbled passages are DESIGN.md R1..R36 (= SURVEY
8(c).2 Z1..Z36).

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) tie every function to something
other than itself: closed forms, mpmath high-precision values, DVD identities,
complex-step derivatives, brute force on tiny grids, dense LU.

Parity status per function (see DESIGN.md section "Oracle pins"):
  scheme.*            pinned (DVD identities, closed forms, symmetries, mpmath)
  jacobian.*          pinned (complex-step J.v, central FD, rank / null space)
  solver.newton_step  pinned (quadratic convergence, dense-LU agreement, mass, energy law)
  solver.controller   pinned (closed forms of Eq. sencondt)
  pc.* (RAS/BILU(0))  pinned (ILU(0) defining property, exact-LU special case, partition of unity)
  absolute physics vs the paper's figures: "parity unpinned" (coefficients are model-default).
"""
from . import scheme, jacobian, solver, pc  # noqa: F401
