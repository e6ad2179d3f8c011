"""Oracle: restricted additive Schwarz with point-block ILU(0) subdomain solves (TEST INFRASTRUCTURE ONLY).

The paper names the preconditioners (classical AS, left-RAS Cai-Sarkis 1999, right-RAS;
P:581-586) and the subdomain solver ILU(0) but gives no algorithm; this module
writes out the textbook definitions with the readings of DESIGN.md:

* boxes (R19/R20): the grid is split into nsub_J boxes per axis (the first n_J mod nsub_J
  boxes get one extra cell); each box is extended by delta cells on each side; the extended
  box is a NON-periodic local grid whose local point l maps to global (start - delta + l) mod n.
  An axis with a single box therefore self-overlaps across the periodic seam.
* A_i = J restricted to the extended box: block (l, l+o) = J block (g(l), offset o) for every
  footprint offset o with l+o inside the box; couplings leaving the box are dropped.
* ILU(0) (R21): natural (x fastest) ordering of the local points, point blocks of size 2+d,
  pattern = the block footprint; the unique unit-lower L, upper U with (LU)_pq = A_pq on the
  pattern, computed by the IKJ elimination.
* ILU(k) (Table 1: ILU(1), ILU(2), LU): the same IKJ elimination on the
  level-of-fill pattern of Saad's ILU(p) (symbolic phase `fill_levels`); no level limit gives the
  exact block LU (no pivoting, natural order).
* left-RAS (R19): z = sum_i R_i^{0T} (L_i U_i)^{-1} R_i^delta r -- gather on the extended box,
  scatter the owned points only.
"""
from __future__ import annotations

import itertools

import numpy as np


def footprint(d: int):
    """Block-stencil offsets of J: |o|_1 <= 2 (13 points in 2D, 25 in 3D); o = (ox, oy[, oz])."""
    rng = range(-2, 3)
    offs = [o for o in itertools.product(rng, repeat=d) if sum(abs(x) for x in o) <= 2]
    return offs


def split_axis(n: int, nsub: int):
    """Owned (start, length) per box along one axis."""
    base, rem = divmod(n, nsub)
    out, s = [], 0
    for b in range(nsub):
        ln = base + (1 if b < rem else 0)
        out.append((s, ln))
        s += ln
    return out


def boxes(shape, nsub, delta, bc="periodic"):
    """List of boxes; each: dict(start[j], own[j], ext[j], s0[j], d0[j]) indexed by axis j (0 = x).  Periodic:
    the box is extended by delta on each side (wrapping, self-overlapping on a one-box axis, R20).  Neumann
    (R38): the extension stops at the walls -- there is nothing beyond them."""
    d = len(shape)
    n_xyz = [shape[d - 1 - j] for j in range(d)]
    per_axis = [split_axis(n_xyz[j], nsub[j]) for j in range(d)]
    out = []
    for combo in itertools.product(*[range(nsub[j]) for j in reversed(range(d))]):
        combo = tuple(reversed(combo))   # combo[j] = box index along axis j; x varies fastest
        start = [per_axis[j][combo[j]][0] for j in range(d)]
        own = [per_axis[j][combo[j]][1] for j in range(d)]
        if bc == "periodic":
            s0 = [start[j] - delta for j in range(d)]
            ext = [own[j] + 2 * delta for j in range(d)]
        else:
            s0 = [max(start[j] - delta, 0) for j in range(d)]
            ext = [min(start[j] + own[j] + delta, n_xyz[j]) - s0[j] for j in range(d)]
        d0 = [start[j] - s0[j] for j in range(d)]
        out.append({"start": start, "own": own, "ext": ext, "delta": delta, "n": n_xyz, "s0": s0, "d0": d0})
    return out


def local_points(box):
    """Local points in natural order (x fastest): list of tuples l = (lx, ly[, lz])."""
    d = len(box["ext"])
    pts = []
    for lz in range(box["ext"][2] if d == 3 else 1):
        for ly in range(box["ext"][1]):
            for lx in range(box["ext"][0]):
                pts.append((lx, ly, lz)[:d])
    return pts


def global_index(box, l):
    """Flat C-order global index of local point l."""
    d = len(l)
    s0 = box.get("s0", [box["start"][j] - box["delta"] for j in range(d)])
    g = [(s0[j] + l[j]) % box["n"][j] for j in range(d)]
    idx = 0
    for j in reversed(range(d)):
        idx = idx * box["n"][j] + g[j]
    return idx


def box_blocks(J, box, nf, npts_global):
    """A_i as a dict {(p, q): nf x nf block} over local point indices (natural order)."""
    d = len(box["ext"])
    pts = local_points(box)
    index = {l: i for i, l in enumerate(pts)}
    Jc = J.tocsr()
    A = {}
    offs = footprint(d)
    for p, l in enumerate(pts):
        gp = global_index(box, l)
        rows = [f * npts_global + gp for f in range(nf)]
        sub = Jc[rows, :].toarray()
        for o in offs:
            lq = tuple(l[j] + o[j] for j in range(d))
            if lq not in index:
                continue
            gq = global_index(box, lq)
            cols = [f * npts_global + gq for f in range(nf)]
            A[(p, index[lq])] = sub[:, cols].copy()
    return A, pts


def bilu0(A, npts):
    """Point-block ILU(0), IKJ variant: returns (L, U) dicts on the pattern of A (L unit lower)."""
    W = {k: v.copy() for k, v in A.items()}
    rows = {}
    for (p, q) in W:
        rows.setdefault(p, []).append(q)
    for p in rows:
        rows[p].sort()
    for i in range(npts):
        for k in [q for q in rows[i] if q < i]:
            W[(i, k)] = W[(i, k)] @ np.linalg.inv(W[(k, k)])
            for j in [q for q in rows[k] if q > k]:
                if (i, j) in W:
                    W[(i, j)] = W[(i, j)] - W[(i, k)] @ W[(k, j)]
    L = {k: v for k, v in W.items() if k[1] < k[0]}
    U = {k: v for k, v in W.items() if k[1] >= k[0]}
    return L, U


def fill_levels(A, npts, k):
    """Symbolic ILU(k) (Saad, Iterative Methods, Sec. 10.3.3 / Alg. 10.5): level-of-fill of every block
    entry, lev(i,j) = 0 on the pattern of A and lev(i,j) = min over k < min(i,j) of
    lev(i,k) + lev(k,j) + 1 for fill, keeping only entries with lev <= k.  k = None: no limit
    (the pattern of the exact LU factors).  Returns {row: {col: level}}."""
    rows = {i: {} for i in range(npts)}
    for (p, q) in A:
        rows[p][q] = 0
    for i in range(npts):
        row = rows[i]
        done = set()
        while True:
            cand = [q for q in row if q < i and q not in done]
            if not cand:
                break
            kk = min(cand)
            done.add(kk)
            lik = row[kk]
            for j, lkj in rows[kk].items():
                if j <= kk:
                    continue
                lev = lik + lkj + 1
                if (k is None or lev <= k) and (j not in row or row[j] > lev):
                    row[j] = lev
    return rows


def biluk(A, npts, k):
    """Point-block ILU(k), IKJ variant on the level-k pattern (Saad Alg. 10.5 with blocks; k = 0 is
    ILU(0), k = None the exact block LU without pivoting).  Returns (L, U) dicts (L unit lower)."""
    levels = fill_levels(A, npts, k)
    nf = next(iter(A.values())).shape[0]
    W = {}
    for i in range(npts):
        for j in levels[i]:
            W[(i, j)] = A[(i, j)].copy() if (i, j) in A else np.zeros((nf, nf))
    cols = {i: sorted(levels[i]) for i in range(npts)}
    for i in range(npts):
        for kk in [q for q in cols[i] if q < i]:
            W[(i, kk)] = W[(i, kk)] @ np.linalg.inv(W[(kk, kk)])
            for j in [q for q in cols[kk] if q > kk]:
                if (i, j) in W:
                    W[(i, j)] = W[(i, j)] - W[(i, kk)] @ W[(kk, j)]
    L = {key: v for key, v in W.items() if key[1] < key[0]}
    U = {key: v for key, v in W.items() if key[1] >= key[0]}
    return L, U


def lu_solve(L, U, r, npts):
    """Solve (L U) x = r with r of shape (npts, nf): forward then backward block substitution."""
    rowsL, rowsU = {}, {}
    for (p, q) in L:
        rowsL.setdefault(p, []).append(q)
    for (p, q) in U:
        rowsU.setdefault(p, []).append(q)
    y = np.zeros_like(r)
    for i in range(npts):
        acc = r[i].copy()
        for k in rowsL.get(i, []):
            acc -= L[(i, k)] @ y[k]
        y[i] = acc
    x = np.zeros_like(r)
    for i in reversed(range(npts)):
        acc = y[i].copy()
        for j in rowsU.get(i, []):
            if j > i:
                acc -= U[(i, j)] @ x[j]
        x[i] = np.linalg.solve(U[(i, i)], acc)
    return x


def is_owned(box, l):
    d = len(l)
    d0 = box.get("d0", [box["delta"]] * d)
    return all(d0[j] <= l[j] < d0[j] + box["own"][j] for j in range(d))


class RAS:
    """Schwarz preconditioner with BILU(0) (or exact LU, ``exact=True``) subdomain solves.

    variant (Cai-Sarkis):
      "ras"  z = sum_i R_i^{0T} A_i^{-1} R_i^delta r      left restricted additive Schwarz
      "as"   z = sum_i R_i^{deltaT} A_i^{-1} R_i^delta r  classical additive Schwarz
      "rras" z = sum_i R_i^{deltaT} A_i^{-1} R_i^0 r      right-restricted (input restricted to owned points)
    """

    def __init__(self, J, shape, nf, nsub, delta, exact: bool = False, variant: str = "ras", fill=0, bc="periodic"):
        """fill: subdomain solver ILU(fill) (0 = BILU(0), the default; k > 0 = level-k ILU; None = the
        exact block LU through the level-of-fill path); exact=True: dense LAPACK solve of A_i."""
        assert variant in ("ras", "as", "rras")
        self.variant = variant
        self.shape = shape
        self.nf = nf
        self.npts = int(np.prod(shape))
        self.boxes = boxes(shape, nsub, delta, bc)
        self.fact = []
        for b in self.boxes:
            A, pts = box_blocks(J, b, nf, self.npts)
            if exact:
                self.fact.append(("lu", self._dense(A, len(pts)), pts))
            elif fill == 0:
                L, U = bilu0(A, len(pts))
                self.fact.append(("ilu", (L, U), pts))
            else:
                L, U = biluk(A, len(pts), fill)
                self.fact.append(("ilu", (L, U), pts))

    def _dense(self, A, npts):
        nf = self.nf
        M = np.zeros((npts * nf, npts * nf))
        for (p, q), blk in A.items():
            M[p * nf:(p + 1) * nf, q * nf:(q + 1) * nf] = blk
        return M

    def apply(self, r):
        """r, z: field-major arrays of shape (nf, *grid)."""
        nf = self.nf
        rf = r.reshape(nf, self.npts)
        z = np.zeros_like(rf)
        for b, (kind, fac, pts) in zip(self.boxes, self.fact):
            gidx = [global_index(b, l) for l in pts]
            rl = rf[:, gidx].T.copy()                  # R_i^delta r   (npts_box, nf)
            if self.variant == "rras":                 # R_i^0 r: zero on the overlap
                for p, l in enumerate(pts):
                    if not is_owned(b, l):
                        rl[p] = 0.0
            if kind == "lu":
                xl = np.linalg.solve(fac, rl.ravel()).reshape(len(pts), nf)
            else:
                xl = lu_solve(fac[0], fac[1], rl, len(pts))
            for p, l in enumerate(pts):
                if self.variant == "ras":              # R_i^{0T}: owned points only
                    if is_owned(b, l):
                        z[:, gidx[p]] = xl[p]
                else:                                  # R_i^{deltaT}: every box point adds its value
                    z[:, gidx[p]] += xl[p]
        return z.reshape(r.shape)
