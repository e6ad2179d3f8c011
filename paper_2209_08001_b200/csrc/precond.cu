// Restricted additive Schwarz preconditioner with point-block ILU(0) subdomain solves (P:581-586,
// P:789-797): box geometry (host), analytic point-block Jacobian assembly (K4), level-scheduled
// BILU(0) factorisation (K5) and the RAS apply with forward/backward wavefront sweeps (K6).
//
// Boxes (R19/R20): nsub_j boxes per axis, the first n_j mod nsub_j one cell longer,
// each extended by delta cells per side into a NON-periodic local grid (an axis with one box
// self-overlaps across the periodic seam).  Local natural order (x fastest); level of a local
// point l = lx + 2 ly + 3 lz (the exact dependency depth of the |o|_1 <= 2 block pattern, R21;
// i+j+k would violate the (1,-1,0)/(1,0,-1)/(0,1,-1) couplings).  Box-local arrays are stored in
// level order ("positions") so one level is a contiguous, coalesced range.
#include <cooperative_groups.h>

#include <algorithm>
#include <numeric>

#include "nks_internal.cuh"

namespace nks {

// ------------------------------------------------------------------------------------------ host geometry
static long long nat_key(const int o[3]) { return ((long long)o[2] * 64 + o[1]) * 64 + o[0]; }

void build_slot_tables(int dim, BoxSet& B) {
  int cnt = 0;
  int offs[kMaxSlots][3];
  for (int oz = (dim == 3 ? -2 : 0); oz <= (dim == 3 ? 2 : 0); ++oz)
    for (int oy = -2; oy <= 2; ++oy)
      for (int ox = -2; ox <= 2; ++ox)
        if (std::abs(ox) + std::abs(oy) + std::abs(oz) <= 2) {
          offs[cnt][0] = ox; offs[cnt][1] = oy; offs[cnt][2] = oz; ++cnt;
        }
  // sort by natural order key
  int idx[kMaxSlots];
  std::iota(idx, idx + cnt, 0);
  std::sort(idx, idx + cnt, [&](int a, int b) { return nat_key(offs[a]) < nat_key(offs[b]); });
  B.nslots = cnt;
  B.nlower = B.nupper = 0;
  for (int s = 0; s < cnt; ++s) {
    for (int k = 0; k < 3; ++k) B.off[s][k] = offs[idx[s]][k];
    const long long key = nat_key(B.off[s]);
    if (key < 0) B.lower[B.nlower++] = s;
    else if (key > 0) B.upper[B.nupper++] = s;
    else B.diag = s;
  }
  auto find = [&](int ox, int oy, int oz) {
    for (int s = 0; s < cnt; ++s)
      if (B.off[s][0] == ox && B.off[s][1] == oy && B.off[s][2] == oz) return s;
    return -1;
  };
  for (int ia = 0; ia < B.nlower; ++ia) {
    const int sa = B.lower[ia];
    B.npairs[ia] = 0;
    for (int ib = 0; ib < B.nupper; ++ib) {
      const int sb = B.upper[ib];
      const int t = find(B.off[sa][0] + B.off[sb][0], B.off[sa][1] + B.off[sb][1], B.off[sa][2] + B.off[sb][2]);
      if (t < 0) continue;
      B.pair_b[ia][B.npairs[ia]] = sb;
      B.pair_t[ia][B.npairs[ia]] = t;
      ++B.npairs[ia];
    }
  }
}


static void split_axis(int n, int nsub, std::vector<int>& start, std::vector<int>& len) {
  const int base = n / nsub, rem = n % nsub;
  int s = 0;
  for (int b = 0; b < nsub; ++b) {
    const int l = base + (b < rem ? 1 : 0);
    start.push_back(s);
    len.push_back(l);
    s += l;
  }
}

// Box extents per axis.  A z-slab state (zghost > 0) splits only its own planes along z, and its
// boxes address the local array directly: the overlap planes are ghost planes, which hold the
// periodic neighbours' values, so no z wrap is needed (RAS needs one width-delta halo
// of its input, assembly one of width delta+1).
static void split_boxes(const nks_grid& g, std::vector<int> (&st)[3], std::vector<int> (&ln)[3]) {
  split_axis(g.n[0], g.nsub[0], st[0], ln[0]);
  if (g.yghost > 0) {             // a pencil: the own rows, boxes addressing the ghost rows as their overlap
    split_axis(g.n[1] - 2 * g.yghost, g.nsub[1], st[1], ln[1]);
    for (auto& v : st[1]) v += g.yghost;
  } else {
    split_axis(g.n[1], g.nsub[1], st[1], ln[1]);
  }
  if (g.zghost > 0) {
    split_axis(g.n[2] - 2 * g.zghost, g.nsub[2], st[2], ln[2]);
    for (auto& v : st[2]) v += g.zghost;
  } else {
    split_axis(g.n[2], g.nsub[2], st[2], ln[2]);
  }
}

// Extended box along one axis: the owned range [start, start + len) plus `dl` cells per side.  Periodic:
// always 2 dl more (wrapping; a one-box axis self-overlaps, R20).  Neumann (bc = 1, R38): clipped at the
// walls.  s0 = global coordinate of local 0 (may be negative on a periodic axis), e = extent, d0 = first
// owned local index.
void box_axis(const nks_grid& g, int j, int start, int len, int dl, int& s0, int& e, int& d0) {
  if (g.bc == 1) {
    s0 = std::max(start - dl, 0);
    e = std::min(start + len + dl, g.n[j]) - s0;
  } else {
    s0 = start - dl;
    e = len + 2 * dl;
  }
  d0 = start - s0;
}

long long box_positions(const nks_grid& g) {
  std::vector<int> st[3], ln[3];
  long long P = 0;
  split_boxes(g, st, ln);
  const int dz = g.dim == 3 ? g.overlap : 0;
  for (int bz = 0; bz < g.nsub[2]; ++bz)
    for (int by = 0; by < g.nsub[1]; ++by)
      for (int bx = 0; bx < g.nsub[0]; ++bx) {
        int s0, e[3], d0;
        box_axis(g, 0, st[0][bx], ln[0][bx], g.overlap, s0, e[0], d0);
        box_axis(g, 1, st[1][by], ln[1][by], g.overlap, s0, e[1], d0);
        box_axis(g, 2, st[2][bz], ln[2][bz], dz, s0, e[2], d0);
        P += (long long)e[0] * e[1] * e[2];
      }
  return P;
}

HostBoxes build_boxes_host(const nks_grid& g, const BoxSet& B, const IlukPattern* K) {
  // wavefront level lx + la ly + lb lz (R21: la = 2, lb = 3 for the ILU(0) pattern); with a level-k
  // pattern K, the slot offsets come from K and a row lacks the entries its level-k pattern drops
  const int la = K ? K->la : 2, lb = K ? K->lb : 3;
  const int nsl = K ? K->nslots : B.nslots;
  HostBoxes H;
  std::vector<int> st[3], ln[3];
  split_boxes(g, st, ln);
  const int delta = g.overlap;
  const int dz = g.dim == 3 ? delta : 0;
  H.P = box_positions(g);
  H.gidx.assign(H.P, 0);
  H.nbr.assign((size_t)nsl * H.P, -1);
  H.box_pos_off.push_back(0);
  H.box_lev_off.push_back(0);
  long long base = 0;
  for (int bz = 0; bz < g.nsub[2]; ++bz)
    for (int by = 0; by < g.nsub[1]; ++by)
      for (int bx = 0; bx < g.nsub[0]; ++bx) {
        int e[3], s0[3], d0[3];
        box_axis(g, 0, st[0][bx], ln[0][bx], delta, s0[0], e[0], d0[0]);
        box_axis(g, 1, st[1][by], ln[1][by], delta, s0[1], e[1], d0[1]);
        box_axis(g, 2, st[2][bz], ln[2][bz], dz, s0[2], e[2], d0[2]);
        const int own[3] = {ln[0][bx], ln[1][by], ln[2][bz]};
        const long long np = (long long)e[0] * e[1] * e[2];
        const int nlev = (e[0] - 1) + la * (e[1] - 1) + lb * (e[2] - 1) + 1;
        int ext_q = -1;
        if (K)
          for (size_t q = 0; q < K->ext.size(); ++q)
            if (K->ext[q][0] == e[0] && K->ext[q][1] == e[1] && K->ext[q][2] == e[2]) ext_q = (int)q;
        // counting sort by level, natural order within a level
        std::vector<int> count(nlev + 1, 0);
        for (int lz = 0; lz < e[2]; ++lz)
          for (int ly = 0; ly < e[1]; ++ly)
            for (int lx = 0; lx < e[0]; ++lx) count[lx + la * ly + lb * lz + 1]++;
        for (int l = 0; l < nlev; ++l) count[l + 1] += count[l];
        std::vector<int> lvstart(count.begin(), count.end());
        for (int l = 0; l < nlev; ++l) H.max_width = std::max(H.max_width, count[l + 1] - count[l]);
        H.max_levels = std::max(H.max_levels, nlev);
        std::vector<int> posof(np);
        std::vector<int> fill(count.begin(), count.end() - 1);
        for (int lz = 0; lz < e[2]; ++lz)
          for (int ly = 0; ly < e[1]; ++ly)
            for (int lx = 0; lx < e[0]; ++lx) {
              const int lin = (lz * e[1] + ly) * e[0] + lx;
              posof[lin] = fill[lx + la * ly + lb * lz]++;
            }
        for (int lz = 0; lz < e[2]; ++lz)
          for (int ly = 0; ly < e[1]; ++ly)
            for (int lx = 0; lx < e[0]; ++lx) {
              const int lin = (lz * e[1] + ly) * e[0] + lx;
              const long long pos = base + posof[lin];
              const int l[3] = {lx, ly, lz};
              int gc[3];
              bool owned = true;
              for (int j = 0; j < 3; ++j) {
                int v = (s0[j] + l[j]) % g.n[j];
                if (v < 0) v += g.n[j];
                gc[j] = v;
                if (l[j] < d0[j] || l[j] >= d0[j] + own[j]) owned = false;
              }
              const int gi = (gc[2] * g.n[1] + gc[1]) * g.n[0] + gc[0];
              H.gidx[pos] = owned ? gi : ~gi;
              for (int s = 0; s < nsl; ++s) {
                const int* o = K ? K->off[s].data() : B.off[s];
                const int q[3] = {lx + o[0], ly + o[1], lz + o[2]};
                if (q[0] < 0 || q[0] >= e[0] || q[1] < 0 || q[1] >= e[1] || q[2] < 0 || q[2] >= e[2]) continue;
                if (K && !K->present[ext_q][(size_t)lin * nsl + s]) continue;
                const int qlin = (q[2] * e[1] + q[1]) * e[0] + q[0];
                H.nbr[(size_t)s * H.P + pos] = (int)(base + posof[qlin]);
              }
            }
        for (int l = 0; l <= nlev; ++l) H.lev_ptr.push_back((int)(base + lvstart[l]));
        H.box_lev_off.push_back((int)H.lev_ptr.size());
        base += np;
        H.box_pos_off.push_back((int)base);
      }
  return H;
}

// ------------------------------------------------------------------------------------------ K4 assembly
__device__ __forceinline__ int wrapi(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// Block (nf x nf) of J at grid point (x,y,z), column point (x,y,z)+o.  Rows/cols: c, eta, u_1..u_d.
__device__ void jac_block(const DevParams& P, const double* __restrict__ Xa, const double* __restrict__ jac4,
                          int x, int y, int z, const int o[3], double* blk, int nf) {
  const int d = P.dim;
  const long long N = P.N;
  auto gid = [&](int dx, int dy, int dz) -> long long {
    return ((long long)wrapi(z + dz, P.nz) * P.ny + wrapi(y + dy, P.ny)) * P.nx + wrapi(x + dx, P.nx);
  };
  for (int k = 0; k < nf * nf; ++k) blk[k] = 0.0;
  const int l1 = abs(o[0]) + abs(o[1]) + abs(o[2]);
  const double ih2 = P.inv_h2;
  // ---- c row: -sum_a W_{i,i+a} dG_c(i+a)/dX(i+o)  (+ 1/dt on the diagonal)
  {
    const double cai = Xa[gid(0, 0, 0)];
    const double mi = cai * (1.0 - cai);
    const double beta_nb = -0.5 * P.gamma_c * ih2;                 // dG4_c(k)/dc(k +- e_L)
    const double cT = 0.5 * P.K * d * P.eps0 * P.eps0 + P.gamma_c * d * ih2;   // diag extra of dG_c/dc
    // a in {0, +-e_J}
    for (int ia = 0; ia < 2 * d + 1; ++ia) {
      int a[3] = {0, 0, 0};
      double wa;
      if (ia == 0) {
        double s = 0.0;
        for (int J = 0; J < d; ++J) {
          int e1[3] = {0, 0, 0};
          e1[J] = 1;
          const double cp = Xa[gid(e1[0], e1[1], e1[2])], cm = Xa[gid(-e1[0], -e1[1], -e1[2])];
          s += (mi + cp * (1.0 - cp)) + (mi + cm * (1.0 - cm));
        }
        wa = 0.5 * P.kappa * s * ih2;           // -W_ii
      } else {
        const int J = (ia - 1) / 2, sg = ((ia - 1) % 2 == 0) ? 1 : -1;
        a[J] = sg;
        const double cn = Xa[gid(a[0], a[1], a[2])];
        wa = -0.5 * P.kappa * (mi + cn * (1.0 - cn)) * ih2;   // -W_{i,i+a}
      }
      const int b[3] = {o[0] - a[0], o[1] - a[1], o[2] - a[2]};
      const int bl1 = abs(b[0]) + abs(b[1]) + abs(b[2]);
      if (bl1 > 1) continue;
      const long long k = gid(a[0], a[1], a[2]);
      if (bl1 == 0) {
        blk[0 * nf + 0] += wa * (jac4[k] + cT);
        blk[0 * nf + 1] += wa * jac4[N + k];
      } else {
        int L = b[0] != 0 ? 0 : (b[1] != 0 ? 1 : 2);
        const int s = b[L];
        blk[0 * nf + 0] += wa * beta_nb;
        blk[0 * nf + 2 + L] += wa * (-P.eps0 * P.K * s * 0.25 / P.h);
      }
    }
    if (l1 == 0) blk[0] += P.inv_dt;
  }
  // ---- eta row
  {
    const long long i = gid(0, 0, 0);
    if (l1 == 0) {
      blk[1 * nf + 0] = jac4[2 * N + i];
      blk[1 * nf + 1] = P.inv_dt + jac4[3 * N + i] + 3.0 * P.gamma_eta * d * ih2;
    } else if (l1 == 1) {
      blk[1 * nf + 1] = -1.5 * P.gamma_eta * ih2;
    }
  }
  // ---- u rows
  const double e4 = P.Ls * P.inv_4h2;
  for (int I = 0; I < d; ++I) {
    double* row = blk + (2 + I) * nf;
    if (l1 == 0) {
      row[2 + I] = e4 * (-2.0 * P.C11 - 2.0 * P.C44 * (d - 1));
    } else if (l1 == 2) {
      // +-2 e_J ?
      int nz = 0, J = -1;
      for (int k = 0; k < 3; ++k)
        if (o[k] != 0) { ++nz; J = k; }
      if (nz == 1) {
        row[2 + I] = e4 * (J == I ? P.C11 : P.C44);
      } else {
        // o = s e_I + t e_M (M != I)
        if (o[I] != 0) {
          for (int M = 0; M < d; ++M)
            if (M != I && o[M] != 0) row[2 + M] = e4 * (P.C12 + P.C44) * o[I] * o[M];
        }
      }
    } else if (l1 == 1) {
      if (o[I] != 0) row[0] = -P.K * P.eps0 * o[I] * P.inv_2h;
    }
  }
}

__global__ void k_assemble(DevParams P, SlotTables T, const double* __restrict__ Xa, const double* __restrict__ jac4,
                           const int* __restrict__ gidx, const int* __restrict__ nbr, long long Ptot,
                           long long ld, double* __restrict__ fac) {
  const int nf = T.nf;
  const long long total = Ptot * T.nslots;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long pos = t % Ptot;
    const int s = (int)(t / Ptot);
    double blk[kMaxNf * kMaxNf];
    if (nbr[(long long)s * Ptot + pos] < 0) {
      for (int k = 0; k < nf * nf; ++k) blk[k] = 0.0;
    } else {
      int gi = gidx[pos];
      if (gi < 0) gi = ~gi;
      const int x = gi % P.nx, y = (gi / P.nx) % P.ny, z = gi / (P.nx * P.ny);
      jac_block(P, Xa, jac4, x, y, z, T.off[s], blk, nf);
    }
    for (int k = 0; k < nf * nf; ++k) fac[((long long)s * nf * nf + k) * ld + pos] = blk[k];
  }
}

// ------------------------------------------------------------------------------------------ K4 by probing
// Assembly of the box blocks from J.v products (Neumann states, reading R38, whose boundary closures the
// analytic jac_block does not know): with v = e_f on the points whose coordinates are congruent to the colour
// q modulo 5, (J v)(g) = J(g, g') e_f for the ONE point g' of that colour within the |o|_inf <= 2 footprint of
// g (J couples only points of the footprint, mirror ghosts included), so 5^d colours x nf fields of J.v give
// every block column exactly.  No wrap: colours repeat across a periodic seam, so periodic states keep the
// analytic assembly.
__global__ void k_probe_vector(DevParams P, int nf, int q0, int q1, int q2, int f, double* __restrict__ v) {
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nf * N; i += (long long)gridDim.x * blockDim.x) {
    const int field = (int)(i / N);
    const long long p = i - field * N;
    const int x = (int)(p % P.nx), y = (int)((p / P.nx) % P.ny), z = (int)(p / ((long long)P.nx * P.ny));
    const bool on = field == f && x % 5 == q0 && y % 5 == q1 && (P.dim < 3 || z % 5 == q2);
    v[i] = on ? 1.0 : 0.0;
  }
}

__global__ void k_probe_scatter(DevParams P, int nslots, int nf, int q0, int q1, int q2, int f, int first,
                                const int* __restrict__ gidx, const int* __restrict__ nbr, long long Ptot, long long ld,
                                const double* __restrict__ Jv, double* __restrict__ fac) {
  const long long total = Ptot * nslots;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total; t += (long long)gridDim.x * blockDim.x) {
    const long long pos = t % Ptot;
    const int s = (int)(t / Ptot);
    const int qp = nbr[(long long)s * Ptot + pos];
    if (qp < 0) {                                    // outside the box: a zero block, written once
      if (first)
        for (int r = 0; r < nf; ++r)
          for (int c = 0; c < nf; ++c) fac[((long long)(s * nf + r) * nf + c) * ld + pos] = 0.0;
      continue;
    }
    int g = gidx[pos], gq = gidx[qp];
    if (g < 0) g = ~g;
    if (gq < 0) gq = ~gq;
    const int xq = gq % P.nx, yq = (gq / P.nx) % P.ny, zq = gq / (P.nx * P.ny);
    if (xq % 5 != q0 || yq % 5 != q1 || (P.dim == 3 && zq % 5 != q2)) continue;
    for (int r = 0; r < nf; ++r) fac[((long long)(s * nf + r) * nf + f) * ld + pos] = Jv[(long long)r * P.N + g];
  }
}

void launch_probe_vector(const DevParams& P, int nf, int q0, int q1, int q2, int f, double* v, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((nf * P.N + 255) / 256, 148 * 16);
  k_probe_vector<<<blocks, 256, 0, s>>>(P, nf, q0, q1, q2, f, v);
}

void launch_probe_scatter(const DevParams& P, const BoxSet& B, int nf, int q0, int q1, int q2, int f, int first,
                          const double* Jv, double* fac, cudaStream_t s) {
  const long long total = B.P * B.nslots;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  k_probe_scatter<<<blocks, 256, 0, s>>>(P, B.nslots, nf, q0, q1, q2, f, first, B.gidx, B.nbr, B.P, B.ld, Jv, fac);
}

// ------------------------------------------------------------------------------------------ K5 factorisation
template <int NF>
__device__ __forceinline__ void load_blk(const double* fac, int s, long long pos, long long ld, double (&b)[NF][NF]) {
#pragma unroll
  for (int r = 0; r < NF; ++r)
#pragma unroll
    for (int c = 0; c < NF; ++c) b[r][c] = fac[((long long)(s * NF + r) * NF + c) * ld + pos];
}
template <int NF>
__device__ __forceinline__ void store_blk(double* fac, int s, long long pos, long long ld, const double (&b)[NF][NF]) {
#pragma unroll
  for (int r = 0; r < NF; ++r)
#pragma unroll
    for (int c = 0; c < NF; ++c) fac[((long long)(s * NF + r) * NF + c) * ld + pos] = b[r][c];
}

// In-register Gauss-Jordan inverse with partial pivoting.
template <int NF>
__device__ __forceinline__ void invert(double (&a)[NF][NF]) {
  double inv[NF][NF];
#pragma unroll
  for (int r = 0; r < NF; ++r)
#pragma unroll
    for (int c = 0; c < NF; ++c) inv[r][c] = r == c ? 1.0 : 0.0;
#pragma unroll
  for (int k = 0; k < NF; ++k) {
    int piv = k;
    double best = fabs(a[k][k]);
#pragma unroll
    for (int r = k + 1; r < NF; ++r)
      if (fabs(a[r][k]) > best) { best = fabs(a[r][k]); piv = r; }
    if (piv != k) {
#pragma unroll
      for (int r = k + 1; r < NF; ++r)
        if (r == piv) {
#pragma unroll
          for (int c = 0; c < NF; ++c) {
            double t = a[k][c]; a[k][c] = a[r][c]; a[r][c] = t;
            t = inv[k][c]; inv[k][c] = inv[r][c]; inv[r][c] = t;
          }
        }
    }
    const double ip = 1.0 / a[k][k];
#pragma unroll
    for (int c = 0; c < NF; ++c) { a[k][c] *= ip; inv[k][c] *= ip; }
#pragma unroll
    for (int r = 0; r < NF; ++r) {
      if (r == k) continue;
      const double f = a[r][k];
#pragma unroll
      for (int c = 0; c < NF; ++c) { a[r][c] -= f * a[k][c]; inv[r][c] -= f * inv[k][c]; }
    }
  }
#pragma unroll
  for (int r = 0; r < NF; ++r)
#pragma unroll
    for (int c = 0; c < NF; ++c) a[r][c] = inv[r][c];
}

template <int NF>
__global__ void k_bilu0(SlotTables T, const int* __restrict__ nbr, const int* __restrict__ box_lev_off,
                        const int* __restrict__ lev_ptr, long long Ptot, long long ld, double* fac) {
  const int b = blockIdx.x;
  const int l0 = box_lev_off[b], l1 = box_lev_off[b + 1] - 1;     // levels l0 .. l1-1
  for (int l = l0; l < l1; ++l) {
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + threadIdx.x; pos < p1; pos += blockDim.x) {
      for (int ia = 0; ia < T.nlower; ++ia) {
        const int sa = T.lower[ia];
        const int k = nbr[(long long)sa * Ptot + pos];
        if (k < 0) continue;
        double A[NF][NF], D[NF][NF], Lk[NF][NF];
        load_blk<NF>(fac, sa, pos, ld, A);
        load_blk<NF>(fac, T.diag, k, ld, D);       // U_kk^{-1}
#pragma unroll
        for (int r = 0; r < NF; ++r)
#pragma unroll
          for (int c = 0; c < NF; ++c) {
            double s = 0.0;
#pragma unroll
            for (int m = 0; m < NF; ++m) s = fma(A[r][m], D[m][c], s);
            Lk[r][c] = s;
          }
        store_blk<NF>(fac, sa, pos, ld, Lk);
        for (int ip = 0; ip < T.npairs[ia]; ++ip) {
          const int sb = T.pair_b[ia][ip], st = T.pair_t[ia][ip];
          if (nbr[(long long)st * Ptot + pos] < 0) continue;
          double U[NF][NF], Tt[NF][NF];
          load_blk<NF>(fac, sb, k, ld, U);
          load_blk<NF>(fac, st, pos, ld, Tt);
#pragma unroll
          for (int r = 0; r < NF; ++r)
#pragma unroll
            for (int c = 0; c < NF; ++c) {
              double s = Tt[r][c];
#pragma unroll
              for (int m = 0; m < NF; ++m) s = fma(-Lk[r][m], U[m][c], s);
              Tt[r][c] = s;
            }
          store_blk<NF>(fac, st, pos, ld, Tt);
        }
      }
      double Dg[NF][NF];
      load_blk<NF>(fac, T.diag, pos, ld, Dg);
      invert<NF>(Dg);
      store_blk<NF>(fac, T.diag, pos, ld, Dg);
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------------------------------------ K6 RAS apply
// Level-synchronous sweeps (one CTA per box; 3D, and 2D cases the pipelined k_ras2d does not cover).
// NL = number of lower (= upper) slots: 6 in 2D, 12 in 3D; the slot loops are unrolled so that every
// neighbour index and neighbour vector of a point is requested before the first one is used (two
// dependent memory latencies per wavefront level instead of 2*NL).
// NKS_RAS3D_SPLIT: the NL neighbour blocks of a point are taken in chunks of NL / SPLIT (fewer live
// registers: 3D with one chunk holds 12 x 5 neighbour values and needs 168 registers, so only 3 CTAs of
// 128 threads fit an SM and config 3's 512 boxes run in two rounds)
#ifndef NKS_RAS3D_SPLIT
#define NKS_RAS3D_SPLIT 1
#endif
#ifndef NKS_RAS3D_LB
#define NKS_RAS3D_LB 0       // > 0: __launch_bounds__(256, LB) (2 caps the registers at 128)
#endif
#if NKS_RAS3D_LB > 0
#define NKS_RAS3D_BOUNDS __launch_bounds__(256, NKS_RAS3D_LB)
#else
#define NKS_RAS3D_BOUNDS
#endif
template <int NF, int NL, typename FT>
__global__ void NKS_RAS3D_BOUNDS k_ras_apply(SlotTables T, const int* __restrict__ gidx, const int* __restrict__ nbr,
                            const int* __restrict__ box_lev_off, const int* __restrict__ lev_ptr,
                            const int* __restrict__ box_pos_off, long long Ptot, long long ld, long long N,
                            const FT* __restrict__ fac, const double* __restrict__ r, double* y,
                            double* __restrict__ z, int variant) {
  const int b = blockIdx.x;
  const int q0 = box_pos_off[b], q1 = box_pos_off[b + 1];
  // R_i^delta r (RAS, AS) or R_i^0 r (RRAS: the overlap points read zero)
  for (int pos = q0 + threadIdx.x; pos < q1; pos += blockDim.x) {
    int gi = gidx[pos];
    const bool owned = gi >= 0;
    if (gi < 0) gi = ~gi;
#pragma unroll
    for (int f = 0; f < NF; ++f) y[f * Ptot + pos] = (variant == 2 && !owned) ? 0.0 : r[f * N + gi];
  }
  __syncthreads();
  const int l0 = box_lev_off[b], l1 = box_lev_off[b + 1] - 1;
  // forward: y_i -= sum_{k<i} L_ik y_k
  for (int l = l0; l < l1; ++l) {
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + threadIdx.x; pos < p1; pos += blockDim.x) {
      constexpr int CH = NL / NKS_RAS3D_SPLIT;
      double acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f] = y[f * Ptot + pos];
#pragma unroll
      for (int h = 0; h < NKS_RAS3D_SPLIT; ++h) {
        int kk[CH];
#pragma unroll
        for (int a = 0; a < CH; ++a) kk[a] = __ldg(nbr + (long long)T.lower[h * CH + a] * Ptot + pos);
        double yk[CH][NF];
#pragma unroll
        for (int a = 0; a < CH; ++a)
#pragma unroll
          for (int f = 0; f < NF; ++f) yk[a][f] = kk[a] >= 0 ? y[f * Ptot + kk[a]] : 0.0;
#pragma unroll
        for (int a = 0; a < CH; ++a) {
          const FT* L = fac + (long long)(T.lower[h * CH + a] * NF * NF) * ld + pos;
#pragma unroll
          for (int rr = 0; rr < NF; ++rr)
#pragma unroll
            for (int c = 0; c < NF; ++c)
              acc[rr] = fma(-(double)__ldg(L + (long long)(rr * NF + c) * ld), yk[a][c], acc[rr]);
        }
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) y[f * Ptot + pos] = acc[f];
    }
    __syncthreads();
  }
  // backward: x_i = U_ii^{-1} (y_i - sum_{j>i} U_ij x_j)
  for (int l = l1 - 1; l >= l0; --l) {
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + threadIdx.x; pos < p1; pos += blockDim.x) {
      constexpr int CH = NL / NKS_RAS3D_SPLIT;
      double acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f] = y[f * Ptot + pos];
#pragma unroll
      for (int h = 0; h < NKS_RAS3D_SPLIT; ++h) {
        int kk[CH];
#pragma unroll
        for (int a = 0; a < CH; ++a) kk[a] = __ldg(nbr + (long long)T.upper[h * CH + a] * Ptot + pos);
        double xk[CH][NF];
#pragma unroll
        for (int a = 0; a < CH; ++a)
#pragma unroll
          for (int f = 0; f < NF; ++f) xk[a][f] = kk[a] >= 0 ? y[f * Ptot + kk[a]] : 0.0;
#pragma unroll
        for (int a = 0; a < CH; ++a) {
          const FT* U = fac + (long long)(T.upper[h * CH + a] * NF * NF) * ld + pos;
#pragma unroll
          for (int rr = 0; rr < NF; ++rr)
#pragma unroll
            for (int c = 0; c < NF; ++c)
              acc[rr] = fma(-(double)__ldg(U + (long long)(rr * NF + c) * ld), xk[a][c], acc[rr]);
        }
      }
      const FT* D = fac + (long long)(T.diag * NF * NF) * ld + pos;
      double xo[NF];
#pragma unroll
      for (int rr = 0; rr < NF; ++rr) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NF; ++c) s = fma((double)__ldg(D + (long long)(rr * NF + c) * ld), acc[c], s);
        xo[rr] = s;
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) y[f * Ptot + pos] = xo[f];
    }
    __syncthreads();
  }
  // R_i^{0T}: owned points only (RAS); AS / RRAS keep the box solutions in y for k_schwarz_gather
  if (variant != 0) return;
  for (int pos = q0 + threadIdx.x; pos < q1; pos += blockDim.x) {
    const int gi = gidx[pos];
    if (gi < 0) continue;
#pragma unroll
    for (int f = 0; f < NF; ++f) z[f * N + gi] = y[f * Ptot + pos];
  }
}

// The same sweeps with a thread-block cluster of CS CTAs per box (cluster rank r takes positions
// p0 + r*blockDim + tid, stride CS*blockDim, of every level; the level barrier is the cluster barrier,
// release/acquire at cluster scope).  Used when the boxes alone would leave SMs idle -- a rank's share of
// a strong-scaled grid (config 4 on 8 GPUs: 64 boxes of 36^3 per GPU on 148 SMs).  The box vector y
// lives in global memory and is written by the other CTAs of the cluster, so its loads bypass L1 (ld.cg).
template <int NF, int NL, typename FT>
__global__ void k_ras_apply_cl(SlotTables T, const int* __restrict__ gidx, const int* __restrict__ nbr,
                               const int* __restrict__ box_lev_off, const int* __restrict__ lev_ptr,
                               const int* __restrict__ box_pos_off, long long Ptot, long long ld, long long N,
                               const FT* __restrict__ fac, const double* __restrict__ r, double* y,
                               double* __restrict__ z, int variant) {
  namespace cg = cooperative_groups;
  cg::cluster_group cl = cg::this_cluster();
  const int CS = (int)cl.num_blocks();
  const int b = blockIdx.x / CS;
  const int t0 = (int)cl.block_rank() * blockDim.x + threadIdx.x, ts = CS * blockDim.x;
  const int q0 = box_pos_off[b], q1 = box_pos_off[b + 1];
  for (int pos = q0 + t0; pos < q1; pos += ts) {
    int gi = gidx[pos];
    const bool owned = gi >= 0;
    if (gi < 0) gi = ~gi;
#pragma unroll
    for (int f = 0; f < NF; ++f) __stcg(y + f * Ptot + pos, (variant == 2 && !owned) ? 0.0 : r[f * N + gi]);
  }
  cl.sync();
  const int l0 = box_lev_off[b], l1 = box_lev_off[b + 1] - 1;
  for (int l = l0; l < l1; ++l) {
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + t0; pos < p1; pos += ts) {
      int kk[NL];
#pragma unroll
      for (int a = 0; a < NL; ++a) kk[a] = __ldg(nbr + (long long)T.lower[a] * Ptot + pos);
      double yk[NL][NF];
#pragma unroll
      for (int a = 0; a < NL; ++a)
#pragma unroll
        for (int f = 0; f < NF; ++f) yk[a][f] = kk[a] >= 0 ? __ldcg(y + f * Ptot + kk[a]) : 0.0;
      double acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f] = __ldcg(y + f * Ptot + pos);
#pragma unroll
      for (int a = 0; a < NL; ++a) {
        const FT* L = fac + (long long)(T.lower[a] * NF * NF) * ld + pos;
#pragma unroll
        for (int rr = 0; rr < NF; ++rr)
#pragma unroll
          for (int c = 0; c < NF; ++c)
            acc[rr] = fma(-(double)__ldg(L + (long long)(rr * NF + c) * ld), yk[a][c], acc[rr]);
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) __stcg(y + f * Ptot + pos, acc[f]);
    }
    cl.sync();
  }
  for (int l = l1 - 1; l >= l0; --l) {
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + t0; pos < p1; pos += ts) {
      int kk[NL];
#pragma unroll
      for (int a = 0; a < NL; ++a) kk[a] = __ldg(nbr + (long long)T.upper[a] * Ptot + pos);
      double xk[NL][NF];
#pragma unroll
      for (int a = 0; a < NL; ++a)
#pragma unroll
        for (int f = 0; f < NF; ++f) xk[a][f] = kk[a] >= 0 ? __ldcg(y + f * Ptot + kk[a]) : 0.0;
      double acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f] = __ldcg(y + f * Ptot + pos);
#pragma unroll
      for (int a = 0; a < NL; ++a) {
        const FT* U = fac + (long long)(T.upper[a] * NF * NF) * ld + pos;
#pragma unroll
        for (int rr = 0; rr < NF; ++rr)
#pragma unroll
          for (int c = 0; c < NF; ++c)
            acc[rr] = fma(-(double)__ldg(U + (long long)(rr * NF + c) * ld), xk[a][c], acc[rr]);
      }
      const FT* D = fac + (long long)(T.diag * NF * NF) * ld + pos;
      double xo[NF];
#pragma unroll
      for (int rr = 0; rr < NF; ++rr) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NF; ++c) s = fma((double)__ldg(D + (long long)(rr * NF + c) * ld), acc[c], s);
        xo[rr] = s;
      }
#pragma unroll
      for (int f = 0; f < NF; ++f) __stcg(y + f * Ptot + pos, xo[f]);
    }
    cl.sync();
  }
  if (variant != 0) return;
  for (int pos = q0 + t0; pos < q1; pos += ts) {
    const int gi = gidx[pos];
    if (gi < 0) continue;
#pragma unroll
    for (int f = 0; f < NF; ++f) z[f * N + gi] = __ldcg(y + f * Ptot + pos);
  }
}

// sum_i R_i^{deltaT} x_i: every grid point adds the solutions of the box positions covering it, in
// increasing position order (deterministic; a periodic self-overlapping box covers a point twice)
__global__ void k_schwarz_gather(long long N, int nf, long long Ptot, const int* __restrict__ cover_off,
                                 const int* __restrict__ cover_pos, const double* __restrict__ y, double* __restrict__ z) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int e0 = cover_off[i], e1 = cover_off[i + 1];
    for (int f = 0; f < nf; ++f) {
      double acc = 0.0;
      for (int e = e0; e < e1; ++e) acc += y[f * Ptot + cover_pos[e]];
      z[f * N + i] = acc;
    }
  }
}

// ------------------------------------------------------------------------------------------ host launchers
SlotTables make_tables(const BoxSet& B, int nf) {
  SlotTables T;
  T.nslots = B.nslots; T.nf = nf; T.diag = B.diag; T.nlower = B.nlower; T.nupper = B.nupper;
  for (int s = 0; s < kMaxSlots; ++s) {
    for (int k = 0; k < 3; ++k) T.off[s][k] = B.off[s][k];
    T.lower[s] = B.lower[s]; T.upper[s] = B.upper[s]; T.npairs[s] = B.npairs[s];
    for (int p = 0; p < kMaxSlots; ++p) { T.pair_b[s][p] = B.pair_b[s][p]; T.pair_t[s][p] = B.pair_t[s][p]; }
  }
  return T;
}

void launch_assemble(const DevParams& P, const BoxSet& B, int nf, const double* Xa, const double* jac4, double* fac,
                     cudaStream_t s) {
  const SlotTables T = make_tables(B, nf);
  const long long total = B.P * B.nslots;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  k_assemble<<<blocks, 256, 0, s>>>(P, T, Xa, jac4, B.gidx, B.nbr, B.P, B.ld, fac);
}

void launch_factor(const BoxSet& B, int nf, double* fac, cudaStream_t s) {
  const SlotTables T = make_tables(B, nf);
  const int threads = std::min(256, std::max(32, ((B.max_level_width + 31) / 32) * 32));
  if (nf == 4) k_bilu0<4><<<B.nbox, threads, 0, s>>>(T, B.nbr, B.box_lev_off, B.lev_ptr, B.P, B.ld, fac);
  else k_bilu0<5><<<B.nbox, threads, 0, s>>>(T, B.nbr, B.box_lev_off, B.lev_ptr, B.P, B.ld, fac);
}

__global__ void k_to_fp32(long long n, const double* __restrict__ a, float* __restrict__ b) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    b[i] = (float)a[i];
}

void launch_fac_to_fp32(const BoxSet& B, int nf, const double* fac, float* fac32, cudaStream_t s) {
  const long long n = (long long)B.nslots * nf * nf * B.ld;
  k_to_fp32<<<148 * 8, 256, 0, s>>>(n, fac, fac32);
}

// CTAs per box of the clustered apply: doubled while the boxes would fill at most half of the SMs, at
// most 4 and never more than the widest level needs (NKS_RAS3D_CSMAX / NKS_RAS3D_WIDTH: build-time
// switches for experiments).  Measured at config 4's per-GPU share (profiles/r02_ras3d_cluster.log):
// 64 boxes of 36^3 (8 GPUs) 5.71 -> 4.54 ms with 2 CTAs per box (4: 7.67 ms); 128 boxes (4 GPUs) are
// slower clustered (7.20 -> 9.11 ms: the cluster barrier per level costs more than the extra SMs give),
// so they keep one CTA per box.
#ifndef NKS_RAS3D_CSMAX
#define NKS_RAS3D_CSMAX 4
#endif
static int ras_cluster_of(const BoxSet& B, int threads) {
  if (B.cta_per_box > 0) return B.cta_per_box;      // nks_params.ras_cta_per_box (forced)
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  int cs = 1;
#ifndef NKS_RAS3D_WIDTH
#define NKS_RAS3D_WIDTH 1
#endif
  while (cs < NKS_RAS3D_CSMAX && 2LL * B.nbox * cs <= sms && (!NKS_RAS3D_WIDTH || cs * threads < B.max_level_width))
    cs *= 2;
  return cs;
}

template <int NF, int NL, typename FT>
static cudaError_t launch_cl(int cs, int threads, const SlotTables& T, const BoxSet& B, long long N, const FT* fac,
                             const double* r, double* y, double* z, cudaStream_t s) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(B.nbox * cs, 1, 1);
  cfg.blockDim = dim3(threads, 1, 1);
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  return cudaLaunchKernelEx(&cfg, k_ras_apply_cl<NF, NL, FT>, T, (const int*)B.gidx, (const int*)B.nbr,
                            (const int*)B.box_lev_off, (const int*)B.lev_ptr, (const int*)B.box_pos_off, B.P, B.ld, N,
                            fac, r, y, z, B.variant);
}

void launch_ras_apply(const BoxSet& B, int nf, long long N, const double* fac, const float* fac32, const double* r,
                      double* y, double* z, cudaStream_t s) {
  const SlotTables T = make_tables(B, nf);
  const int threads = std::min(256, std::max(32, ((B.max_level_width + 31) / 32) * 32));
  const int cs = ras_cluster_of(B, threads);
  if (cs > 1) {
    if (nf == 4) {
      if (fac32) launch_cl<4, 6, float>(cs, threads, T, B, N, fac32, r, y, z, s);
      else launch_cl<4, 6, double>(cs, threads, T, B, N, fac, r, y, z, s);
    } else {
      if (fac32) launch_cl<5, 12, float>(cs, threads, T, B, N, fac32, r, y, z, s);
      else launch_cl<5, 12, double>(cs, threads, T, B, N, fac, r, y, z, s);
    }
    if (B.variant != 0) {
      const int blocks = (int)std::min<long long>((N + 255) / 256, 148 * 8);
      k_schwarz_gather<<<blocks, 256, 0, s>>>(N, nf, B.P, B.cover_off, B.cover_pos, y, z);
    }
    return;
  }
  if (nf == 4) {
    if (fac32)
      k_ras_apply<4, 6, float><<<B.nbox, threads, 0, s>>>(T, B.gidx, B.nbr, B.box_lev_off, B.lev_ptr, B.box_pos_off,
                                                          B.P, B.ld, N, fac32, r, y, z, B.variant);
    else
      k_ras_apply<4, 6, double><<<B.nbox, threads, 0, s>>>(T, B.gidx, B.nbr, B.box_lev_off, B.lev_ptr, B.box_pos_off,
                                                           B.P, B.ld, N, fac, r, y, z, B.variant);
  } else {
    if (fac32)
      k_ras_apply<5, 12, float><<<B.nbox, threads, 0, s>>>(T, B.gidx, B.nbr, B.box_lev_off, B.lev_ptr, B.box_pos_off,
                                                           B.P, B.ld, N, fac32, r, y, z, B.variant);
    else
      k_ras_apply<5, 12, double><<<B.nbox, threads, 0, s>>>(T, B.gidx, B.nbr, B.box_lev_off, B.lev_ptr,
                                                            B.box_pos_off, B.P, B.ld, N, fac, r, y, z, B.variant);
  }
  if (B.variant != 0) {
    const int blocks = (int)std::min<long long>((N + 255) / 256, 148 * 8);
    k_schwarz_gather<<<blocks, 256, 0, s>>>(N, nf, B.P, B.cover_off, B.cover_pos, y, z);
  }
}

}  // namespace nks

#include "precond_iluk.cuh"
