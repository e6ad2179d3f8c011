// (Included at the end of precond.cu: it shares jac_block and k_schwarz_gather.)
// Level-k point-block ILU subdomain solvers of the Schwarz preconditioner: ILU(1), ILU(2), ... and the
// exact block LU (no level limit) -- SURVEY 8(f)-1, the fill levels of Table 1 ("ILU(0),
// ILU(1), ILU(2), LU").  The default BILU(0) keeps its specialised kernels (precond.cu, ras2d_rows.cu).
//
// Symbolic phase (host, once per distinct box extent): Saad's ILU(p) level of fill (Iterative Methods,
// Sec. 10.3.3) on the natural-order block graph of the box matrix A_i: lev = 0 on the 13/25-point
// pattern of J, lev(i,j) = min_k lev(i,k) + lev(k,j) + 1 over eliminated k, entries with lev <= k kept
// (reading R21's natural order, no pivoting).  Every kept entry is an offset (dx,dy,dz) between two box
// points; the union of those offsets over all rows is the slot set, and a row simply has no entry in
// the slots its level-k pattern lacks (nbr = -1) -- so the same slot-indexed factor layout, assembly and
// wavefront machinery as BILU(0) carry any fill level.  The wavefront level of a point is
// lx + a ly + b lz with the smallest a, b that put every lower slot on an earlier level (a = 2, b = 3 for
// the ILU(0) pattern, reading R21; a = ex for the exact LU in 2D, i.e. the natural order itself).
//
// Numeric phase (device): one CTA per box, one WARP per row of a wavefront level: IKJ elimination, the
// lower entries of the row in ascending order; for each, lane-parallel L_ik = A_ik U_kk^-1 and then the
// pair updates A_ij -= L_ik U_kj spread over the lanes (distinct j per pair).  Triangular solves: one warp
// per row, the lanes splitting the row's slots, warp-shuffle reduction.
#include <algorithm>
#include <array>
#include <cstdio>
#include <map>
#include <stdexcept>


namespace nks {

// ------------------------------------------------------------------------------------------ host symbolic
namespace {

long long nat_key3(const std::array<int, 3>& o) { return ((long long)o[2] * 4096 + o[1]) * 4096 + o[0]; }

struct ExtentPattern {
  std::array<int, 3> e;
  std::vector<std::vector<int>> cols;    // per local natural index: kept columns (natural index)
};

// Level-of-fill of one box extent.  level < 0: no limit (exact LU).
ExtentPattern symbolic(const std::array<int, 3>& e, int dim, int level) {
  const int ex = e[0], ey = e[1], ez = e[2];
  const int n = ex * ey * ez;
  const int B = dim == 3 ? 2 * ex * ey : 2 * ex;            // band half-width of the footprint
  ExtentPattern P;
  P.e = e;
  P.cols.resize(n);
  std::vector<std::vector<std::pair<int, int>>> upper(n);   // (col, level) with col > row
  std::vector<int> lev(2 * B + 1);
  const int INF = 1 << 29;
  for (int i = 0; i < n; ++i) {
    std::fill(lev.begin(), lev.end(), INF);
    const int x = i % ex, y = (i / ex) % ey, z = i / (ex * ey);
    for (int oz = (dim == 3 ? -2 : 0); oz <= (dim == 3 ? 2 : 0); ++oz)
      for (int oy = -2; oy <= 2; ++oy)
        for (int ox = -2; ox <= 2; ++ox) {
          if (std::abs(ox) + std::abs(oy) + std::abs(oz) > 2) continue;
          const int qx = x + ox, qy = y + oy, qz = z + oz;
          if (qx < 0 || qx >= ex || qy < 0 || qy >= ey || qz < 0 || qz >= ez) continue;
          const int j = (qz * ey + qy) * ex + qx;
          lev[j - i + B] = 0;
        }
    // IKJ symbolic: scan the lower band left to right; fill lands right of the eliminated column only
    for (int t = 0; t < B; ++t) {
      if (lev[t] >= INF) continue;
      const int k = i - B + t;
      const int lik = lev[t];
      for (const auto& ent : upper[k]) {
        const int nl = lik + ent.second + 1;
        if (level >= 0 && nl > level) continue;
        const int idx = ent.first - i + B;
        if (idx < 0 || idx > 2 * B) continue;                // cannot happen within the band
        if (nl < lev[idx]) lev[idx] = nl;
      }
    }
    for (int t = 0; t <= 2 * B; ++t) {
      if (lev[t] >= INF) continue;
      const int j = i - B + t;
      if (j < 0 || j >= n) continue;
      P.cols[i].push_back(j);
      if (j > i) upper[i].push_back({j, lev[t]});
    }
  }
  return P;
}

void split_axis_k(int n, int nsub, std::vector<int>& start, std::vector<int>& len) {
  const int base = n / nsub, rem = n % nsub;
  int s = 0;
  for (int b = 0; b < nsub; ++b) {
    const int l = base + (b < rem ? 1 : 0);
    start.push_back(s);
    len.push_back(l);
    s += l;
  }
}

}  // namespace

// Slot set, pairs and level function of the level-k pattern over every box extent of the grid.
IlukPattern build_iluk_pattern(const nks_grid& g, int level) {
  IlukPattern T;
  const int dim = g.dim;
  std::vector<int> st[3], ln[3];
  for (int j = 0; j < 2; ++j) split_axis_k(g.n[j], g.nsub[j], st[j], ln[j]);
  split_axis_k(g.zghost > 0 ? g.n[2] - 2 * g.zghost : g.n[2], g.nsub[2], st[2], ln[2]);
  const int dz = dim == 3 ? g.overlap : 0;
  std::map<std::array<int, 3>, int> ext_id;
  for (int bz = 0; bz < g.nsub[2]; ++bz)
    for (int by = 0; by < g.nsub[1]; ++by)
      for (int bx = 0; bx < g.nsub[0]; ++bx) {
        const std::array<int, 3> e = {ln[0][bx] + 2 * g.overlap, ln[1][by] + 2 * g.overlap, ln[2][bz] + 2 * dz};
        if (!ext_id.count(e)) {
          ext_id[e] = (int)T.ext.size();
          T.ext.push_back(e);
        }
      }
  std::vector<ExtentPattern> pats;
  std::map<std::array<int, 3>, int> slot_of;
  for (const auto& e : T.ext) {
    pats.push_back(symbolic(e, dim, level));
    const ExtentPattern& P = pats.back();
    const int ex = e[0], ey = e[1];
    for (size_t i = 0; i < P.cols.size(); ++i) {
      const int x = (int)i % ex, y = ((int)i / ex) % ey, z = (int)i / (ex * ey);
      for (int j : P.cols[i]) {
        const std::array<int, 3> o = {j % ex - x, (j / ex) % ey - y, j / (ex * ey) - z};
        slot_of.emplace(o, 0);
      }
    }
  }
  // slots in ascending natural order of the offset
  std::vector<std::array<int, 3>> offs;
  for (auto& kv : slot_of) offs.push_back(kv.first);
  std::sort(offs.begin(), offs.end(), [](const std::array<int, 3>& a, const std::array<int, 3>& b) {
    return nat_key3(a) < nat_key3(b);
  });
  for (size_t s = 0; s < offs.size(); ++s) slot_of[offs[s]] = (int)s;
  T.nslots = (int)offs.size();
  T.off = offs;
  for (int s = 0; s < T.nslots; ++s) {
    const long long k = nat_key3(offs[s]);
    if (k < 0) T.lower.push_back(s);
    else if (k > 0) T.upper.push_back(s);
    else T.diag = s;
  }
  T.pair_ptr.push_back(0);
  for (int a : T.lower) {
    for (int b : T.upper) {
      const std::array<int, 3> t = {offs[a][0] + offs[b][0], offs[a][1] + offs[b][1], offs[a][2] + offs[b][2]};
      auto it = slot_of.find(t);
      if (it == slot_of.end()) continue;
      T.pair_b.push_back(b);
      T.pair_t.push_back(it->second);
    }
    T.pair_ptr.push_back((int)T.pair_b.size());
  }
  // level function l = lx + a ly + b lz: every lower slot strictly earlier
  int a = 1;                       // dz = 0, dy < 0: dx + a dy < 0  <=>  a > dx / (-dy)
  for (int s : T.lower)
    if (offs[s][2] == 0 && offs[s][1] < 0 && offs[s][0] >= 0) a = std::max(a, offs[s][0] / (-offs[s][1]) + 1);
  int b = 1;                       // dz < 0: dx + a dy + b dz < 0  <=>  b > (dx + a dy) / (-dz)
  for (int s : T.lower)
    if (offs[s][2] < 0) {
      const int v = offs[s][0] + a * offs[s][1];
      if (v >= 0) b = std::max(b, v / (-offs[s][2]) + 1);
    }
  for (int s : T.lower) {
    const long long l = offs[s][0] + (long long)a * offs[s][1] + (long long)b * offs[s][2];
    if (l >= 0) throw std::runtime_error("ILU(k) level function");
  }
  T.la = a;
  T.lb = dim == 3 ? b : 0;
  // per-extent presence: bit (row, slot)
  T.present.resize(T.ext.size());
  for (size_t q = 0; q < T.ext.size(); ++q) {
    const auto& e = T.ext[q];
    const ExtentPattern& P = pats[q];
    const int ex = e[0], ey = e[1];
    auto& pr = T.present[q];
    pr.assign(P.cols.size() * (size_t)T.nslots, 0);
    for (size_t i = 0; i < P.cols.size(); ++i) {
      const int x = (int)i % ex, y = ((int)i / ex) % ey, z = (int)i / (ex * ey);
      for (int j : P.cols[i]) {
        const std::array<int, 3> o = {j % ex - x, (j / ex) % ey - y, j / (ex * ey) - z};
        pr[i * T.nslots + slot_of[o]] = 1;
      }
    }
  }
  return T;
}

// ------------------------------------------------------------------------------------------ device
struct GenTables {
  int nslots, nlower, nupper, diag;
  const int* off;        // [nslots][3]
  const int* lower;      // [nlower] ascending natural order
  const int* upper;      // [nupper]
  const int* pair_ptr;   // [nlower + 1]
  const int* pair_b;
  const int* pair_t;
};

__device__ __forceinline__ int wrapk(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }

// (jac_block of precond.cu is zero for offsets outside J's footprint, so the fill slots start from zero.)
__global__ void k_assemble_gen(DevParams P, GenTables T, int nf, const double* __restrict__ Xa,
                               const double* __restrict__ jac4, const int* __restrict__ gidx,
                               const int* __restrict__ nbr, long long Ptot, long long ld, double* __restrict__ fac) {
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
      const int o[3] = {T.off[3 * s], T.off[3 * s + 1], T.off[3 * s + 2]};
      jac_block(P, Xa, jac4, x, y, z, o, blk, nf);
    }
    for (int k = 0; k < nf * nf; ++k) fac[((long long)s * nf * nf + k) * ld + pos] = blk[k];
  }
}

template <int NF>
__device__ __forceinline__ double* blkp(double* fac, int s, int rc, long long pos, long long ld) {
  return fac + ((long long)s * NF * NF + rc) * ld + pos;
}

template <int NF>
__device__ void invert_nf(double (&a)[NF][NF]) {
  double inv[NF][NF];
  for (int r = 0; r < NF; ++r)
    for (int c = 0; c < NF; ++c) inv[r][c] = r == c ? 1.0 : 0.0;
  for (int k = 0; k < NF; ++k) {
    int piv = k;
    double best = fabs(a[k][k]);
    for (int r = k + 1; r < NF; ++r)
      if (fabs(a[r][k]) > best) { best = fabs(a[r][k]); piv = r; }
    if (piv != k)
      for (int c = 0; c < NF; ++c) {
        double t = a[k][c]; a[k][c] = a[piv][c]; a[piv][c] = t;
        t = inv[k][c]; inv[k][c] = inv[piv][c]; inv[piv][c] = t;
      }
    const double ip = 1.0 / a[k][k];
    for (int c = 0; c < NF; ++c) { a[k][c] *= ip; inv[k][c] *= ip; }
    for (int r = 0; r < NF; ++r) {
      if (r == k) continue;
      const double f = a[r][k];
      for (int c = 0; c < NF; ++c) { a[r][c] -= f * a[k][c]; inv[r][c] -= f * inv[k][c]; }
    }
  }
  for (int r = 0; r < NF; ++r)
    for (int c = 0; c < NF; ++c) a[r][c] = inv[r][c];
}

// IKJ on the level-k pattern: one warp per row of the current wavefront level.
template <int NF>
__global__ void __launch_bounds__(256) k_biluk(GenTables T, const int* __restrict__ nbr,
                                               const int* __restrict__ box_lev_off, const int* __restrict__ lev_ptr,
                                               long long Ptot, long long ld, double* fac) {
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int l0 = box_lev_off[b], l1 = box_lev_off[b + 1] - 1;
  for (int l = l0; l < l1; ++l) {
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + wid; pos < p1; pos += nw) {
      for (int ia = 0; ia < T.nlower; ++ia) {
        const int sa = T.lower[ia];
        const int k = nbr[(long long)sa * Ptot + pos];
        if (k < 0) continue;
        // L_ik = A_ik D_k^-1 (D_k^-1 stored in the diagonal slot once row k is done): lanes 0..NF*NF-1
        double lrc = 0.0;
        if (lane < NF * NF) {
          const int r = lane / NF, c = lane % NF;
#pragma unroll
          for (int m = 0; m < NF; ++m) lrc = fma(*blkp<NF>(fac, sa, r * NF + m, pos, ld), *blkp<NF>(fac, T.diag, m * NF + c, k, ld), lrc);
        }
        __syncwarp();
        if (lane < NF * NF) *blkp<NF>(fac, sa, lane, pos, ld) = lrc;
        __syncwarp();
        double L[NF][NF];
#pragma unroll
        for (int r = 0; r < NF; ++r)
#pragma unroll
          for (int c = 0; c < NF; ++c) L[r][c] = *blkp<NF>(fac, sa, r * NF + c, pos, ld);
        // pair updates A_ij -= L_ik U_kj, one pair per lane (distinct targets)
        const int q0 = T.pair_ptr[ia], q1 = T.pair_ptr[ia + 1];
        for (int q = q0 + lane; q < q1; q += 32) {
          const int sb = T.pair_b[q], stt = T.pair_t[q];
          if (nbr[(long long)stt * Ptot + pos] < 0) continue;
          if (nbr[(long long)sb * Ptot + k] < 0) continue;
#pragma unroll
          for (int r = 0; r < NF; ++r)
#pragma unroll
            for (int c = 0; c < NF; ++c) {
              double s = *blkp<NF>(fac, stt, r * NF + c, pos, ld);
#pragma unroll
              for (int m = 0; m < NF; ++m) s = fma(-L[r][m], *blkp<NF>(fac, sb, m * NF + c, k, ld), s);
              *blkp<NF>(fac, stt, r * NF + c, pos, ld) = s;
            }
        }
        __syncwarp();
      }
      if (lane == 0) {
        double Dg[NF][NF];
        for (int r = 0; r < NF; ++r)
          for (int c = 0; c < NF; ++c) Dg[r][c] = *blkp<NF>(fac, T.diag, r * NF + c, pos, ld);
        invert_nf<NF>(Dg);
        for (int r = 0; r < NF; ++r)
          for (int c = 0; c < NF; ++c) *blkp<NF>(fac, T.diag, r * NF + c, pos, ld) = Dg[r][c];
      }
      __syncwarp();
    }
    __syncthreads();
  }
}

// Level-synchronous Schwarz apply with ILU(k) box solves: one warp per row, lanes over the row's slots.
template <int NF>
__global__ void __launch_bounds__(1024) k_ras_apply_gen(GenTables T, const int* __restrict__ gidx,
                                                       const int* __restrict__ nbr, const int* __restrict__ box_lev_off,
                                                       const int* __restrict__ lev_ptr,
                                                       const int* __restrict__ box_pos_off, long long Ptot, long long ld,
                                                       long long N, const double* __restrict__ fac,
                                                       const double* __restrict__ r, double* y, double* __restrict__ z,
                                                       int variant) {
  const int b = blockIdx.x;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int q0 = box_pos_off[b], q1 = box_pos_off[b + 1];
  for (int pos = q0 + threadIdx.x; pos < q1; pos += blockDim.x) {
    int gi = gidx[pos];
    const bool owned = gi >= 0;
    if (gi < 0) gi = ~gi;
#pragma unroll
    for (int f = 0; f < NF; ++f) y[f * Ptot + pos] = (variant == 2 && !owned) ? 0.0 : r[f * N + gi];
  }
  __syncthreads();
  const int l0 = box_lev_off[b], l1 = box_lev_off[b + 1] - 1;
  for (int l = l0; l < l1; ++l) {                 // forward: y_i -= sum_k L_ik y_k
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + wid; pos < p1; pos += nw) {
      double acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f] = 0.0;
      for (int a = lane; a < T.nlower; a += 32) {
        const int s = T.lower[a];
        const int k = nbr[(long long)s * Ptot + pos];
        if (k < 0) continue;
        double yk[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) yk[f] = y[f * Ptot + k];
#pragma unroll
        for (int rr = 0; rr < NF; ++rr)
#pragma unroll
          for (int c = 0; c < NF; ++c) acc[rr] = fma(__ldg(fac + ((long long)s * NF * NF + rr * NF + c) * ld + pos), yk[c], acc[rr]);
      }
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o);
      if (lane < NF) {
        double a0 = acc[0];
#pragma unroll
        for (int f = 1; f < NF; ++f) a0 = lane == f ? acc[f] : a0;
        y[lane * Ptot + pos] -= a0;
      }
    }
    __syncthreads();
  }
  for (int l = l1 - 1; l >= l0; --l) {            // backward: x_i = D_i^-1 (y_i - sum_j U_ij x_j)
    const int p0 = lev_ptr[l], p1 = lev_ptr[l + 1];
    for (int pos = p0 + wid; pos < p1; pos += nw) {
      double acc[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) acc[f] = 0.0;
      for (int a = lane; a < T.nupper; a += 32) {
        const int s = T.upper[a];
        const int k = nbr[(long long)s * Ptot + pos];
        if (k < 0) continue;
        double xk[NF];
#pragma unroll
        for (int f = 0; f < NF; ++f) xk[f] = y[f * Ptot + k];
#pragma unroll
        for (int rr = 0; rr < NF; ++rr)
#pragma unroll
          for (int c = 0; c < NF; ++c) acc[rr] = fma(__ldg(fac + ((long long)s * NF * NF + rr * NF + c) * ld + pos), xk[c], acc[rr]);
      }
#pragma unroll
      for (int f = 0; f < NF; ++f)
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) acc[f] += __shfl_xor_sync(0xffffffffu, acc[f], o);
      double rhs[NF];
#pragma unroll
      for (int f = 0; f < NF; ++f) rhs[f] = y[f * Ptot + pos] - acc[f];
      __syncwarp();
      if (lane < NF) {
        double s = 0.0;
#pragma unroll
        for (int c = 0; c < NF; ++c) s = fma(__ldg(fac + ((long long)T.diag * NF * NF + lane * NF + c) * ld + pos), rhs[c], s);
        y[lane * Ptot + pos] = s;
      }
    }
    __syncthreads();
  }
  if (variant != 0) return;
  for (int pos = q0 + threadIdx.x; pos < q1; pos += blockDim.x) {
    const int gi = gidx[pos];
    if (gi < 0) continue;
#pragma unroll
    for (int f = 0; f < NF; ++f) z[f * N + gi] = y[f * Ptot + pos];
  }
}

static GenTables gen_tables(const BoxSet& B) {
  GenTables T;
  T.nslots = B.nslots;
  T.nlower = B.g_nlower;
  T.nupper = B.g_nupper;
  T.diag = B.diag;
  T.off = B.g_off;
  T.lower = B.g_lower;
  T.upper = B.g_upper;
  T.pair_ptr = B.g_pair_ptr;
  T.pair_b = B.g_pair_b;
  T.pair_t = B.g_pair_t;
  return T;
}

void launch_assemble_gen(const DevParams& P, const BoxSet& B, int nf, const double* Xa, const double* jac4, double* fac,
                         cudaStream_t s) {
  const long long total = B.P * B.nslots;
  const int blocks = (int)std::min<long long>((total + 255) / 256, 148 * 32);
  k_assemble_gen<<<blocks, 256, 0, s>>>(P, gen_tables(B), nf, Xa, jac4, B.gidx, B.nbr, B.P, B.ld, fac);
}

void launch_factor_gen(const BoxSet& B, int nf, double* fac, cudaStream_t s) {
  const GenTables T = gen_tables(B);
  if (nf == 4) k_biluk<4><<<B.nbox, 256, 0, s>>>(T, B.nbr, B.box_lev_off, B.lev_ptr, B.P, B.ld, fac);
  else k_biluk<5><<<B.nbox, 256, 0, s>>>(T, B.nbr, B.box_lev_off, B.lev_ptr, B.P, B.ld, fac);
}

void launch_ras_apply_gen(const BoxSet& B, int nf, long long N, const double* fac, const double* r, double* y,
                          double* z, cudaStream_t s) {
  const GenTables T = gen_tables(B);
  if (nf == 4)
    // one warp per row of a wavefront level: 32 warps cover a 2D level (~ex/a rows) in one or two rounds
    k_ras_apply_gen<4><<<B.nbox, 1024, 0, s>>>(T, B.gidx, B.nbr, B.box_lev_off, B.lev_ptr, B.box_pos_off, B.P, B.ld, N, fac,
                                               r, y, z, B.variant);
  else
    k_ras_apply_gen<5><<<B.nbox, 1024, 0, s>>>(T, B.gidx, B.nbr, B.box_lev_off, B.lev_ptr, B.box_pos_off, B.P, B.ld, N, fac,
                                               r, y, z, B.variant);
  if (B.variant != 0) {
    const int blocks = (int)std::min<long long>((N + 255) / 256, 148 * 8);
    k_schwarz_gather<<<blocks, 256, 0, s>>>(N, nf, B.P, B.cover_off, B.cover_pos, y, z);
  }
}

}  // namespace nks
