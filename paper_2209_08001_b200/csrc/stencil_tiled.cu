// K2 (matrix-free J.v) as a shared-memory plane-marching stencil.
//
// The 25-point (3D) / 13-point (2D) operator of the Jacobian action (the
// linearisation of Eq. NSOA-1, with the cached pointwise partials a11..a22) is
//   w_c  = (a11 + cT) v_c + a12 v_eta + cU sum_J D^_J v_{u,J} + cL Lap v_c        (inner term, every point)
//   Jv_c = v_c/dt - (kappa/2h^2) sum_J [(m_i + m_{i+e})(w_{i+e} - w_i) - (m_i + m_{i-e})(w_i - w_{i-e})]
//   Jv_e = v_e/dt + a21 v_c + a22 v_e - (3 gamma_eta/2h^2) Lap v_e
//   Jv_uI = L[C11 D^_I^2 v_uI + C44 sum_{J!=I} D^_J^2 v_uI + (C12+C44) sum_{M!=I} D^_I D^_M v_uM] - K eps0 D^_I v_c
// with m = c^a(1-c^a).  A CTA owns a 32x8 (x,y) tile and marches z: every field plane is loaded from
// HBM once into a shared-memory ring with a 2-cell halo (u: 5 planes z-2..z+2, v_c: 4, v_eta, m: 3),
// the inner term w is evaluated once per point on the tile plus a one-cell ring (ring of 3 planes), and
// every neighbour access is a shared-memory load at a compile-time offset.  In 2D the same code runs
// on one plane.
#include "model.cuh"
#include "nks_internal.cuh"

namespace nks {

namespace tj {
#ifndef NKS_TILE_Y
#define NKS_TILE_Y 16
#endif
constexpr int TX = 32, TY = NKS_TILE_Y, NT = TX * TY;   // 32x16: 512 threads, 1 CTA/SM (J.v 30 -> 36 % of HBM at 256^3 vs 32x8)
constexpr int HX = TX + 4, HY = TY + 4, PL = HX * HY;     // plane with 2-cell halo
constexpr int RX = TX + 2, RY = TY + 2, RL = RX * RY;     // one-cell ring
// F: 640 threads, so the ring pass (612 evaluations of the pointwise DVD quotients, the expensive part)
// is one pass instead of 512 + 100; threads >= TX*TY idle in the interior pass
constexpr int NTF = (RL + 31) / 32 * 32;
}  // namespace tj

__device__ __forceinline__ int tslot(int z, int n) { return ((z % n) + n) % n; }

// sum_J D^_J sigma^el_IJ at the tile centre hc of plane z:
//   L/(4h^2) [C11 D^_I^2 u_I + C44 sum_{J!=I} D^_J^2 u_I + (C12+C44) sum_{M!=I} D^_I D^_M u_M] - K eps0 D^_I c
// u planes: su[(I*NU + slot)*PL], c planes: sc[slot*PL]; z offsets pick ring slots, x/y offsets cells.
template <int DIM, int NU, int NC>
__device__ __forceinline__ double elastic_row_tile(const DevParams& P, int I, const double* su, const double* sc,
                                                   int z, int hc) {
  using namespace tj;
  const int off[3] = {1, HX, PL};
  const double* UI = su + (I * NU + tslot(z, NU)) * PL;
  const double uc = UI[hc];
  double diag = 0.0, offd = 0.0;
#pragma unroll
  for (int J = 0; J < DIM; ++J) {
    double s2;
    if (J < 2) s2 = UI[hc + 2 * off[J]] + UI[hc - 2 * off[J]] - 2.0 * uc;
    else s2 = su[(I * NU + tslot(z + 2, NU)) * PL + hc] + su[(I * NU + tslot(z - 2, NU)) * PL + hc] - 2.0 * uc;
    if (J == I) diag = s2; else offd += s2;
  }
  double mixed = 0.0;
#pragma unroll
  for (int M = 0; M < DIM; ++M) {
    if (M == I) continue;
    const int a = I < M ? I : M, bb = I < M ? M : I;    // bb may be z
    double pp, pm, mp, mm;                               // u_M at (+-e_I, +-e_M)
    if (bb < 2) {
      const double* UM = su + (M * NU + tslot(z, NU)) * PL;
      const int oI = off[I], oM = off[M];
      pp = UM[hc + oI + oM]; pm = UM[hc + oI - oM]; mp = UM[hc - oI + oM]; mm = UM[hc - oI - oM];
    } else {
      const int oa = off[a];
      const double* Mzp = su + (M * NU + tslot(z + 1, NU)) * PL;
      const double* Mzm = su + (M * NU + tslot(z - 1, NU)) * PL;
      if (I == 2) { pp = Mzp[hc + oa]; pm = Mzp[hc - oa]; mp = Mzm[hc + oa]; mm = Mzm[hc - oa]; }
      else { pp = Mzp[hc + oa]; pm = Mzm[hc + oa]; mp = Mzp[hc - oa]; mm = Mzm[hc - oa]; }
    }
    mixed += (pp - pm) - (mp - mm);
  }
  const double el = P.Ls * P.inv_4h2 * (P.C11 * diag + P.C44 * offd + (P.C12 + P.C44) * mixed);
  double dc;
  if (I < 2) {
    const double* C0 = sc + tslot(z, NC) * PL;
    dc = C0[hc + off[I]] - C0[hc - off[I]];
  } else {
    dc = sc[tslot(z + 1, NC) * PL + hc] - sc[tslot(z - 1, NC) * PL + hc];
  }
  return el - P.K * P.eps0 * P.inv_2h * dc;
}

template <int DIM>
__global__ void __launch_bounds__(tj::NTF) k_jv_tiled(DevParams P, const double* __restrict__ Xa,
                                                     const double* __restrict__ jac4, const double* __restrict__ v,
                                                     double* __restrict__ out, int zc) {
  using namespace tj;
  constexpr int NU = DIM == 3 ? 5 : 1;     // u planes
  constexpr int NC = DIM == 3 ? 4 : 1;     // v_c planes (z-1..z+2)
  constexpr int N3 = DIM == 3 ? 3 : 1;     // v_eta, m, w planes
  extern __shared__ __align__(16) double sm[];
  double* su = sm;                           // [DIM][NU][PL]
  double* sc = su + DIM * NU * PL;           // [NC][PL]
  double* se = sc + NC * PL;                 // [N3][PL]
  double* smo = se + N3 * PL;                // [N3][PL]   mobility m = c^a (1 - c^a)
  double* sa = smo + N3 * PL;                // [2][PL]    a11, a12 of the plane whose w is computed
  double* sw = sa + 2 * PL;                  // [N3][RL]

  const long long N = P.N;
  const int nx = P.nx, ny = P.ny, nz = P.nz, zg = P.zg, yg = P.yg;
  const int ncz = nz - 2 * zg;                 // computed planes (all, or the slab's own planes)
  const int ncy = ny - 2 * yg;                 // computed rows (all, or the pencil's own rows)
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = DIM == 3 ? blockIdx.z * zc : 0;
  const int z1 = DIM == 3 ? min(z0 + zc, ncz) : 1;
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;

  // per-thread halo cells (2 per thread: PL = 432 <= 2 * 256) -> in-plane global offset (wrapped)
  int cell[2];
  long long goff[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int c = tid + r * NTF;
    cell[r] = c < PL ? c : -1;
    int gx = x0 + (c % HX) - 2, gy = y0 + (c / HX) - 2 + yg;   // pencil: own rows start at yg, ghost rows below
    gx = ((gx % nx) + nx) % nx;        // tiles may be wider than the grid
    gy = ((gy % ny) + ny) % ny;
    goff[r] = (long long)gy * nx + gx;
  }
  auto zw = [&](int z) { return zg ? z + zg : (z < 0 ? z + nz : (z >= nz ? z - nz : z)); };   // memory plane
  auto load_plane = [&](double* dst, const double* src, int z) {
    const long long base = (long long)zw(z) * nx * ny;
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (cell[r] >= 0) dst[cell[r]] = __ldg(src + base + goff[r]);
  };
  auto load_mob = [&](double* dst, int z) {
    const long long base = (long long)zw(z) * nx * ny;
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (cell[r] >= 0) {
        const double c = __ldg(Xa + base + goff[r]);
        dst[cell[r]] = c * (1.0 - c);
      }
  };
  auto slot = [](int z, int n) { return ((z % n) + n) % n; };
  const double* vc_ = v;
  const double* ve_ = v + N;
  const double* vu_ = v + 2 * N;
  const double cT = 0.5 * P.K * DIM * P.eps0 * P.eps0;     // d(G3_c)/d(c^b)
  const double cU = -0.5 * P.eps0 * P.K * P.inv_2h;        // d(G3_c)/d(sum D^ u) (D^ scale folded)
  const double cL = -0.5 * P.gamma_c * P.inv_h2;           // d(G4_c)/d(c^b) Laplacian weight

  // inner term on the ring of plane z (reads planes z-1..z+1 of v_c, u_z; plane z of the rest)
  auto compute_w = [&](int z) {
    const double* C0 = sc + slot(z, NC) * PL;
    const double* E0 = se + slot(z, N3) * PL;
    const double* Ux = su + (0 * NU + slot(z, NU)) * PL;
    const double* Uy = su + (1 * NU + slot(z, NU)) * PL;
    double* W = sw + slot(z, N3) * RL;
    for (int r = tid; r < RL; r += NTF) {
      const int rx = r % RX, ry = r / RX;
      const int k = (ry + 1) * HX + (rx + 1);
      const double vc = C0[k];
      double lap = C0[k - 1] + C0[k + 1] + C0[k - HX] + C0[k + HX] - 4.0 * vc;
      double div = (Ux[k + 1] - Ux[k - 1]) + (Uy[k + HX] - Uy[k - HX]);
      if (DIM == 3) {
        const double* Cm = sc + slot(z - 1, NC) * PL;
        const double* Cp = sc + slot(z + 1, NC) * PL;
        const double* Uzm = su + (2 * NU + slot(z - 1, NU)) * PL;
        const double* Uzp = su + (2 * NU + slot(z + 1, NU)) * PL;
        lap += Cm[k] + Cp[k] - 2.0 * vc;
        div += Uzp[k] - Uzm[k];
      }
      W[r] = (sa[k] + cT) * vc + sa[PL + k] * E0[k] + cU * div + cL * lap;
    }
  };

  // ---- prologue: planes needed before the first output plane
  if (DIM == 3) {
    for (int z = z0 - 2; z <= z0 + 1; ++z)
      for (int I = 0; I < 3; ++I) load_plane(su + (I * NU + slot(z, NU)) * PL, vu_ + (long long)I * N, z);
    for (int z = z0 - 2; z <= z0 + 1; ++z) load_plane(sc + slot(z, NC) * PL, vc_, z);
    for (int z = z0 - 1; z <= z0; ++z) {
      load_plane(se + slot(z, N3) * PL, ve_, z);
      load_mob(smo + slot(z, N3) * PL, z);
    }
    load_plane(sa, jac4, z0 - 1);
    load_plane(sa + PL, jac4 + N, z0 - 1);
    __syncthreads();
    compute_w(z0 - 1);
    __syncthreads();
    load_plane(sa, jac4, z0);
    load_plane(sa + PL, jac4 + N, z0);
    __syncthreads();
    compute_w(z0);
    __syncthreads();
  } else {
    for (int I = 0; I < 2; ++I) load_plane(su + I * PL, vu_ + (long long)I * N, 0);
    load_plane(sc, vc_, 0);
    load_plane(se, ve_, 0);
    load_mob(smo, 0);
    load_plane(sa, jac4, 0);
    load_plane(sa + PL, jac4 + N, 0);
    __syncthreads();
    compute_w(0);
    __syncthreads();
  }

  const double kap = 0.5 * P.kappa * P.inv_h2;
  const double eta_l = -1.5 * P.gamma_eta * P.inv_h2;
  const int hc = (ty + 2) * HX + (tx + 2);     // centre in the halo plane
  const int rc = (ty + 1) * RX + (tx + 1);     // centre in the ring
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < nx && y < ncy && tid < NT;

  // register prefetch of the planes the NEXT iteration commits to shared memory (hides HBM latency
  // behind this iteration's arithmetic): u_x,u_y,u_z, v_c at z+2; v_eta, c^a, a11, a12 at z+1
  double R[8][2];
  double A21 = 0.0, A22 = 0.0;                   // centre a21, a22 of the plane the iteration outputs
  const long long gc_off = (long long)(min(y0 + ty, ncy - 1) + yg) * nx + min(x0 + tx, nx - 1);
  auto fetch = [&](int z) {
    const long long b2 = (long long)zw(z + 2) * nx * ny, b1 = (long long)zw(z + 1) * nx * ny;
    const long long b0 = (long long)zw(z) * nx * ny;
    A21 = __ldg(jac4 + 2 * N + b0 + gc_off);
    A22 = __ldg(jac4 + 3 * N + b0 + gc_off);
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (cell[r] < 0) continue;
      R[0][r] = __ldg(vu_ + b2 + goff[r]);
      R[1][r] = __ldg(vu_ + N + b2 + goff[r]);
      R[2][r] = __ldg(vu_ + 2 * N + b2 + goff[r]);
      R[3][r] = __ldg(vc_ + b2 + goff[r]);
      R[4][r] = __ldg(ve_ + b1 + goff[r]);
      R[5][r] = __ldg(Xa + b1 + goff[r]);
      R[6][r] = __ldg(jac4 + b1 + goff[r]);
      R[7][r] = __ldg(jac4 + N + b1 + goff[r]);
    }
  };
  auto commit = [&](int z) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (cell[r] < 0) continue;
      const int c = cell[r];
      su[(0 * NU + slot(z + 2, NU)) * PL + c] = R[0][r];
      su[(1 * NU + slot(z + 2, NU)) * PL + c] = R[1][r];
      su[(2 * NU + slot(z + 2, NU)) * PL + c] = R[2][r];
      sc[slot(z + 2, NC) * PL + c] = R[3][r];
      se[slot(z + 1, N3) * PL + c] = R[4][r];
      smo[slot(z + 1, N3) * PL + c] = R[5][r] * (1.0 - R[5][r]);
      sa[c] = R[6][r];
      sa[PL + c] = R[7][r];
    }
  };
  if (DIM == 3) fetch(z0);
  else {
    A21 = __ldg(jac4 + 2 * N + gc_off);
    A22 = __ldg(jac4 + 3 * N + gc_off);
  }

  for (int z = z0; z < z1; ++z) {
    const double a21 = A21, a22 = A22;
    if (DIM == 3) {
      commit(z);
      if (z + 1 < z1) fetch(z + 1);
      __syncthreads();
      compute_w(z + 1);
      __syncthreads();
    }
    if (inside) {
      const long long i = ((long long)(z + zg) * ny + (y + yg)) * nx + x;
      const double* C0 = sc + slot(z, NC) * PL;
      const double* E0 = se + slot(z, N3) * PL;
      const double* M0 = smo + slot(z, N3) * PL;
      const double* W0 = sw + slot(z, N3) * RL;
      // ---- c row: v_c/dt - D M~ D w
      const double mi = M0[hc];
      const double Wc = W0[rc];
      double div = (mi + M0[hc + 1]) * (W0[rc + 1] - Wc) - (mi + M0[hc - 1]) * (Wc - W0[rc - 1]) +
                   (mi + M0[hc + HX]) * (W0[rc + RX] - Wc) - (mi + M0[hc - HX]) * (Wc - W0[rc - RX]);
      if (DIM == 3) {
        const double* Mm = smo + slot(z - 1, N3) * PL;
        const double* Mp = smo + slot(z + 1, N3) * PL;
        const double* Wm = sw + slot(z - 1, N3) * RL;
        const double* Wp = sw + slot(z + 1, N3) * RL;
        div += (mi + Mp[hc]) * (Wp[rc] - Wc) - (mi + Mm[hc]) * (Wc - Wm[rc]);
      }
      const double vc = C0[hc];
      out[i] = vc * P.inv_dt - kap * div;
      // ---- eta row
      const double ve = E0[hc];
      double lape = E0[hc - 1] + E0[hc + 1] + E0[hc - HX] + E0[hc + HX] - 4.0 * ve;
      if (DIM == 3) lape += se[slot(z - 1, N3) * PL + hc] + se[slot(z + 1, N3) * PL + hc] - 2.0 * ve;
      out[N + i] = ve * P.inv_dt + a21 * vc + a22 * ve + eta_l * lape;
      // ---- u rows: elastic operator on v_u with the eigen-term -K eps0 D^_I v_c
#pragma unroll
      for (int I = 0; I < DIM; ++I) out[(2 + I) * N + i] = elastic_row_tile<DIM, NU, NC>(P, I, su, sc, z, hc);
    }
    if (DIM == 3) __syncthreads();     // the next iteration overwrites planes this one read
  }
}

template <int DIM>
__global__ void __launch_bounds__(tj::NTF) k_residual_tiled(DevParams P, const double* __restrict__ Xa,
                                                           const double* __restrict__ Xb, const double* __restrict__ Ta,
                                                           double* __restrict__ F, int zc) {
  using namespace tj;
  constexpr int NU = DIM == 3 ? 5 : 1;     // u^b planes z-2..z+2
  constexpr int NC = DIM == 3 ? 4 : 1;     // c^a, c^b planes z-1..z+2
  constexpr int N3 = DIM == 3 ? 3 : 1;     // eta^a, eta^b, G planes z-1..z+1
  extern __shared__ __align__(16) double sm[];
  double* su = sm;                           // [DIM][NU][PL]  u^b
  double* scb = su + DIM * NU * PL;          // [NC][PL]       c^b
  double* sca = scb + NC * PL;               // [NC][PL]       c^a
  double* sea = sca + NC * PL;               // [N3][PL]       eta^a
  double* seb = sea + N3 * PL;               // [N3][PL]       eta^b
  double* sT = seb + N3 * PL;                // [PL]           T^a of the plane whose G is computed
  double* sg = sT + PL;                      // [N3][RL]       G_c

  const long long N = P.N;
  const int nx = P.nx, ny = P.ny, nz = P.nz, zg = P.zg, yg = P.yg;
  const int ncz = nz - 2 * zg;                 // computed planes (all, or the slab's own planes)
  const int ncy = ny - 2 * yg;                 // computed rows (all, or the pencil's own rows)
  const int x0 = blockIdx.x * TX, y0 = blockIdx.y * TY;
  const int z0 = DIM == 3 ? blockIdx.z * zc : 0;
  const int z1 = DIM == 3 ? min(z0 + zc, ncz) : 1;
  const int tid = threadIdx.x;
  const int tx = tid % TX, ty = tid / TX;
  int cell[2];
  long long goff[2];
#pragma unroll
  for (int r = 0; r < 2; ++r) {
    const int c = tid + r * NTF;
    cell[r] = c < PL ? c : -1;
    int gx = x0 + (c % HX) - 2, gy = y0 + (c / HX) - 2 + yg;
    gx = ((gx % nx) + nx) % nx;
    gy = ((gy % ny) + ny) % ny;
    goff[r] = (long long)gy * nx + gx;
  }
  auto zw = [&](int z) { return zg ? z + zg : (z < 0 ? z + nz : (z >= nz ? z - nz : z)); };   // memory plane
  auto load_plane = [&](double* dst, const double* src, int z) {
    const long long base = (long long)zw(z) * nx * ny;
#pragma unroll
    for (int r = 0; r < 2; ++r)
      if (cell[r] >= 0) dst[cell[r]] = __ldg(src + base + goff[r]);
  };
  const double* ca_ = Xa;
  const double* ea_ = Xa + N;
  const double* cb_ = Xb;
  const double* eb_ = Xb + N;
  const double* ub_ = Xb + 2 * N;
  const double gcl = -P.gamma_c * P.inv_h2;

  // G_c on the ring of plane z: needs c^a, c^b at z-1..z+1, u^b_z at z+-1, u^b_x,y and eta at z, T^a at z
  // ... and, for the tile's own points of a plane this CTA owns, the whole eta row F_eta (its
  // pointwise part comes out of the same pointwise_G call; Lap eta^h needs eta at z-1..z+1)
  const double gel = -1.5 * P.gamma_eta * P.inv_h2;      // -3 gamma_eta Lap eta^h, eta^h = (eta^a + eta^b)/2
  auto compute_g = [&](int z, bool write_eta) {
    const double* CA = sca + tslot(z, NC) * PL;
    const double* CB = scb + tslot(z, NC) * PL;
    const double* EA = sea + tslot(z, N3) * PL;
    const double* EB = seb + tslot(z, N3) * PL;
    const double* Ux = su + (0 * NU + tslot(z, NU)) * PL;
    const double* Uy = su + (1 * NU + tslot(z, NU)) * PL;
    double* Gp = sg + tslot(z, N3) * RL;
    for (int r = tid; r < RL; r += NTF) {
      const int rx = r % RX, ry = r / RX;
      const int k = (ry + 1) * HX + (rx + 1);
      const double ca = CA[k], cb = CB[k];
      double gc, ge;
      pointwise_G(P, ca, cb, EA[k], EB[k], gc, ge);
      double lap = (CA[k - 1] + CB[k - 1]) + (CA[k + 1] + CB[k + 1]) + (CA[k - HX] + CB[k - HX]) +
                   (CA[k + HX] + CB[k + HX]) - 4.0 * (ca + cb);
      double div = (Ux[k + 1] - Ux[k - 1]) + (Uy[k + HX] - Uy[k - HX]);
      if (DIM == 3) {
        const double* CAm = sca + tslot(z - 1, NC) * PL;
        const double* CAp = sca + tslot(z + 1, NC) * PL;
        const double* CBm = scb + tslot(z - 1, NC) * PL;
        const double* CBp = scb + tslot(z + 1, NC) * PL;
        const double* Uzm = su + (2 * NU + tslot(z - 1, NU)) * PL;
        const double* Uzp = su + (2 * NU + tslot(z + 1, NU)) * PL;
        lap += (CAm[k] + CBm[k]) + (CAp[k] + CBp[k]) - 2.0 * (ca + cb);
        div += Uzp[k] - Uzm[k];
      }
      const double Tb = P.K * (div * P.inv_2h - DIM * P.eps0 * (cb - P.cbar0));
      Gp[r] = gc - 0.5 * P.eps0 * (sT[k] + Tb) + gcl * 0.5 * lap;
      const int px = x0 + rx - 1, py = y0 + ry - 1;
      if (write_eta && rx >= 1 && rx <= TX && ry >= 1 && ry <= TY && px < nx && py < ncy) {
        const double ea = EA[k], eb = EB[k];
        double le = (EA[k - 1] + EB[k - 1]) + (EA[k + 1] + EB[k + 1]) + (EA[k - HX] + EB[k - HX]) +
                    (EA[k + HX] + EB[k + HX]) - 4.0 * (ea + eb);
        if (DIM == 3) {
          const int m1 = tslot(z - 1, N3) * PL + k, p1 = tslot(z + 1, N3) * PL + k;
          le += (sea[m1] + seb[m1]) + (sea[p1] + seb[p1]) - 2.0 * (ea + eb);
        }
        const long long i = ((long long)(z + zg) * ny + (py + yg)) * nx + px;
        F[N + i] = (eb - ea) * P.inv_dt + ge + gel * le;
      }
    }
  };

  if (DIM == 3) {
    for (int z = z0 - 2; z <= z0 + 1; ++z)
      for (int I = 0; I < 3; ++I) load_plane(su + (I * NU + tslot(z, NU)) * PL, ub_ + (long long)I * N, z);
    for (int z = z0 - 2; z <= z0 + 1; ++z) {
      load_plane(scb + tslot(z, NC) * PL, cb_, z);
      load_plane(sca + tslot(z, NC) * PL, ca_, z);
    }
    for (int z = z0 - 1; z <= z0 + 1; ++z) {
      load_plane(sea + tslot(z, N3) * PL, ea_, z);
      load_plane(seb + tslot(z, N3) * PL, eb_, z);
    }
    load_plane(sT, Ta, z0 - 1);
    __syncthreads();
    compute_g(z0 - 1, false);
    __syncthreads();
    load_plane(sT, Ta, z0);
    __syncthreads();
    compute_g(z0, true);
    __syncthreads();
  } else {
    for (int I = 0; I < 2; ++I) load_plane(su + I * PL, ub_ + (long long)I * N, 0);
    load_plane(scb, cb_, 0);
    load_plane(sca, ca_, 0);
    load_plane(sea, ea_, 0);
    load_plane(seb, eb_, 0);
    load_plane(sT, Ta, 0);
    __syncthreads();
    compute_g(0, true);
    __syncthreads();
  }

  const double kap = 0.5 * P.kappa * P.inv_h2;
  const int hc = (ty + 2) * HX + (tx + 2);
  const int rc = (ty + 1) * RX + (tx + 1);
  const int x = x0 + tx, y = y0 + ty;
  const bool inside = x < nx && y < ncy && tid < NT;

  // register prefetch of the next iteration's planes: u^b (3), c^b, c^a, eta^a, eta^b at z+2; T^a at z+1
  double R[8][2];
  auto fetch = [&](int z) {
    const long long b2 = (long long)zw(z + 2) * nx * ny, b1 = (long long)zw(z + 1) * nx * ny;
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (cell[r] < 0) continue;
      R[0][r] = __ldg(ub_ + b2 + goff[r]);
      R[1][r] = __ldg(ub_ + N + b2 + goff[r]);
      R[2][r] = __ldg(ub_ + 2 * N + b2 + goff[r]);
      R[3][r] = __ldg(cb_ + b2 + goff[r]);
      R[4][r] = __ldg(ca_ + b2 + goff[r]);
      R[5][r] = __ldg(ea_ + b2 + goff[r]);
      R[6][r] = __ldg(eb_ + b2 + goff[r]);
      R[7][r] = __ldg(Ta + b1 + goff[r]);
    }
  };
  auto commit = [&](int z) {
#pragma unroll
    for (int r = 0; r < 2; ++r) {
      if (cell[r] < 0) continue;
      const int c = cell[r];
      su[(0 * NU + tslot(z + 2, NU)) * PL + c] = R[0][r];
      su[(1 * NU + tslot(z + 2, NU)) * PL + c] = R[1][r];
      su[(2 * NU + tslot(z + 2, NU)) * PL + c] = R[2][r];
      scb[tslot(z + 2, NC) * PL + c] = R[3][r];
      sca[tslot(z + 2, NC) * PL + c] = R[4][r];
      sea[tslot(z + 2, N3) * PL + c] = R[5][r];
      seb[tslot(z + 2, N3) * PL + c] = R[6][r];
      sT[c] = R[7][r];
    }
  };
  if (DIM == 3) fetch(z0);

  for (int z = z0; z < z1; ++z) {
    if (DIM == 3) {
      commit(z);
      if (z + 1 < z1) fetch(z + 1);
      __syncthreads();
      compute_g(z + 1, z + 1 < z1);
      __syncthreads();
    }
    if (inside) {
      const long long i = ((long long)(z + zg) * ny + (y + yg)) * nx + x;
      const double* CA = sca + tslot(z, NC) * PL;
      const double* CB = scb + tslot(z, NC) * PL;
      const double* G0 = sg + tslot(z, N3) * RL;
      // ---- c row
      const double cai = CA[hc];
      const double mi = cai * (1.0 - cai);
      auto mob = [](double c) { return c * (1.0 - c); };
      const double Gc = G0[rc];
      double div = (mi + mob(CA[hc + 1])) * (G0[rc + 1] - Gc) - (mi + mob(CA[hc - 1])) * (Gc - G0[rc - 1]) +
                   (mi + mob(CA[hc + HX])) * (G0[rc + RX] - Gc) - (mi + mob(CA[hc - HX])) * (Gc - G0[rc - RX]);
      if (DIM == 3) {
        const double cm = sca[tslot(z - 1, NC) * PL + hc], cp = sca[tslot(z + 1, NC) * PL + hc];
        const double Gm = sg[tslot(z - 1, N3) * RL + rc], Gpp = sg[tslot(z + 1, N3) * RL + rc];
        div += (mi + mob(cp)) * (Gpp - Gc) - (mi + mob(cm)) * (Gc - Gm);
      }
      F[i] = (CB[hc] - cai) * P.inv_dt - kap * div;
      // ---- u rows
#pragma unroll
      for (int I = 0; I < DIM; ++I) F[(2 + I) * N + i] = elastic_row_tile<DIM, NU, NC>(P, I, su, scb, z, hc);
    }
    if (DIM == 3) __syncthreads();
  }
}

size_t residual_tiled_smem(int dim) {
  using namespace tj;
  const int NU = dim == 3 ? 5 : 1, NC = dim == 3 ? 4 : 1, N3 = dim == 3 ? 3 : 1;
  return sizeof(double) * ((size_t)dim * NU * PL + 2 * NC * PL + 2 * N3 * PL + PL + (size_t)N3 * RL);
}

void launch_residual_tiled(const DevParams& P, const double* Xa, const double* Xb, const double* Ta, double* F,
                           cudaStream_t s) {
  using namespace tj;
  const int dim = P.dim;
  const size_t smem = residual_tiled_smem(dim);
  // the smem opt-in is per device: cached per (device, dim); a failure surfaces at the launch below
  static bool attr[64][4] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev][dim]) {
    if (dim == 2) cudaFuncSetAttribute(k_residual_tiled<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else cudaFuncSetAttribute(k_residual_tiled<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr[dev][dim] = true;
  }
  const int tiles = ((P.nx + TX - 1) / TX) * ((P.ny - 2 * P.yg + TY - 1) / TY);
  int zc = 1;
  if (dim == 3) {
    const int ncz = P.nz - 2 * P.zg;
    zc = ncz;
    while (zc > 16 && (long long)tiles * ((ncz + zc - 1) / zc) < 148 * 2 * 4) zc = (zc + 1) / 2;
  }
  dim3 grid((P.nx + TX - 1) / TX, (P.ny - 2 * P.yg + TY - 1) / TY, dim == 3 ? (P.nz - 2 * P.zg + zc - 1) / zc : 1);
  if (dim == 2) k_residual_tiled<2><<<grid, NTF, smem, s>>>(P, Xa, Xb, Ta, F, zc);
  else k_residual_tiled<3><<<grid, NTF, smem, s>>>(P, Xa, Xb, Ta, F, zc);
}

size_t jv_tiled_smem(int dim) {
  using namespace tj;
  const int NU = dim == 3 ? 5 : 1, NC = dim == 3 ? 4 : 1, N3 = dim == 3 ? 3 : 1;
  return sizeof(double) * ((size_t)dim * NU * PL + NC * PL + N3 * PL + N3 * PL + 2 * PL + (size_t)N3 * RL);
}

void launch_jv_tiled(const DevParams& P, const double* Xa, const double* jac4, const double* v, double* out,
                     cudaStream_t s) {
  using namespace tj;
  const int dim = P.dim;
  const size_t smem = jv_tiled_smem(dim);
  // the smem opt-in is per device: cached per (device, dim); a failure surfaces at the launch below
  static bool attr[64][4] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || !attr[dev][dim]) {
    if (dim == 2) cudaFuncSetAttribute(k_jv_tiled<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    else cudaFuncSetAttribute(k_jv_tiled<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (dev >= 0 && dev < 64) attr[dev][dim] = true;
  }
  const int tiles = ((P.nx + TX - 1) / TX) * ((P.ny - 2 * P.yg + TY - 1) / TY);
  int zc = 1;
  if (dim == 3) {
    // z chunks: enough CTAs for ~4 waves of 2 CTAs/SM, chunks long enough to amortise the 4-plane prologue
    const int ncz = P.nz - 2 * P.zg;
    zc = ncz;
    while (zc > 16 && (long long)tiles * ((ncz + zc - 1) / zc) < 148 * 2 * 4) zc = (zc + 1) / 2;
  }
  dim3 grid((P.nx + TX - 1) / TX, (P.ny - 2 * P.yg + TY - 1) / TY, dim == 3 ? (P.nz - 2 * P.zg + zc - 1) / zc : 1);
  if (dim == 2) k_jv_tiled<2><<<grid, NTF, smem, s>>>(P, Xa, jac4, v, out, zc);
  else k_jv_tiled<3><<<grid, NTF, smem, s>>>(P, Xa, jac4, v, out, zc);
}

}  // namespace nks

// ===================================================================================================
// K1: residual F of Eq. NSOA-1 on the same plane-marching tiles.
//   G_c = G1_c + G2S_c - (eps0/2)(T^a + T^b) - gamma_c Lap c^h      on the tile + one-cell ring (ring of 3 planes)
//   F_c = (c^b - c^a)/dt - (kappa/2h^2) sum_J [(m_i + m_{i+e})(G_{i+e} - G_i) - (m_i + m_{i-e})(G_i - G_{i-e})]
//   F_e = (eta^b - eta^a)/dt + G1_e + G2S_e - 3 gamma_eta Lap eta^h   (centre only)
//   F_uI = sum_J D^_J sigma^el_IJ(u^b, c^b)
// T^b = K (sum_J D^_J u^b_J - d eps0 (c^b - cbar0)); m = c^a (1 - c^a).
