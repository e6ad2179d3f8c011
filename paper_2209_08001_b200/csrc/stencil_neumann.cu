// Residual F (K1) and J.v (K2) with homogeneous Neumann boundaries (Eq. (boundaryequ); SURVEY
// 8(f)-2; reading R38 of DESIGN.md): cell-centred grid, mirror ghosts reflected about the boundary face
// (f_{-1-k} = f_k, f_{N+k} = f_{N-1-k}) for c, eta, u and the mobility -- so the Laplacians and the flux
// form D M~ D carry no flux through a boundary face -- and ODD ghosts of the stress in the outer derivative
// of the u rows, F_uI = sum_J D^_J sigma_IJ with sigma_IJ(-1) = -sigma_IJ(0) across a J face: the u rows
// are then minus the gradient of the discrete elastic energy, whose natural boundary condition is the
// traction-free n . sigma = 0.  One thread per point, every neighbour read through the mirror map (the
// periodic path keeps the tiled kernels of stencil_tiled.cu; this one is for correctness first).
#include "model.cuh"
#include "nks_internal.cuh"

namespace nks {
namespace nm {

__device__ __forceinline__ int mir(int i, int n) { return i < 0 ? -1 - i : (i >= n ? 2 * n - 1 - i : i); }

struct G3 {
  int nx, ny, nz;
  long long N;
  __device__ __forceinline__ long long id(int x, int y, int z) const {
    return ((long long)mir(z, nz) * ny + mir(y, ny)) * nx + mir(x, nx);
  }
  __device__ __forceinline__ bool inside(int x, int y, int z) const {
    return x >= 0 && x < nx && y >= 0 && y < ny && z >= 0 && z < nz;
  }
};

template <int DIM>
__device__ __forceinline__ void step3(int J, int s, int& dx, int& dy, int& dz) {
  dx = J == 0 ? s : 0;
  dy = J == 1 ? s : 0;
  dz = J == 2 ? s : 0;
}

// D^_J f at q (even mirror ghosts)
template <int DIM>
__device__ __forceinline__ double dhat(const G3& g, const double* __restrict__ f, int x, int y, int z, int J,
                                       double inv_2h) {
  int dx, dy, dz;
  step3<DIM>(J, 1, dx, dy, dz);
  return (__ldg(f + g.id(x + dx, y + dy, z + dz)) - __ldg(f + g.id(x - dx, y - dy, z - dz))) * inv_2h;
}

// Laplacian (mirror ghosts) of f at q, scaled by 1/h^2 outside
template <int DIM>
__device__ __forceinline__ double lap(const G3& g, const double* __restrict__ f, int x, int y, int z) {
  const double c = __ldg(f + g.id(x, y, z));
  double a = 0.0;
#pragma unroll
  for (int J = 0; J < DIM; ++J) {
    int dx, dy, dz;
    step3<DIM>(J, 1, dx, dy, dz);
    a += __ldg(f + g.id(x + dx, y + dy, z + dz)) + __ldg(f + g.id(x - dx, y - dy, z - dz)) - 2.0 * c;
  }
  return a;
}

// sigma_IJ at an in-domain point q from eps(u) (even mirror ghosts of u) and the eigenstrain of c
template <int DIM>
__device__ __forceinline__ double sigma(const DevParams& P, const G3& g, const double* __restrict__ u,
                                        const double* __restrict__ c, double cshift, int I, int J, int x, int y, int z) {
  const long long N = g.N;
  if (I == J) {
    double tr = 0.0, eII = 0.0;
    const double e0 = P.eps0 * (__ldg(c + g.id(x, y, z)) - cshift);
#pragma unroll
    for (int M = 0; M < DIM; ++M) {
      const double e = dhat<DIM>(g, u + M * N, x, y, z, M, P.inv_2h) - e0;
      tr += e;
      if (M == I) eII = e;
    }
    return P.Ls * (P.C12 * tr + (P.C11 - P.C12) * eII);
  }
  const double eIJ = 0.5 * (dhat<DIM>(g, u + I * N, x, y, z, J, P.inv_2h) + dhat<DIM>(g, u + J * N, x, y, z, I, P.inv_2h));
  return P.Ls * 2.0 * P.C44 * eIJ;
}

// sum_J D^_J sigma_IJ at p with odd stress ghosts across the J faces
template <int DIM>
__device__ __forceinline__ double urow(const DevParams& P, const G3& g, const double* __restrict__ u,
                                       const double* __restrict__ c, double cshift, int I, int x, int y, int z) {
  double acc = 0.0;
#pragma unroll
  for (int J = 0; J < DIM; ++J) {
    int dx, dy, dz;
    step3<DIM>(J, 1, dx, dy, dz);
    const double sp = g.inside(x + dx, y + dy, z + dz) ? sigma<DIM>(P, g, u, c, cshift, I, J, x + dx, y + dy, z + dz)
                                                      : -sigma<DIM>(P, g, u, c, cshift, I, J, x, y, z);
    const double sm = g.inside(x - dx, y - dy, z - dz) ? sigma<DIM>(P, g, u, c, cshift, I, J, x - dx, y - dy, z - dz)
                                                      : -sigma<DIM>(P, g, u, c, cshift, I, J, x, y, z);
    acc += sp - sm;
  }
  return acc * P.inv_2h;
}

// G_c (all four parts of the DVD gradient, c component) at an in-domain point q
template <int DIM>
__device__ __forceinline__ double Gc_at(const DevParams& P, const G3& g, const double* __restrict__ Xa,
                                        const double* __restrict__ Xb, const double* __restrict__ Ta, int x, int y,
                                        int z, double& ge_out) {
  const long long N = g.N;
  const long long i = g.id(x, y, z);
  const double ca = __ldg(Xa + i), cb = __ldg(Xb + i), ea = __ldg(Xa + N + i), eb = __ldg(Xb + N + i);
  double gc, ge;
  pointwise_G(P, ca, cb, ea, eb, gc, ge);
  double divu = 0.0;
#pragma unroll
  for (int J = 0; J < DIM; ++J) divu += dhat<DIM>(g, Xb + (2 + J) * N, x, y, z, J, P.inv_2h);
  const double Tb = P.K * (divu - DIM * P.eps0 * (cb - P.cbar0));
  const double lc = 0.5 * (lap<DIM>(g, Xa, x, y, z) + lap<DIM>(g, Xb, x, y, z));
  const double le = 0.5 * (lap<DIM>(g, Xa + N, x, y, z) + lap<DIM>(g, Xb + N, x, y, z));
  ge_out = ge - 3.0 * P.gamma_eta * P.inv_h2 * le;
  return gc - 0.5 * P.eps0 * (__ldg(Ta + i) + Tb) - P.gamma_c * P.inv_h2 * lc;
}

template <int DIM>
__global__ void k_residual_neumann(DevParams P, const double* __restrict__ Xa, const double* __restrict__ Xb,
                                   const double* __restrict__ Ta, double* __restrict__ F) {
  const G3 g{P.nx, P.ny, P.nz, P.N};
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx), y = (int)((i / P.nx) % P.ny), z = (int)(i / ((long long)P.nx * P.ny));
    double ge;
    const double Gc = Gc_at<DIM>(P, g, Xa, Xb, Ta, x, y, z, ge);
    const double ma = __ldg(Xa + i) * (1.0 - __ldg(Xa + i));
    double div = 0.0;
#pragma unroll
    for (int J = 0; J < DIM; ++J)
#pragma unroll
      for (int s = -1; s <= 1; s += 2) {
        int dx, dy, dz;
        step3<DIM>(J, s, dx, dy, dz);
        if (!g.inside(x + dx, y + dy, z + dz)) continue;          // no flux through a boundary face
        double gq;
        const double Gq = Gc_at<DIM>(P, g, Xa, Xb, Ta, x + dx, y + dy, z + dz, gq);
        const double cq = __ldg(Xa + g.id(x + dx, y + dy, z + dz));
        div += (ma + cq * (1.0 - cq)) * (Gq - Gc);
      }
    F[i] = (__ldg(Xb + i) - __ldg(Xa + i)) * P.inv_dt - 0.5 * P.kappa * P.inv_h2 * div;
    F[N + i] = (__ldg(Xb + N + i) - __ldg(Xa + N + i)) * P.inv_dt + ge;
#pragma unroll
    for (int I = 0; I < DIM; ++I) F[(2 + I) * N + i] = urow<DIM>(P, g, Xb + 2 * N, Xb, P.cbar0, I, x, y, z);
  }
}

// inner term of J.v at an in-domain point q
template <int DIM>
__device__ __forceinline__ double wc_at(const DevParams& P, const G3& g, const double* __restrict__ jac4,
                                        const double* __restrict__ v, int x, int y, int z) {
  const long long N = g.N;
  const long long i = g.id(x, y, z);
  const double vc = __ldg(v + i);
  double divu = 0.0;
#pragma unroll
  for (int J = 0; J < DIM; ++J) divu += dhat<DIM>(g, v + (2 + J) * N, x, y, z, J, P.inv_2h);
  const double cT = 0.5 * P.K * DIM * P.eps0 * P.eps0;
  return (__ldg(jac4 + i) + cT) * vc + __ldg(jac4 + N + i) * __ldg(v + N + i) - 0.5 * P.eps0 * P.K * divu -
         0.5 * P.gamma_c * P.inv_h2 * lap<DIM>(g, v, x, y, z);
}

template <int DIM>
__global__ void k_jv_neumann(DevParams P, const double* __restrict__ Xa, const double* __restrict__ jac4,
                             const double* __restrict__ v, double* __restrict__ out) {
  const G3 g{P.nx, P.ny, P.nz, P.N};
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx), y = (int)((i / P.nx) % P.ny), z = (int)(i / ((long long)P.nx * P.ny));
    const double W = wc_at<DIM>(P, g, jac4, v, x, y, z);
    const double ma = __ldg(Xa + i) * (1.0 - __ldg(Xa + i));
    double div = 0.0;
#pragma unroll
    for (int J = 0; J < DIM; ++J)
#pragma unroll
      for (int s = -1; s <= 1; s += 2) {
        int dx, dy, dz;
        step3<DIM>(J, s, dx, dy, dz);
        if (!g.inside(x + dx, y + dy, z + dz)) continue;
        const double cq = __ldg(Xa + g.id(x + dx, y + dy, z + dz));
        div += (ma + cq * (1.0 - cq)) * (wc_at<DIM>(P, g, jac4, v, x + dx, y + dy, z + dz) - W);
      }
    const double vc = __ldg(v + i), ve = __ldg(v + N + i);
    out[i] = vc * P.inv_dt - 0.5 * P.kappa * P.inv_h2 * div;
    out[N + i] = ve * P.inv_dt + __ldg(jac4 + 2 * N + i) * vc + __ldg(jac4 + 3 * N + i) * ve -
                 1.5 * P.gamma_eta * P.inv_h2 * lap<DIM>(g, v + N, x, y, z);
    // u rows: the same operator on v_u with the eigenstrain -eps0 v_c (the constant cbar0 drops out)
#pragma unroll
    for (int I = 0; I < DIM; ++I) out[(2 + I) * N + i] = urow<DIM>(P, g, v + 2 * N, v, 0.0, I, x, y, z);
  }
}

// ---- gauge (R38): translations (mean of every u component) and the discrete rotations, one per pair of
// even extents: r_I = s(x_J) - mean, r_J = -(s(x_I) - mean), s(k) = floor((k+1)/2); the modes are mutually
// orthogonal after the mean subtraction, so the projection is a sum of independent ones.
__device__ __forceinline__ double stair(int k) { return (double)((k + 1) >> 1); }

template <int DIM>
__global__ void k_gauge_sums_neumann(DevParams P, const double* __restrict__ X, int rotmask, double smean0,
                                     double smean1, double smean2, double* __restrict__ part) {
  constexpr int NV = DIM + 3;
  __shared__ double sred[NV][kRedThreads / 32];
  double v[NV];
#pragma unroll
  for (int k = 0; k < NV; ++k) v[k] = 0.0;
  const long long N = P.N;
  const double sm[3] = {smean0, smean1, smean2};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int co[3] = {(int)(i % P.nx), (int)((i / P.nx) % P.ny), (int)(i / ((long long)P.nx * P.ny))};
    double u[3] = {0, 0, 0};
#pragma unroll
    for (int I = 0; I < DIM; ++I) { u[I] = X[(2 + I) * N + i]; v[I] += u[I]; }
    int q = 0;
#pragma unroll
    for (int I = 0; I < DIM; ++I)
#pragma unroll
      for (int J = I + 1; J < DIM; ++J, ++q)
        if (rotmask & (1 << q)) v[DIM + q] += u[I] * (stair(co[J]) - sm[J]) - u[J] * (stair(co[I]) - sm[I]);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double a = v[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) a += __shfl_down_sync(0xffffffffu, a, o);
    if (lane == 0) sred[k][wid] = a;
  }
  __syncthreads();
  if (threadIdx.x < NV) {
    double a = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) a += sred[threadIdx.x][w];
    part[blockIdx.x * NV + threadIdx.x] = a;
  }
}

template <int DIM>
__global__ void k_gauge_apply_neumann(DevParams P, double* __restrict__ X, int rotmask, double smean0, double smean1,
                                      double smean2, const double* __restrict__ sums, double inv_n, double rn0,
                                      double rn1, double rn2) {
  const long long N = P.N;
  const double sm[3] = {smean0, smean1, smean2};
  const double rn[3] = {rn0, rn1, rn2};       // 1 / |r_q|^2
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int co[3] = {(int)(i % P.nx), (int)((i / P.nx) % P.ny), (int)(i / ((long long)P.nx * P.ny))};
    double du[3] = {0, 0, 0};
#pragma unroll
    for (int I = 0; I < DIM; ++I) du[I] = sums[I] * inv_n;
    int q = 0;
#pragma unroll
    for (int I = 0; I < DIM; ++I)
#pragma unroll
      for (int J = I + 1; J < DIM; ++J, ++q)
        if (rotmask & (1 << q)) {
          const double a = sums[DIM + q] * rn[q];
          du[I] += a * (stair(co[J]) - sm[J]);
          du[J] -= a * (stair(co[I]) - sm[I]);
        }
#pragma unroll
    for (int I = 0; I < DIM; ++I) X[(2 + I) * N + i] -= du[I];
  }
}

__global__ void k_reduce_parts(const double* __restrict__ part, int nb, int nv, double* __restrict__ out) {
  if ((int)threadIdx.x < nv) {
    double a = 0.0;
    for (int b = 0; b < nb; ++b) a += part[b * nv + threadIdx.x];      // fixed order
    out[threadIdx.x] = a;
  }
}

}  // namespace nm

void launch_residual_neumann(const DevParams& P, const double* Xa, const double* Xb, const double* Ta, double* F,
                             cudaStream_t s) {
  const int blocks = (int)std::min<long long>((P.N + 127) / 128, 148 * 16);
  if (P.dim == 2) nm::k_residual_neumann<2><<<blocks, 128, 0, s>>>(P, Xa, Xb, Ta, F);
  else nm::k_residual_neumann<3><<<blocks, 128, 0, s>>>(P, Xa, Xb, Ta, F);
}

void launch_jv_neumann(const DevParams& P, const double* Xa, const double* jac4, const double* v, double* out,
                       cudaStream_t s) {
  const int blocks = (int)std::min<long long>((P.N + 127) / 128, 148 * 16);
  if (P.dim == 2) nm::k_jv_neumann<2><<<blocks, 128, 0, s>>>(P, Xa, jac4, v, out);
  else nm::k_jv_neumann<3><<<blocks, 128, 0, s>>>(P, Xa, jac4, v, out);
}

// Gauge of a Neumann state: sums (d translations + up to 3 rotation products) -> out, then the projection.
void launch_gauge_neumann(const DevParams& P, double* X, double* part, double* out, cudaStream_t s) {
  const int d = P.dim;
  const int n[3] = {P.nx, P.ny, P.nz};
  double smean[3] = {0, 0, 0}, svar[3] = {0, 0, 0};
  for (int J = 0; J < d; ++J) {       // mean and variance of the staircase along axis J (host, exact sums)
    double a = 0.0, b = 0.0;
    for (int k = 0; k < n[J]; ++k) a += (double)((k + 1) >> 1);
    a /= n[J];
    for (int k = 0; k < n[J]; ++k) { const double t = (double)((k + 1) >> 1) - a; b += t * t; }
    smean[J] = a;
    svar[J] = b / n[J];
  }
  int rotmask = 0, q = 0;
  double rn[3] = {0, 0, 0};
  const double Nd = (double)P.N;
  for (int I = 0; I < d; ++I)
    for (int J = I + 1; J < d; ++J, ++q)
      if (n[I] % 2 == 0 && n[J] % 2 == 0) {
        rotmask |= 1 << q;
        rn[q] = 1.0 / (Nd * (svar[J] + svar[I]));    // |r|^2 = N (var_J + var_I)
      }
  const int nv = d + 3;
  if (d == 2) nm::k_gauge_sums_neumann<2><<<kRedBlocks, kRedThreads, 0, s>>>(P, X, rotmask, smean[0], smean[1], smean[2], part);
  else nm::k_gauge_sums_neumann<3><<<kRedBlocks, kRedThreads, 0, s>>>(P, X, rotmask, smean[0], smean[1], smean[2], part);
  nm::k_reduce_parts<<<1, 32, 0, s>>>(part, kRedBlocks, nv, out);
  const int blocks = (int)std::min<long long>((P.N + 255) / 256, 148 * 16);
  if (d == 2)
    nm::k_gauge_apply_neumann<2><<<blocks, 256, 0, s>>>(P, X, rotmask, smean[0], smean[1], smean[2], out, 1.0 / Nd, rn[0],
                                                         rn[1], rn[2]);
  else
    nm::k_gauge_apply_neumann<3><<<blocks, 256, 0, s>>>(P, X, rotmask, smean[0], smean[1], smean[2], out, 1.0 / Nd, rn[0],
                                                         rn[1], rn[2]);
}

}  // namespace nks
