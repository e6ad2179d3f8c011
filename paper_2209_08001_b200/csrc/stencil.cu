// Pointwise kernels of the NKS step: level-n prep (K3), pointwise Jacobian cache, energy/mass (K8),
// gauge (K9), admissibility + norm, fixed-order reductions.  (The residual F (K1) and J.v (K2) are the
// z-marching tiled kernels of stencil_tiled.cu.)
//
// Layout: SoA fp64, field f of a state vector at base + f*N, point index (z*ny + y)*nx + x,
// periodic wrap in the index arithmetic.
#include "model.cuh"
#include "nks_internal.cuh"

namespace nks {

__device__ __forceinline__ int wrapc(int v, int n) { return v < 0 ? v + n : (v >= n ? v - n : v); }
__device__ __forceinline__ int mirc(int v, int n) { return v < 0 ? -1 - v : (v >= n ? 2 * n - 1 - v : v); }

// Index of a (possibly ghost) neighbour: periodic wrap, or the Neumann mirror ghost (bc = 1, reading R38),
// which makes D^ / D+ / D- / the Laplacian of the level prep and the energy take the boundary closure.
struct Geo {
  int nx, ny, nz;
  long long N;
  int bc;
  __device__ __forceinline__ long long id(int x, int y, int z) const {
    if (bc) return ((long long)mirc(z, nz) * ny + mirc(y, ny)) * nx + mirc(x, nx);
    return ((long long)wrapc(z, nz) * ny + wrapc(y, ny)) * nx + wrapc(x, nx);
  }
};

template <int DIM>
__device__ __forceinline__ long long nb(const Geo& g, int x, int y, int z, int J, int s) {
  return g.id(x + (J == 0 ? s : 0), y + (J == 1 ? s : 0), z + (J == 2 ? s : 0));
}

// sum_J D^_J u_J at (x,y,z); u = base of u_1 (field stride N).
template <int DIM>
__device__ __forceinline__ double div_hat(const Geo& g, const double* __restrict__ u, int x, int y, int z, double inv_2h) {
  double acc = 0.0;
#pragma unroll
  for (int J = 0; J < DIM; ++J) {
    const double* uj = u + (long long)J * g.N;
    acc += __ldg(uj + nb<DIM>(g, x, y, z, J, 1)) - __ldg(uj + nb<DIM>(g, x, y, z, J, -1));
  }
  return acc * inv_2h;
}

// -------------------------------------------------------------------------------------- K3
template <int DIM>
__global__ void k_level_prep(DevParams P, const double* __restrict__ X, double* __restrict__ T) {
  const Geo g{P.nx, P.ny, P.nz, P.N, P.bc};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx);
    const int y = (int)((i / P.nx) % P.ny);
    const int z = (int)(i / ((long long)P.nx * P.ny));
    const double c = X[i];
    T[i] = P.K * (div_hat<DIM>(g, X + 2 * P.N, x, y, z, P.inv_2h) - DIM * P.eps0 * (c - P.cbar0));
  }
}

// Pointwise partials a11, a12, a21, a22 (cached per Newton iterate; used by J.v and assembly).
__global__ void k_pointwise_jac(DevParams P, const double* __restrict__ Xa, const double* __restrict__ Xb,
                                double* __restrict__ jac4) {
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    double a11, a12, a21, a22;
    pointwise_dG(P, Xa[i], Xb[i], Xa[N + i], Xb[N + i], a11, a12, a21, a22);
    jac4[i] = a11;
    jac4[N + i] = a12;
    jac4[2 * N + i] = a21;
    jac4[3 * N + i] = a22;
  }
}

// -------------------------------------------------------------------------------------- reductions
// Block reduction of NV doubles; result in thread 0's vals.
template <int NV>
__device__ __forceinline__ void block_reduce(double (&vals)[NV]) {
  __shared__ double sred[NV][kRedThreads / 32];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double v = vals[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sred[k][wid] = v;
  }
  __syncthreads();
  if (wid == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double v = lane < (int)(blockDim.x >> 5) ? sred[k][lane] : 0.0;
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
      vals[k] = v;
    }
  }
  __syncthreads();
}

// Second stage: out[k] = sum over nb partial rows (fixed order) -- one block of kRedThreads.
__global__ void k_reduce_final(const double* __restrict__ part, int nb, int nv, double* __restrict__ out) {
  __shared__ double s[kRedThreads];
  for (int k = 0; k < nv; ++k) {
    double acc = 0.0;
    for (int b = threadIdx.x; b < nb; b += blockDim.x) acc += part[(long long)b * nv + k];
    s[threadIdx.x] = acc;
    __syncthreads();
    for (int w = blockDim.x / 2; w > 0; w >>= 1) {
      if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
      __syncthreads();
    }
    if (threadIdx.x == 0) out[k] = s[0];
    __syncthreads();
  }
}

// ||F||^2 over nvec entries + count of inadmissible points of X (c, p, q in (0,1), finite).
__global__ void k_norm_admissible(long long N, int nf, const double* __restrict__ F, const double* __restrict__ X,
                                  double* __restrict__ part) {
  double v[2] = {0.0, 0.0};
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long nvec = N * nf;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < nvec; i += stride) {
    const double f = F[i];
    v[0] += f * f;
  }
  if (X != nullptr) {
    for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += stride) {
      const double c = X[i], e = X[N + i];
      const double p = c * e, q = c * (4.0 - 3.0 * e);
      bool ok = c > 0.0 && c < 1.0 && p > 0.0 && p < 1.0 && q > 0.0 && q < 1.0;
      for (int f = 2; f < nf; ++f) ok = ok && isfinite(X[f * N + i]);
      if (!ok) v[1] += 1.0;
    }
  }
  block_reduce<2>(v);
  if (threadIdx.x == 0) {
    part[blockIdx.x * 2] = v[0];
    part[blockIdx.x * 2 + 1] = v[1];
  }
}

// Energy parts E1..E4 and sum c.
template <int DIM>
__global__ void k_energy(DevParams P, const double* __restrict__ X, double* __restrict__ part) {
  const Geo g{P.nx, P.ny, P.nz, P.N, P.bc};
  const long long N = P.N;
  const double* c_ = X;
  const double* e_ = X + N;
  const double* u_ = X + 2 * N;
  double v[5] = {0, 0, 0, 0, 0};
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx);
    const int y = (int)((i / P.nx) % P.ny);
    const int z = (int)(i / ((long long)P.nx * P.ny));
    if (z < P.zg || z >= P.nz - P.zg) continue;       // slab: own planes only
    if (y < P.yg || y >= P.ny - P.yg) continue;       // pencil: own rows only
    const double c = c_[i], eta = e_[i];
    double e1, e2;
    local_energy(P, c, eta, e1, e2);
    // elastic strain: eps_IJ = (D^_J u_I + D^_I u_J)/2
    double du[3][3];
#pragma unroll
    for (int I = 0; I < DIM; ++I)
#pragma unroll
      for (int J = 0; J < DIM; ++J)
        du[I][J] = (__ldg(u_ + I * N + nb<DIM>(g, x, y, z, J, 1)) - __ldg(u_ + I * N + nb<DIM>(g, x, y, z, J, -1))) * P.inv_2h;
    const double e0 = P.eps0 * (c - P.cbar0);
    double tr = 0.0, sq = 0.0, off = 0.0;
#pragma unroll
    for (int I = 0; I < DIM; ++I) {
      const double eII = du[I][I] - e0;
      tr += eII;
      sq += eII * eII;
#pragma unroll
      for (int J = I + 1; J < DIM; ++J) {
        const double eIJ = 0.5 * (du[I][J] + du[J][I]);
        off += eIJ * eIJ;
      }
    }
    const double e3 = 0.5 * P.Ls * (P.C12 * tr * tr + (P.C11 - P.C12) * sq + 4.0 * P.C44 * off);
    double gc2 = 0.0, ge2 = 0.0;
#pragma unroll
    for (int J = 0; J < DIM; ++J) {
      const double cp = __ldg(c_ + nb<DIM>(g, x, y, z, J, 1)), cm = __ldg(c_ + nb<DIM>(g, x, y, z, J, -1));
      const double ep = __ldg(e_ + nb<DIM>(g, x, y, z, J, 1)), em = __ldg(e_ + nb<DIM>(g, x, y, z, J, -1));
      gc2 += (cp - c) * (cp - c) + (c - cm) * (c - cm);
      ge2 += (ep - eta) * (ep - eta) + (eta - em) * (eta - em);
    }
    const double e4 = (0.25 * P.gamma_c * gc2 + 0.75 * P.gamma_eta * ge2) * P.inv_h2;
    v[0] += e1; v[1] += e2; v[2] += e3; v[3] += e4; v[4] += c;
  }
  block_reduce<5>(v);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < 5; ++k) part[blockIdx.x * 5 + k] = v[k];
}

// Gauge: sums of u_I over each parity class of the even axes (class bit j = parity along even axis j).
template <int DIM>
__global__ void k_gauge_sums(DevParams P, const double* __restrict__ X, int evenmask, double* __restrict__ part) {
  constexpr int NC = 1 << DIM;
  double v[DIM * NC];
#pragma unroll
  for (int k = 0; k < DIM * NC; ++k) v[k] = 0.0;
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx);
    const int y = (int)((i / P.nx) % P.ny);
    const int z = (int)(i / ((long long)P.nx * P.ny));
    if (z < P.zg || z >= P.nz - P.zg) continue;       // slab: own planes only
    if (y < P.yg || y >= P.ny - P.yg) continue;       // pencil: own rows only
    int cls = 0, bit = 0;
    const int co[3] = {x, y - P.yg + P.yoff, z - P.zg + P.zoff};   // global coordinates (parity classes)
#pragma unroll
    for (int j = 0; j < DIM; ++j)
      if (evenmask & (1 << j)) { cls |= (co[j] & 1) << bit; ++bit; }
#pragma unroll
    for (int I = 0; I < DIM; ++I) {
      const double u = X[(2 + I) * N + i];
#pragma unroll
      for (int k = 0; k < NC; ++k) v[I * NC + k] += (k == cls) ? u : 0.0;
    }
  }
  block_reduce<DIM * NC>(v);
  if (threadIdx.x == 0)
#pragma unroll
    for (int k = 0; k < DIM * NC; ++k) part[blockIdx.x * (DIM * NC) + k] = v[k];
}

template <int DIM>
__global__ void k_gauge_apply(DevParams P, double* __restrict__ X, int evenmask, const double* __restrict__ sums,
                              double inv_count) {
  constexpr int NC = 1 << DIM;
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx);
    const int y = (int)((i / P.nx) % P.ny);
    const int z = (int)(i / ((long long)P.nx * P.ny));
    int cls = 0, bit = 0;
    const int co[3] = {x, y - P.yg + P.yoff, z - P.zg + P.zoff};   // ghost planes / rows get their (global) class too
#pragma unroll
    for (int j = 0; j < DIM; ++j)
      if (evenmask & (1 << j)) { cls |= (co[j] & 1) << bit; ++bit; }
#pragma unroll
    for (int I = 0; I < DIM; ++I) X[(2 + I) * N + i] -= sums[I * NC + cls] * inv_count;
  }
}

// -------------------------------------------------------------------------------------- host launchers
void launch_level_prep(const DevParams& P, const double* X, double* T, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((P.N + 255) / 256, 148 * 16);
  if (P.dim == 2) k_level_prep<2><<<blocks, 256, 0, s>>>(P, X, T);
  else k_level_prep<3><<<blocks, 256, 0, s>>>(P, X, T);
}

void launch_pointwise_jac(const DevParams& P, const double* Xa, const double* Xb, double* jac4, cudaStream_t s) {
  const int blocks = (int)std::min<long long>((P.N + 255) / 256, 148 * 16);
  k_pointwise_jac<<<blocks, 256, 0, s>>>(P, Xa, Xb, jac4);
}

void launch_norm_admissible(long long N, int nf, const double* F, const double* X, double* part, double* out,
                            cudaStream_t s) {
  k_norm_admissible<<<kRedBlocks, kRedThreads, 0, s>>>(N, nf, F, X, part);
  k_reduce_final<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, 2, out);
}

void launch_energy(const DevParams& P, const double* X, double* part, double* out, cudaStream_t s) {
  if (P.dim == 2) k_energy<2><<<kRedBlocks, kRedThreads, 0, s>>>(P, X, part);
  else k_energy<3><<<kRedBlocks, kRedThreads, 0, s>>>(P, X, part);
  k_reduce_final<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, 5, out);
}

int gauge_classes(const DevParams& P, int& evenmask) {
  evenmask = 0;
  int nbits = 0;
  const int n[3] = {P.nx, P.nyg > 0 ? P.nyg : P.ny, P.nzg > 0 ? P.nzg : P.nz};
  for (int j = 0; j < P.dim; ++j)
    if (n[j] % 2 == 0) { evenmask |= 1 << j; ++nbits; }
  return 1 << nbits;
}

// Gauge in two halves so that a sharded state can allreduce the class sums in between.
int launch_gauge_sums(const DevParams& P, const double* X, double* part, double* out, cudaStream_t s) {
  int evenmask;
  const int ncls = gauge_classes(P, evenmask);
  if (P.dim == 2) {
    k_gauge_sums<2><<<kRedBlocks, kRedThreads, 0, s>>>(P, X, evenmask, part);
    k_reduce_final<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, 2 * 4, out);
  } else {
    k_gauge_sums<3><<<kRedBlocks, kRedThreads, 0, s>>>(P, X, evenmask, part);
    k_reduce_final<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, 3 * 8, out);
  }
  return P.dim * (P.dim == 2 ? 4 : 8);   // number of sums (component x class slots)
  (void)ncls;
}

void launch_gauge_apply(const DevParams& P, double* X, const double* out, cudaStream_t s) {
  int evenmask;
  const int ncls = gauge_classes(P, evenmask);
  const long long nglob = (long long)P.nx * (P.nyg > 0 ? P.nyg : P.ny) * (P.nzg > 0 ? P.nzg : P.nz);
  const double inv_count = (double)ncls / (double)nglob;
  const int blocks = (int)std::min<long long>((P.N + 255) / 256, 148 * 16);
  if (P.dim == 2) k_gauge_apply<2><<<blocks, 256, 0, s>>>(P, X, evenmask, out, inv_count);
  else k_gauge_apply<3><<<blocks, 256, 0, s>>>(P, X, evenmask, out, inv_count);
}

void launch_gauge(const DevParams& P, double* X, double* part, double* out, cudaStream_t s) {
  launch_gauge_sums(P, X, part, out, s);
  launch_gauge_apply(P, X, out, s);
}

// Zero the ghost planes of nf fields (slab states): vectors that enter dot products keep zero ghosts.
__global__ void k_zero_ghosts(long long nxy, int nz, int zg, int nf, long long N, double* __restrict__ v) {
  const long long per = 2LL * zg * nxy;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < per * nf; t += (long long)gridDim.x * blockDim.x) {
    const int f = (int)(t / per);
    const long long r = t % per;
    const long long plane = r / nxy, off = r % nxy;
    const long long z = plane < zg ? plane : (nz - 2 * zg + plane);
    v[f * N + z * nxy + off] = 0.0;
  }
}

// Zero the ghost rows (y) of every plane of nf fields (pencil states).
__global__ void k_zero_ghost_rows(int nx, int ny, int nz, int yg, int nf, long long N, double* __restrict__ v) {
  const long long per = 2LL * yg * nx;                 // ghost cells per plane
  const long long tot = per * nz * nf;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < tot; t += (long long)gridDim.x * blockDim.x) {
    const long long f = t / (per * nz), r = t % (per * nz);
    const long long z = r / per, q = r % per;
    const long long row = q / nx, x = q % nx;
    const long long y = row < yg ? row : (ny - 2 * yg + row);
    v[f * N + (z * ny + y) * nx + x] = 0.0;
  }
}

void launch_zero_ghosts(const DevParams& P, int nf, double* v, cudaStream_t s) {
  if (P.zg <= 0) return;
  const long long nxy = (long long)P.nx * P.ny;
  const long long work = 2LL * P.zg * nxy * nf;
  const int blocks = (int)std::min<long long>((work + 255) / 256, 148 * 8);
  k_zero_ghosts<<<blocks, 256, 0, s>>>(nxy, P.nz, P.zg, nf, P.N, v);
  if (P.yg > 0) {
    const long long w2 = 2LL * P.yg * P.nx * P.nz * nf;
    k_zero_ghost_rows<<<(int)std::min<long long>((w2 + 255) / 256, 148 * 8), 256, 0, s>>>(P.nx, P.ny, P.nz, P.yg, nf, P.N, v);
  }
}

}  // namespace nks
