// GMRES vector kernels (K7): the two passes of a DCGS2 Arnoldi step (one fused multi-dot reduction,
// one fused update), linear combination, axpy.  All dot products of one Arnoldi step are reduced in
// fixed order (deterministic) and read by the host once per iteration.
#include "nks_internal.cuh"

namespace nks {

struct Coefs {
  double c[64];
};

// ------------------------------------------------------------------------------------------------
// Delayed classical Gram-Schmidt with one reduction per Arnoldi step (DCGS2; the reorthogonalisation of
// the candidate u is delayed by one step and merged with the next step's projection -- Swirydowicz et al.,
// "Low synchronization Gram-Schmidt and GMRES algorithms", 2020).  Step j holds the orthonormal
// v_0..v_{j-1}, the once-orthogonalised candidate u (slot j) and w = A M^-1 u (slot j+1):
//   one reduction:  a = V^T u, b = V^T w, alpha = u.u, beta = u.w                  (k_dcgs_dot)
//   r = sqrt(alpha - |a|^2),  gamma = (beta - a.b)/r
//   v_j    = (u - V a)/r                                (u reorthogonalised and normalised, slot j)
//   u_next = (w - V b - gamma v_j)/r                    (the next candidate, slot j+1; k_dcgs_update)
// and the Arnoldi columns (host): column j-1 = h_prev + a with subdiagonal r; the tentative column j is
// h' = ([b; gamma] - H a)/r, so that A M^-1 v_j = V h' + u_next.  Both passes read the basis once.
// Output layout of the reduction: out[0..31] = a, out[32..63] = b, out[64] = alpha, out[65] = beta.
constexpr int kDOut = 66;

__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// Row-streaming reduction: block (bx, g) walks rows of the vectors grid-stride (16-byte loads when VW = 2) and
// accumulates, per thread, the dots of u and w with the CG basis columns of group g (and, group 0, u.u and
// u.w) -- every column and u, w read in long coalesced runs, u and w once per group (L2 hits after the first).
// The partials go to part[bx][kDOut] (each group writes its own entries); k_dcgs_final sums every entry over
// bx with a fixed tree (deterministic), one block per entry.
template <int CG, int VW>
__global__ void __launch_bounds__(256) k_dcgs_dot(long long n, int nk, const double* __restrict__ V, long long ld,
                                                const double* __restrict__ u, const double* __restrict__ w,
                                                double* __restrict__ part) {
  constexpr int NA = 2 * CG + 2;
  __shared__ double sred[8][NA];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int g = blockIdx.y, k0 = g * CG;
  double acc[NA];
#pragma unroll
  for (int q = 0; q < NA; ++q) acc[q] = 0.0;
  const long long m = n / VW;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    double ux, uy = 0.0, wx, wy = 0.0;
    if (VW == 2) {
      const double2 uv = __ldg(reinterpret_cast<const double2*>(u) + t), wv = __ldg(reinterpret_cast<const double2*>(w) + t);
      ux = uv.x; uy = uv.y; wx = wv.x; wy = wv.y;
    } else {
      ux = __ldg(u + t); wx = __ldg(w + t);
    }
#pragma unroll
    for (int c = 0; c < CG; ++c)
      if (k0 + c < nk) {
        double vx, vy = 0.0;
        if (VW == 2) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + (long long)(k0 + c) * ld) + t);
          vx = v.x; vy = v.y;
        } else {
          vx = __ldg(V + (long long)(k0 + c) * ld + t);
        }
        acc[c] = fma(vx, ux, fma(vy, uy, acc[c]));
        acc[CG + c] = fma(vx, wx, fma(vy, wy, acc[CG + c]));
      }
    if (g == 0) {
      acc[2 * CG] = fma(ux, ux, fma(uy, uy, acc[2 * CG]));
      acc[2 * CG + 1] = fma(ux, wx, fma(uy, wy, acc[2 * CG + 1]));
    }
  }
#pragma unroll
  for (int q = 0; q < NA; ++q) {
    double v = acc[q];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) sred[wid][q] = v;
  }
  __syncthreads();
  if (threadIdx.x < NA) {
    const int q = threadIdx.x;
    double v = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) v += sred[k][q];
    double* row = part + (long long)blockIdx.x * kDOut;
    if (q < CG) { if (k0 + q < 32) row[k0 + q] = v; }
    else if (q < 2 * CG) { if (k0 + q - CG < 32) row[32 + k0 + q - CG] = v; }
    else if (g == 0) row[64 + q - 2 * CG] = v;
  }
}

// Final stage of k_dcgs_dot: one block per output entry sums the nb block partials with a fixed tree
// (deterministic); entries the step does not use are written as 0.
__global__ void __launch_bounds__(256) k_dcgs_final(const double* __restrict__ part, int nb, int nk,
                                                  double* __restrict__ out) {
  __shared__ double s[256];
  const int e = blockIdx.x;
  const bool used = (e < 32 && e < nk) || (e >= 32 && e < 64 && e - 32 < nk) || e >= 64;
  double a = 0.0;
  if (used)
    for (int b = threadIdx.x; b < nb; b += blockDim.x) a += part[(long long)b * kDOut + e];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[e] = s[0];
}

// r and gamma from the reduced values, in the host's order (so the host replays identical doubles).
__device__ __forceinline__ void dcgs_scalars(const double* __restrict__ hv, int nk, double& inv_r, double& gamma_r) {
  double aa = 0.0, ab = 0.0;
  for (int k = 0; k < nk; ++k) {
    aa += hv[k] * hv[k];
    ab += hv[k] * hv[32 + k];
  }
  const double r = sqrt(fmax(hv[64] - aa, 0.0));
  inv_r = r > 1e-300 ? 1.0 / r : 0.0;
  gamma_r = (hv[65] - ab) * inv_r;          // gamma = (beta - a.b)/r
}

// slot j <- v_j = (u - V a)/r ; slot j+1 <- (w - V b - gamma v_j)/r   (u = slot j, w = slot j+1)
template <int NK, int VW>
__global__ void __launch_bounds__(256) k_dcgs_update(long long n, int nk, double* __restrict__ V, long long ld,
                                                   const double* __restrict__ hv) {
  __shared__ double sa[NK], sb[NK];
  __shared__ double s_inv_r, s_gamma;
  for (int k = threadIdx.x; k < NK; k += blockDim.x) {
    sa[k] = k < nk ? hv[k] : 0.0;
    sb[k] = k < nk ? hv[32 + k] : 0.0;
  }
  if (threadIdx.x == 0) {
    double ir, g;
    dcgs_scalars(hv, nk, ir, g);
    s_inv_r = ir;
    s_gamma = g;
  }
  __syncthreads();
  const double ir = s_inv_r, g = s_gamma;
  double* u = V + (long long)nk * ld;
  double* w = u + ld;
  const long long m = n / VW;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    if (VW == 2) {
      double2 uv = reinterpret_cast<double2*>(u)[t], wv = reinterpret_cast<double2*>(w)[t];
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k < nk) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
          uv.x = fma(-sa[k], v.x, uv.x);
          uv.y = fma(-sa[k], v.y, uv.y);
          wv.x = fma(-sb[k], v.x, wv.x);
          wv.y = fma(-sb[k], v.y, wv.y);
        }
      uv.x *= ir;
      uv.y *= ir;
      wv.x = (wv.x - g * uv.x) * ir;
      wv.y = (wv.y - g * uv.y) * ir;
      reinterpret_cast<double2*>(u)[t] = uv;
      reinterpret_cast<double2*>(w)[t] = wv;
    } else {
      double ui = u[t], wi = w[t];
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k < nk) {
          const double v = __ldg(V + k * ld + t);
          ui = fma(-sa[k], v, ui);
          wi = fma(-sb[k], v, wi);
        }
      ui *= ir;
      u[t] = ui;
      w[t] = (wi - g * ui) * ir;
    }
  }
}

// Plain dot product (fixed-order two-stage): part[block] = block sums, then one block sums them in order.
__global__ void __launch_bounds__(256) k_dot_part(long long n, const double* __restrict__ a, const double* __restrict__ b,
                                                double* __restrict__ part) {
  __shared__ double sred[8];
  double v = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    v = fma(a[i], b[i], v);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) sred[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int k = 0; k < 8; ++k) t += sred[k];
    part[blockIdx.x] = t;
  }
}

__global__ void k_dot_final(const double* __restrict__ part, int nb, double* __restrict__ out) {
  __shared__ double s[256];
  double a = 0.0;
  for (int k = threadIdx.x; k < nb; k += blockDim.x) a += part[k];
  s[threadIdx.x] = a;
  __syncthreads();
  for (int w = blockDim.x / 2; w > 0; w >>= 1) {
    if ((int)threadIdx.x < w) s[threadIdx.x] += s[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) out[0] = s[0];
}

// out = sum_k y[k] V_k
__global__ void k_lincomb(long long n, int nk, const double* __restrict__ V, long long ld, Coefs y,
                          double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int k = 0; k < nk; ++k) s = fma(y.c[k], __ldg(V + k * ld + i), s);
    out[i] = s;
  }
}

// y = a x + b y
__global__ void k_axpby(long long n, double a, const double* x, double b, double* y) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    y[i] = b == 0.0 ? a * x[i] : fma(a, x[i], b * y[i]);
}

// z = x + a y
__global__ void k_xpay(long long n, const double* __restrict__ x, double a, const double* __restrict__ y,
                       double* __restrict__ z) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    z[i] = fma(a, y[i], x[i]);
}

static int vec_blocks(long long n) { return (int)std::min<long long>((n + 255) / 256, 148 * 8); }

#define NK_DISPATCH(nk, KERNEL, ...)                           \
  do {                                                         \
    if ((nk) <= 8) KERNEL<8>__VA_ARGS__;                       \
    else if ((nk) <= 16) KERNEL<16>__VA_ARGS__;                \
    else if ((nk) <= 32) KERNEL<32>__VA_ARGS__;                \
    else KERNEL<64>__VA_ARGS__;                                \
  } while (0)

static bool vec2(long long n, long long ld) { return (n % 2) == 0 && (ld % 2) == 0; }

// One reduction of step nk (nk <= 31 basis columns before the candidate): out[] as documented above.
static void dcgs_dot(long long n, int nk, const double* V, long long ld, const double* u, const double* w, double* part,
                     double* out, unsigned* counter, cudaStream_t s) {
  const bool v2 = vec2(n, ld);
  const long long m = v2 ? n / 2 : n;
  // 4 columns per group: 10 accumulators and 6 loads in flight per thread keep the registers (and so the
  // occupancy) of a streaming kernel; u and w are re-read per group from L2
  const int ng = std::max(1, (nk + 3) / 4);
  const int nbx = (int)std::min<long long>((m + 255) / 256, std::max(4 * 148 / ng, 74));   // part: kRedBlocks rows
  const dim3 grid(nbx, ng);
  if (v2) k_dcgs_dot<4, 2><<<grid, 256, 0, s>>>(n, nk, V, ld, u, w, part);
  else k_dcgs_dot<4, 1><<<grid, 256, 0, s>>>(n, nk, V, ld, u, w, part);
  k_dcgs_final<<<kDOut, 256, 0, s>>>(part, nbx, nk, out);
  (void)counter;
}

void launch_dcgs_dot(long long n, int nk, const double* V, long long ld, double* part, double* out, unsigned* counter,
                     cudaStream_t s) {
  const double* u = V + (long long)nk * ld;
  dcgs_dot(n, nk, V, ld, u, u + ld, part, out, counter, s);
}

// The candidate-only reduction that closes a restart cycle (there is no w = A M^-1 u_m): the same kernel
// with w aliased to u; the host uses only a and alpha of it.
void launch_dcgs_dot_u(long long n, int nk, const double* V, long long ld, double* part, double* out, unsigned* counter,
                       cudaStream_t s) {
  const double* u = V + (long long)nk * ld;
  dcgs_dot(n, nk, V, ld, u, u, part, out, counter, s);
}

void launch_dcgs_update(long long n, int nk, double* V, long long ld, const double* hv, cudaStream_t s) {
  if (vec2(n, ld)) {
    const int nb = vec_blocks(n / 2);
    if (nk <= 8) k_dcgs_update<8, 2><<<nb, 256, 0, s>>>(n, nk, V, ld, hv);
    else if (nk <= 16) k_dcgs_update<16, 2><<<nb, 256, 0, s>>>(n, nk, V, ld, hv);
    else k_dcgs_update<32, 2><<<nb, 256, 0, s>>>(n, nk, V, ld, hv);
  } else {
    const int nb = vec_blocks(n);
    if (nk <= 8) k_dcgs_update<8, 1><<<nb, 256, 0, s>>>(n, nk, V, ld, hv);
    else if (nk <= 16) k_dcgs_update<16, 1><<<nb, 256, 0, s>>>(n, nk, V, ld, hv);
    else k_dcgs_update<32, 1><<<nb, 256, 0, s>>>(n, nk, V, ld, hv);
  }
}

void launch_lincomb(long long n, int nk, const double* V, long long ld, const double* y, double* out, cudaStream_t s) {
  Coefs c;
  for (int k = 0; k < nk && k < 64; ++k) c.c[k] = y[k];
  k_lincomb<<<vec_blocks(n), 256, 0, s>>>(n, nk, V, ld, c, out);
}

void launch_dot(long long n, const double* a, const double* b, double* part, double* out, cudaStream_t s) {
  const int nb = (int)std::min<long long>((n + 255) / 256, kRedBlocks);
  k_dot_part<<<nb, 256, 0, s>>>(n, a, b, part);
  k_dot_final<<<1, 256, 0, s>>>(part, nb, out);
}

void launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t s) {
  k_axpby<<<vec_blocks(n), 256, 0, s>>>(n, a, x, b, y);
}

void launch_xpay(long long n, const double* x, double a, const double* y, double* z, cudaStream_t s) {
  k_xpay<<<vec_blocks(n), 256, 0, s>>>(n, x, a, y, z);
}

}  // namespace nks
