// GMRES vector kernels (K7): fused multi-dot, fused update + re-orthogonalisation dots, fused
// update + normalise, linear combination, axpy.  Classical Gram-Schmidt with one
// re-orthogonalisation (CGS2), all dot products of one Arnoldi step reduced in fixed order
// (deterministic) and read by the host once per iteration.
#include "nks_internal.cuh"

namespace nks {

struct Coefs {
  double c[64];
};

template <int NV>
__device__ __forceinline__ void block_reduce_k(double (&vals)[NV]) {
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

// part[b][k] = sum_i V_k[i] w[i] (k < nk), part[b][nk] = sum_i w[i]^2.
template <int NK>
__global__ void __launch_bounds__(kRedThreads) k_mdot(long long n, int nk, const double* __restrict__ V, long long ld,
                                                      const double* __restrict__ w, double* __restrict__ part) {
  double acc[NK + 1];
#pragma unroll
  for (int k = 0; k <= NK; ++k) acc[k] = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    const double wi = w[i];
#pragma unroll
    for (int k = 0; k < NK; ++k)
      if (k < nk) acc[k] = fma(__ldg(V + k * ld + i), wi, acc[k]);
    acc[NK] = fma(wi, wi, acc[NK]);
  }
  block_reduce_k<NK + 1>(acc);
  if (threadIdx.x == 0) {
    for (int k = 0; k < nk; ++k) part[blockIdx.x * (nk + 1) + k] = acc[k];
    part[blockIdx.x * (nk + 1) + nk] = acc[NK];
  }
}

// w -= sum_k h[k] V_k (h on device), then part = [V^T w_new, |w_new|^2].
template <int NK>
__global__ void __launch_bounds__(kRedThreads) k_update_dot(long long n, int nk, const double* __restrict__ V, long long ld,
                                                            const double* __restrict__ h, double* __restrict__ w,
                                                            double* __restrict__ part) {
  __shared__ double sh[NK];
  if (threadIdx.x < nk) sh[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  double acc[NK + 1];
#pragma unroll
  for (int k = 0; k <= NK; ++k) acc[k] = 0.0;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double vk[NK];
    double wi = w[i];
#pragma unroll
    for (int k = 0; k < NK; ++k)
      if (k < nk) { vk[k] = __ldg(V + k * ld + i); wi = fma(-sh[k], vk[k], wi); }
    w[i] = wi;
#pragma unroll
    for (int k = 0; k < NK; ++k)
      if (k < nk) acc[k] = fma(vk[k], wi, acc[k]);
    acc[NK] = fma(wi, wi, acc[NK]);
  }
  block_reduce_k<NK + 1>(acc);
  if (threadIdx.x == 0) {
    for (int k = 0; k < nk; ++k) part[blockIdx.x * (nk + 1) + k] = acc[k];
    part[blockIdx.x * (nk + 1) + nk] = acc[NK];
  }
}

// w = (w - sum_k h[k] V_k) * scale
template <int NK>
__global__ void k_update_scale(long long n, int nk, const double* __restrict__ V, long long ld,
                               const double* __restrict__ h, double scale, double* __restrict__ w) {
  __shared__ double sh[NK];
  if (threadIdx.x < nk) sh[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double wi = w[i];
#pragma unroll
    for (int k = 0; k < NK; ++k)
      if (k < nk) wi = fma(-sh[k], __ldg(V + k * ld + i), wi);
    w[i] = wi * scale;
  }
}

// w = (w - sum_k h2[k] V_k) / nrm with nrm = sqrt(max(ww - sum_k h2[k]^2, 0)) computed on the device from
// the re-orthogonalisation dots (h2 = hv[0..nk), ww = hv[nk]) in the same order as the host's copy, so
// the host (one iteration behind) and the device agree on the value and on breakdown (nrm <= 1e-300).
template <int NK, int VW>
__global__ void k_update_scale_dev(long long n, int nk, const double* __restrict__ V, long long ld,
                                   const double* __restrict__ hv, double* __restrict__ w) {
  __shared__ double sh[NK];
  __shared__ double s_scale;
  if (threadIdx.x < nk) sh[threadIdx.x] = hv[threadIdx.x];
  if (threadIdx.x < 32) {            // sum_k h2[k]^2 in the host's order: lane 0 adds the lane partials in order
    double part = 0.0;
    if (threadIdx.x == 0)
      for (int k = 0; k < nk; ++k) part += hv[k] * hv[k];
    if (threadIdx.x == 0) {
      const double nrm = sqrt(fmax(hv[nk] - part, 0.0));
      s_scale = nrm > 1e-300 ? 1.0 / nrm : 0.0;
    }
  }
  __syncthreads();
  const double scale = s_scale;
  const long long m = n / VW;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    if (VW == 2) {
      double2 wi = reinterpret_cast<double2*>(w)[t];
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k < nk) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
          wi.x = fma(-sh[k], v.x, wi.x);
          wi.y = fma(-sh[k], v.y, wi.y);
        }
      wi.x *= scale;
      wi.y *= scale;
      reinterpret_cast<double2*>(w)[t] = wi;
    } else {
      double wi = w[t];
#pragma unroll
      for (int k = 0; k < NK; ++k)
        if (k < nk) wi = fma(-sh[k], __ldg(V + k * ld + t), wi);
      w[t] = wi * scale;
    }
  }
}

// ------------------------------------------------------------------------------------------------
// Register-resident CGS2 passes for nk + 1 <= 32 columns (restart <= 31).  A thread streams rows of
// the basis (grid-stride), keeps the 32 column values of its row and 32 dot accumulators in registers,
// and the warp reduces its 32 accumulators with a butterfly reduce-scatter (31 f64 shuffles: lane l
// ends with the warp sum of column l).  Block partials [block][32]; the last block to finish sums them
// in block order (deterministic) into out[0..32).
template <int OFF>
__device__ __forceinline__ void rs_round(double (&v)[32], int lane) {
  const bool up = (lane & OFF) != 0;
#pragma unroll
  for (int i = 0; i < OFF; ++i) {
    const double lo = v[i], hi = v[i + OFF];
    const double send = up ? lo : hi;
    const double keep = up ? hi : lo;
    v[i] = keep + __shfl_xor_sync(0xffffffffu, send, OFF);
  }
}

__device__ __forceinline__ double warp_reduce_scatter32(double (&v)[32], int lane) {
  rs_round<16>(v, lane);
  rs_round<8>(v, lane);
  rs_round<4>(v, lane);
  rs_round<2>(v, lane);
  rs_round<1>(v, lane);
  return v[0];
}

__device__ __forceinline__ void block_partials_32(double (&acc)[32], double* __restrict__ part,
                                                  double* __restrict__ out, unsigned* __restrict__ counter) {
  __shared__ double sw[kRedThreads / 32][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const double ws = warp_reduce_scatter32(acc, lane);
  sw[wid][lane] = ws;
  __syncthreads();
  if (wid == 0) {
    double b = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) b += sw[k][lane];
    part[blockIdx.x * 32 + lane] = b;
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // last block: column = lane, block range split over warps, then warps combined in order
  double a = 0.0;
  for (int blk = wid; blk < (int)gridDim.x; blk += blockDim.x >> 5) a += part[blk * 32 + lane];
  sw[wid][lane] = a;
  __syncthreads();
  if (wid == 0) {
    double t = 0.0;
    for (int k = 0; k < (int)(blockDim.x >> 5); ++k) t += sw[k][lane];
    out[lane] = t;
    if (lane == 0) *counter = 0u;
  }
}

// out[k] = V_k . w (k < nk), out[nk] = w . w, out[nk+1..31] = 0.  VW = 2: 16-byte loads (n even), which
// doubles the contiguous run per column and warp -- 1D streams over 30 columns reach ~85 % of HBM with
// 16-byte loads against ~60 % with 8-byte ones (tools/cgs_probe.cu).
template <int NK, int VW>
__global__ void __launch_bounds__(kRedThreads, 2) k_cgs_dot(long long n, int nk, const double* __restrict__ V, long long ld,
                                                       const double* __restrict__ w, double* __restrict__ part,
                                                       double* __restrict__ out, unsigned* __restrict__ counter) {
  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
  double ww = 0.0;
  const long long m = n / VW;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    if (VW == 2) {
      const double2 wi = reinterpret_cast<const double2*>(w)[t];
#pragma unroll
      for (int k = 0; k < (NK < 31 ? NK : 31); ++k)
        if (k < nk) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
          acc[k] = fma(v.x, wi.x, fma(v.y, wi.y, acc[k]));
        }
      ww = fma(wi.x, wi.x, fma(wi.y, wi.y, ww));
    } else {
      const double wi = w[t];
#pragma unroll
      for (int k = 0; k < (NK < 31 ? NK : 31); ++k) {
        const double vk = k < nk ? __ldg(V + k * ld + t) : 0.0;
        acc[k] = fma(vk, wi, acc[k]);
      }
      ww = fma(wi, wi, ww);
    }
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = k == nk ? ww : acc[k];
  block_partials_32(acc, part, out, counter);
}

// Column-split variant of k_cgs_dot (16-byte loads, n even): the 8 warps of a block walk the same
// 32-element-pair tiles and warp q owns columns q, q+8, q+16, q+24, so a thread keeps <= 4 accumulators,
// occupancy is high and every column is read in 512-byte runs.  Block sums of each column go to
// part[block][32]; the last block to finish adds them in block order (deterministic).
__device__ __forceinline__ double warp_sum(double v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

template <int NK>
__global__ void __launch_bounds__(256) k_cgs_dot_cs(long long n, int nk, const double* __restrict__ V, long long ld,
                                                  const double* __restrict__ w, double* __restrict__ part,
                                                  double* __restrict__ out, unsigned* __restrict__ counter) {
  constexpr int CPW = NK / 8;
  __shared__ double cs[32];
  __shared__ double sw[8][32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  double acc[CPW];
#pragma unroll
  for (int q = 0; q < CPW; ++q) acc[q] = 0.0;
  double ww = 0.0;
  const long long m = n / 2;
  const double2* w2 = reinterpret_cast<const double2*>(w);
  for (long long t = blockIdx.x * 32LL + lane; t < m; t += (long long)gridDim.x * 32) {
    const double2 wv = w2[t];
#pragma unroll
    for (int q = 0; q < CPW; ++q) {
      const int k = wid + 8 * q;
      if (k < nk) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
        acc[q] = fma(v.x, wv.x, fma(v.y, wv.y, acc[q]));
      }
    }
    if (wid == 0) ww = fma(wv.x, wv.x, fma(wv.y, wv.y, ww));
  }
  if (threadIdx.x < 32) cs[threadIdx.x] = 0.0;
  __syncthreads();
#pragma unroll
  for (int q = 0; q < CPW; ++q) {
    const int k = wid + 8 * q;
    const double v = warp_sum(acc[q]);
    if (lane == 0 && k < nk) cs[k] = v;
  }
  if (wid == 0) {
    const double v = warp_sum(ww);
    if (lane == 0) cs[nk] = v;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    part[blockIdx.x * 32 + threadIdx.x] = cs[threadIdx.x];
    __threadfence();
  }
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(counter, 1u) == gridDim.x - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  double a = 0.0;
  for (int blk = wid; blk < (int)gridDim.x; blk += 8) a += part[blk * 32 + lane];
  sw[wid][lane] = a;
  __syncthreads();
  if (wid == 0) {
    double tsum = 0.0;
#pragma unroll
    for (int k = 0; k < 8; ++k) tsum += sw[k][lane];
    out[lane] = tsum;
    if (lane == 0) *counter = 0u;
  }
}

// w <- w - sum_k h[k] V_k ; out[k] = V_k . w_new (k < nk), out[nk] = w_new . w_new.  The columns are
// read twice (the second pass mostly from L1/L2) so that only the 32 accumulators live in registers.
template <int NK, int VW>
__global__ void __launch_bounds__(kRedThreads, NK <= 16 ? 2 : 1) k_cgs_update_dot(long long n, int nk, const double* __restrict__ V,
                                                                 long long ld, const double* __restrict__ h,
                                                                 double* __restrict__ w, double* __restrict__ part,
                                                                 double* __restrict__ out, unsigned* __restrict__ counter) {
  __shared__ double sh[32];
  if (threadIdx.x < 32) sh[threadIdx.x] = threadIdx.x < nk ? h[threadIdx.x] : 0.0;
  __syncthreads();
  double acc[32];
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = 0.0;
  double ww = 0.0;
  const long long m = n / VW;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    if (VW == 2) {
      double2 wi = reinterpret_cast<double2*>(w)[t];
#pragma unroll
      for (int k = 0; k < (NK < 31 ? NK : 31); ++k)
        if (k < nk) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
          wi.x = fma(-sh[k], v.x, wi.x);
          wi.y = fma(-sh[k], v.y, wi.y);
        }
      reinterpret_cast<double2*>(w)[t] = wi;
#pragma unroll
      for (int k = 0; k < (NK < 31 ? NK : 31); ++k)
        if (k < nk) {
          const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
          acc[k] = fma(v.x, wi.x, fma(v.y, wi.y, acc[k]));
        }
      ww = fma(wi.x, wi.x, fma(wi.y, wi.y, ww));
    } else {
      double wi = w[t];
#pragma unroll
      for (int k = 0; k < (NK < 31 ? NK : 31); ++k)
        if (k < nk) wi = fma(-sh[k], __ldg(V + k * ld + t), wi);
      w[t] = wi;
#pragma unroll
      for (int k = 0; k < (NK < 31 ? NK : 31); ++k)
        if (k < nk) acc[k] = fma(__ldg(V + k * ld + t), wi, acc[k]);
      ww = fma(wi, wi, ww);
    }
  }
#pragma unroll
  for (int k = 0; k < 32; ++k) acc[k] = k == nk ? ww : acc[k];
  block_partials_32(acc, part, out, counter);
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

__global__ void k_reduce_final2(const double* __restrict__ part, int nb, int nv, double* __restrict__ out) {
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

static int vec_blocks(long long n) { return (int)std::min<long long>((n + 255) / 256, 148 * 8); }

#define NK_DISPATCH(nk, KERNEL, ...)                           \
  do {                                                         \
    if ((nk) <= 8) KERNEL<8>__VA_ARGS__;                       \
    else if ((nk) <= 16) KERNEL<16>__VA_ARGS__;                \
    else if ((nk) <= 32) KERNEL<32>__VA_ARGS__;                \
    else KERNEL<64>__VA_ARGS__;                                \
  } while (0)

// h[0..nk) = V^T w, h[nk] = w.w  -> out (device)
void launch_mdot(long long n, int nk, const double* V, long long ld, const double* w, double* part, double* out,
                 cudaStream_t s) {
  NK_DISPATCH(nk, k_mdot, <<<kRedBlocks, kRedThreads, 0, s>>>(n, nk, V, ld, w, part));
  k_reduce_final2<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, nk + 1, out);
}

void launch_update_dot(long long n, int nk, const double* V, long long ld, const double* h, double* w, double* part,
                       double* out, cudaStream_t s) {
  NK_DISPATCH(nk, k_update_dot, <<<kRedBlocks, kRedThreads, 0, s>>>(n, nk, V, ld, h, w, part));
  k_reduce_final2<<<1, kRedThreads, 0, s>>>(part, kRedBlocks, nk + 1, out);
}

void launch_update_scale(long long n, int nk, const double* V, long long ld, const double* h, double scale, double* w,
                         cudaStream_t s) {
  NK_DISPATCH(nk, k_update_scale, <<<vec_blocks(n), 256, 0, s>>>(n, nk, V, ld, h, scale, w));
}

static int cgs_blocks(long long n) { return (int)std::min<long long>((n + kRedThreads - 1) / kRedThreads, 148 * 2); }

// 16-byte columns need an even length and leading dimension (every real grid has an even N)
static bool vec2(long long n, long long ld) { return (n % 2) == 0 && (ld % 2) == 0; }

void launch_cgs_dot(long long n, int nk, const double* V, long long ld, const double* w, double* part, double* out,
                    unsigned* counter, cudaStream_t s) {
  // the unrolled column loop is as long as the template NK (8, 16 or 31 live columns), not always 31
  if (vec2(n, ld)) {
    // column-split kernel; blocks <= kRedBlocks (the partials buffer holds kRedBlocks x 32)
    const int nbc = (int)std::min<long long>((n / 2 + 31) / 32, kRedBlocks);
    // measured at config 2: column split wins up to 15 columns, the register-resident kernel above
    if (nk <= 7) k_cgs_dot_cs<8><<<nbc, 256, 0, s>>>(n, nk, V, ld, w, part, out, counter);
    else if (nk <= 15) k_cgs_dot_cs<16><<<nbc, 256, 0, s>>>(n, nk, V, ld, w, part, out, counter);
    else k_cgs_dot<32, 2><<<cgs_blocks(n / 2), kRedThreads, 0, s>>>(n, nk, V, ld, w, part, out, counter);
  } else {
    k_cgs_dot<32, 1><<<cgs_blocks(n), kRedThreads, 0, s>>>(n, nk, V, ld, w, part, out, counter);
  }
}

void launch_cgs_update_dot(long long n, int nk, const double* V, long long ld, const double* h, double* w, double* part,
                           double* out, unsigned* counter, cudaStream_t s) {
  // one 256-thread block per SM: the 32 accumulators + the second column pass need > 128 registers
  const int nb1 = (int)std::min<long long>((n + kRedThreads - 1) / kRedThreads, 148);
  const int nb2 = cgs_blocks(vec2(n, ld) ? n / 2 : n);
  if (vec2(n, ld)) {
    if (nk <= 8) k_cgs_update_dot<8, 2><<<nb2, kRedThreads, 0, s>>>(n, nk, V, ld, h, w, part, out, counter);
    else if (nk <= 16) k_cgs_update_dot<16, 2><<<nb2, kRedThreads, 0, s>>>(n, nk, V, ld, h, w, part, out, counter);
    else k_cgs_update_dot<32, 2><<<nb1, kRedThreads, 0, s>>>(n, nk, V, ld, h, w, part, out, counter);
  } else {
    k_cgs_update_dot<32, 1><<<nb1, kRedThreads, 0, s>>>(n, nk, V, ld, h, w, part, out, counter);
  }
}

#define NK_DISPATCH2(nk, VW, KERNEL, ...)                      \
  do {                                                         \
    if ((nk) <= 8) KERNEL<8, VW>__VA_ARGS__;                   \
    else if ((nk) <= 16) KERNEL<16, VW>__VA_ARGS__;            \
    else if ((nk) <= 32) KERNEL<32, VW>__VA_ARGS__;            \
    else KERNEL<64, VW>__VA_ARGS__;                            \
  } while (0)

void launch_update_scale_dev(long long n, int nk, const double* V, long long ld, const double* hv, double* w,
                             cudaStream_t s) {
  if (vec2(n, ld)) NK_DISPATCH2(nk, 2, k_update_scale_dev, <<<vec_blocks(n / 2), 256, 0, s>>>(n, nk, V, ld, hv, w));
  else NK_DISPATCH2(nk, 1, k_update_scale_dev, <<<vec_blocks(n), 256, 0, s>>>(n, nk, V, ld, hv, w));
}

void launch_lincomb(long long n, int nk, const double* V, long long ld, const double* y, double* out, cudaStream_t s) {
  Coefs c;
  for (int k = 0; k < nk && k < 64; ++k) c.c[k] = y[k];
  k_lincomb<<<vec_blocks(n), 256, 0, s>>>(n, nk, V, ld, c, out);
}

void launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t s) {
  k_axpby<<<vec_blocks(n), 256, 0, s>>>(n, a, x, b, y);
}

void launch_xpay(long long n, const double* x, double a, const double* y, double* z, cudaStream_t s) {
  k_xpay<<<vec_blocks(n), 256, 0, s>>>(n, x, a, y, z);
}

}  // namespace nks
