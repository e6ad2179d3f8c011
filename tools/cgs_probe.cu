// Bandwidth of the GMRES update kernel w = (w - sum_k h_k V_k) * s for n = 2^20, nk columns:
// scalar loads vs double2 / double4 per thread, grid-stride vs one element-group per thread.
#include <cstdio>
#include <cuda_runtime.h>

template <int NK, int VW>
__global__ void k_upd(long long n, int nk, const double* __restrict__ V, long long ld, const double* __restrict__ h,
                      double* __restrict__ w, double scale) {
  __shared__ double sh[NK];
  if (threadIdx.x < nk) sh[threadIdx.x] = h[threadIdx.x];
  __syncthreads();
  const long long m = n / VW;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < m; t += (long long)gridDim.x * blockDim.x) {
    if (VW == 1) {
      double wi = w[t];
#pragma unroll
      for (int k = 0; k < NK; ++k) if (k < nk) wi = fma(-sh[k], __ldg(V + k * ld + t), wi);
      w[t] = wi * scale;
    } else if (VW == 2) {
      double2 wi = reinterpret_cast<double2*>(w)[t];
#pragma unroll
      for (int k = 0; k < NK; ++k) if (k < nk) {
        const double2 v = __ldg(reinterpret_cast<const double2*>(V + k * ld) + t);
        wi.x = fma(-sh[k], v.x, wi.x); wi.y = fma(-sh[k], v.y, wi.y);
      }
      wi.x *= scale; wi.y *= scale;
      reinterpret_cast<double2*>(w)[t] = wi;
    } else {
      double4 wi = reinterpret_cast<double4*>(w)[t];
#pragma unroll
      for (int k = 0; k < NK; ++k) if (k < nk) {
        const double4 v = reinterpret_cast<const double4*>(V + k * ld)[t];
        wi.x = fma(-sh[k], v.x, wi.x); wi.y = fma(-sh[k], v.y, wi.y);
        wi.z = fma(-sh[k], v.z, wi.z); wi.w = fma(-sh[k], v.w, wi.w);
      }
      wi.x *= scale; wi.y *= scale; wi.z *= scale; wi.w *= scale;
      reinterpret_cast<double4*>(w)[t] = wi;
    }
  }
}

template <int VW>
void run(const char* name, long long n, int nk, double* V, double* h, double* w, int blocks) {
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  k_upd<32, VW><<<blocks, 256>>>(n, nk, V, n, h, w, 1.0);
  cudaEventRecord(a);
  for (int r = 0; r < 20; ++r) k_upd<32, VW><<<blocks, 256>>>(n, nk, V, n, h, w, 1.0);
  cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b); ms /= 20;
  const double bytes = (double)(nk + 2) * n * 8;
  printf("%-10s nk %2d blocks %5d: %7.1f us  %6.0f GB/s (%s)\n", name, nk, blocks, ms * 1e3, bytes / (ms * 1e-3) / 1e9,
         cudaGetErrorString(cudaGetLastError()));
}

int main() {
  const long long n = 1 << 20;
  double *V, *h, *w;
  cudaMalloc(&V, 32 * n * 8); cudaMalloc(&h, 64 * 8); cudaMalloc(&w, n * 8);
  cudaMemset(V, 0, 32 * n * 8); cudaMemset(h, 0, 64 * 8); cudaMemset(w, 0, n * 8);
  for (int nk : {8, 24, 31}) {
    run<1>("scalar", n, nk, V, h, w, 1184);
    run<1>("scalar", n, nk, V, h, w, 4096);
    run<2>("double2", n, nk, V, h, w, 1184);
    run<2>("double2", n, nk, V, h, w, 2048);
    run<4>("double4", n, nk, V, h, w, 592);
    run<4>("double4", n, nk, V, h, w, 1024);
  }
  return 0;
}
