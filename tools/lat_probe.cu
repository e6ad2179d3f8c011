// Probe instruction latencies on this device: dependent DFMA chain, 64-bit SHFL chain, LDS chain,
// and DFMA throughput (independent chains, all warps).
#include <cuda_runtime.h>
#include <cstdio>

__global__ void k_dfma_lat(double* out, double a, double b, int n, long long* cyc) {
  double x = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) x = fma(x, a, b);
  long long c1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
__global__ void k_shfl_lat(double* out, int n, long long* cyc) {
  double x = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) x = __shfl_sync(0xffffffffu, x, (threadIdx.x + 1) & 31) + 1.0;
  long long c1 = clock64();
  out[threadIdx.x] = x;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
__global__ void k_lds_lat(double* out, int n, long long* cyc) {
  __shared__ int idx[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) idx[i] = (i + 1) & 1023;
  __syncthreads();
  int p = threadIdx.x;
  long long c0 = clock64();
  for (int i = 0; i < n; ++i) p = idx[p];
  long long c1 = clock64();
  out[threadIdx.x] = p;
  if (threadIdx.x == 0) *cyc = c1 - c0;
}
__global__ void k_dfma_tput(double* out, double a, double b, int n) {
  double x0 = threadIdx.x, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3, x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < n; ++i) {
    x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
    x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

int main() {
  double* out; long long* cyc; long long h;
  cudaMalloc(&out, 148 * 1024 * 8 * 8); cudaMalloc(&cyc, 8);
  const int n = 4096;
  k_dfma_lat<<<1, 32>>>(out, 1.0000001, 1e-9, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cyc\n", (double)h / n);
  k_shfl_lat<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("SHFL(f64)+DADD dependent latency: %.2f cyc\n", (double)h / n);
  k_lds_lat<<<1, 32>>>(out, n, cyc); cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
  printf("LDS dependent latency: %.2f cyc\n", (double)h / n);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  const int m = 20000;
  k_dfma_tput<<<148 * 4, 256>>>(out, 1.0000001, 1e-9, m);
  cudaEventRecord(e0);
  k_dfma_tput<<<148 * 4, 256>>>(out, 1.0000001, 1e-9, m);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double flops = 2.0 * 8 * m * 148.0 * 4 * 256;
  printf("DFMA throughput: %.2f TFLOP/s fp64\n", flops / (ms * 1e-3) / 1e12);
  return 0;
}
