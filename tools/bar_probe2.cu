// Named-barrier cost on B200: bar.sync 0 vs bar.sync 1,160 vs bar.sync 1 (no count), with and without a
// cluster launch, 160 threads (five warps) looping on the barrier.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bar_probe2 tools/bar_probe2.cu
#include <cstdio>
template <int MODE>
__global__ void k(int iters, long long* out) {
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    if (MODE == 0) asm volatile("bar.sync 0;" ::: "memory");
    if (MODE == 1) asm volatile("bar.sync 1, 160;" ::: "memory");
    if (MODE == 2) asm volatile("bar.sync 1;" ::: "memory");
    if (MODE == 3) __syncthreads();
  }
  const long long t1 = clock64();
  if (threadIdx.x == 0) out[blockIdx.x] = t1 - t0;
}
template <int MODE>
void run(bool cluster, long long* o) {
  const int iters = 20000;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(2, 1, 1);
  cfg.blockDim = dim3(160, 1, 1);
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = 2; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = cluster ? 1 : 0;
  cudaLaunchKernelEx(&cfg, k<MODE>, iters, o);
  cudaError_t e = cudaDeviceSynchronize();
  long long h[2];
  cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
  printf("mode %d (%s) cluster=%d: %.1f cycles/iteration (%s)\n", MODE,
         MODE == 0 ? "bar.sync 0" : MODE == 1 ? "bar.sync 1,160" : MODE == 2 ? "bar.sync 1" : "__syncthreads",
         (int)cluster, (double)h[0] / iters, cudaGetErrorString(e));
}
int main() {
  long long* o;
  cudaMalloc(&o, 64 * sizeof(long long));
  for (int c = 0; c < 2; ++c) { run<0>(c, o); run<1>(c, o); run<2>(c, o); run<3>(c, o); }
  return 0;
}
