// Cost of a named barrier (bar.sync 1,160: 5 warps) per iteration when each iteration also issues
// one memory operation of a given kind (does the barrier wait for it?).  Cluster of 2 CTAs.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/bar_probe tools/bar_probe.cu
#include <cstdio>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(2, 1, 1) k(int mode, int iters, double* g, long long* out) {
  __shared__ double sh[256];
  __shared__ __align__(8) unsigned long long mb;
  cg::cluster_group cl = cg::this_cluster();
  const int tid = threadIdx.x;
  sh[tid % 256] = tid;
  if (tid == 0) asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&mb)), "r"(1 << 20));
  __syncthreads();
  cl.sync();
  unsigned remote;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(remote) : "r"((unsigned)__cvta_generic_to_shared(&sh[tid % 32])), "r"(cl.block_rank() ^ 1));
  double acc = 0.0;
  const long long t0 = clock64();
  for (int it = 0; it < iters; ++it) {
    const bool w0 = tid < 32;
    if (mode == 1 && w0) asm volatile("st.relaxed.cluster.shared::cluster.f64 [%0], %1;" ::"r"(remote), "d"(acc) : "memory");
    if (mode == 2 && w0) g[blockIdx.x * 1024 + (it & 1023)] = acc;
    if (mode == 3 && w0) acc += __ldg(g + ((it * 4099 + blockIdx.x * 77) & ((1 << 24) - 1)));
    if (mode == 4 && w0 && tid == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"((unsigned)__cvta_generic_to_shared(&mb)) : "memory");
    if (mode == 5 && w0) { unsigned long long v; asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(&sh[tid]))); acc += (double)v; }
    if (mode == 6 && w0) asm volatile("st.shared.f64 [%0], %1;" ::"r"((unsigned)__cvta_generic_to_shared(&sh[tid])), "d"(acc) : "memory");
    if (mode == 7 && w0) { double v; asm volatile("ld.shared.f64 %0, [%1];" : "=d"(v) : "r"((unsigned)__cvta_generic_to_shared(&sh[(tid + it) & 255])) : "memory"); acc = fma(acc, 0.5, v); }
    if (mode == 8 && w0) { unsigned long long v; asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"((unsigned)__cvta_generic_to_shared(&sh[tid]))); if (__all_sync(0xffffffffu, v != 12345ull)) acc += 1.0; }
    asm volatile("bar.sync 1, 160;" ::: "memory");
  }
  const long long t1 = clock64();
  if (tid == 0) out[blockIdx.x] = t1 - t0;
  if (acc == 1234.5) g[0] = acc;
  cl.sync();
}

int main() {
  double* g; long long* o;
  cudaMalloc(&g, (1 << 24) * sizeof(double) + 8 * 1024 * 1024);
  cudaMemset(g, 0, (1 << 24) * sizeof(double));
  cudaMalloc(&o, 64 * sizeof(long long));
  const char* names[] = {"bar only", "DSMEM st.relaxed.cluster", "STG", "LDG (used)", "mbarrier arrive", "ld.volatile.shared",
                         "st.shared", "ld.shared dep chain", "volatile poll + vote"};
  for (int mode = 0; mode < 9; ++mode) {
    const int iters = 20000;
    k<<<2, 160>>>(mode, iters, g, o);
    cudaError_t e = cudaDeviceSynchronize();
    long long h[2];
    cudaMemcpy(h, o, sizeof(h), cudaMemcpyDeviceToHost);
    printf("mode %d %-28s: %.1f cycles/iteration (%s)\n", mode, names[mode], (double)h[0] / iters, cudaGetErrorString(e));
  }
  return 0;
}
