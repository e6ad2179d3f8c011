// Streaming throughput of 1D cp.async.bulk (global -> shared, mbarrier complete_tx) per SM:
// one producer lane, one consumer warp that only waits full / arrives empty.  Prints B/cycle/SM.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned sa(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait_(unsigned bar, unsigned par) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(par) : "memory");
}

__global__ void k(const char* src, size_t per_cta, int chunk, int nsw, int nchunks, long long* out, int split) {
  extern __shared__ __align__(128) unsigned char smem[];
  uint64_t* full = (uint64_t*)(smem + (size_t)nsw * chunk);
  uint64_t* empty = full + nsw;
  if (threadIdx.x == 0) {
    for (int i = 0; i < nsw; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[i])));
    }
  }
  __syncthreads();
  const char* base = src + (size_t)blockIdx.x * per_cta;
  long long t0 = clock64();
  if (threadIdx.x >= 32 && threadIdx.x < 32 + split) {
    const int l = threadIdx.x - 32, sub = chunk / split;
    for (int q = 0; q < nchunks; ++q) {
      const int st = q % nsw, use = q / nsw;
      if (use > 0) wait_(sa(&empty[st]), (use - 1) & 1);
      const unsigned bar = sa(&full[st]);
      if (l == 0) asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(chunk) : "memory");
      __syncwarp((1u << split) - 1);
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                       sa(smem + (size_t)st * chunk + (size_t)l * sub)), "l"(base + ((size_t)q * chunk) % per_cta + (size_t)l * sub), "r"(sub), "r"(bar) : "memory");
    }
  } else if (threadIdx.x < 32) {
    for (int q = 0; q < nchunks; ++q) {
      const int st = q % nsw;
      wait_(sa(&full[st]), (q / nsw) & 1);
      __syncwarp();
      if (threadIdx.x == 0) asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[st])) : "memory");
    }
    if (threadIdx.x == 0) out[blockIdx.x] = clock64() - t0;
  }
}

int main() {
  const size_t per_cta = 64ull << 20;   // distinct data per CTA (> L2 overall)
  const int grids[] = {1, 96};
  const int chunks[] = {20480, 65536, 98304};
  const int splits[] = {1, 4, 16};
  char* src; long long* out;
  cudaMalloc(&src, per_cta * 148); cudaMemset(src, 1, per_cta * 148);
  cudaMalloc(&out, 148 * sizeof(long long));
  for (int chunk : chunks)
    for (int split : splits)
    for (int g : grids) {
      const int nsw = (200 * 1024) / chunk;
      const int nch = (int)((256ull << 20) / 148 / chunk) ;
      const size_t sm = (size_t)nsw * chunk + 2 * nsw * 8;
      cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
      k<<<g, 64, sm>>>(src, per_cta, chunk, nsw, nch, out, split);
      cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
      cudaEventRecord(a);
      k<<<g, 64, sm>>>(src, per_cta, chunk, nsw, nch, out, split);
      cudaEventRecord(b); cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      long long h[148]; cudaMemcpy(h, out, g * 8, cudaMemcpyDeviceToHost);
      double cyc = 0; for (int i = 0; i < g; ++i) cyc += h[i]; cyc /= g;
      const double bytes = (double)nch * chunk;
      printf("chunk %6d split %2d nsw %3d grid %3d: %.1f B/cyc/SM, %.0f cyc/chunk, total %.0f GB/s (%s)\n", chunk, split, nsw, g,
             bytes / cyc, cyc / nch, bytes * g / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
    }
  return 0;
}
