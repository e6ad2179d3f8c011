// Probe: DSMEM ping-pong latency between two CTAs of a cluster, for several store/load forms.
// mode 0: st.relaxed.cluster.shared::cluster + ld.volatile.shared spin
// mode 1: same + fence.acq_rel.cluster after the store
// mode 2: generic store through cluster.map_shared_rank (volatile)
// mode 3: st.release.cluster + ld.acquire.cluster spin
#include <cooperative_groups.h>
#include <cuda_runtime.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void __cluster_dims__(2, 1, 1) k(int mode, int iters, long long* out) {
  __shared__ volatile long long box;
  cg::cluster_group cl = cg::this_cluster();
  const unsigned me = cl.block_rank(), other = me ^ 1;
  if (threadIdx.x == 0) box = -1;
  cl.sync();
  if (threadIdx.x != 0) { cl.sync(); return; }
  unsigned laddr = (unsigned)__cvta_generic_to_shared((void*)&box), raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(laddr), "r"(other));
  volatile long long* rgen = (volatile long long*)cl.map_shared_rank((long long*)&box, other);
  long long c0 = clock64();
  for (long long v = 0; v < iters; ++v) {
    const long long expect = 2 * v + (me == 0 ? 1 : 0);   // rank 0 sends 2v, waits 2v+1
    const long long send = 2 * v + (me == 0 ? 0 : 1);
    if (me == 1) {   // wait first
      long long x;
      do {
        if (mode == 3) asm volatile("ld.acquire.cluster.shared::cta.u64 %0, [%1];" : "=l"(x) : "r"(laddr) : "memory");
        else x = box;
      } while (x != send - 1);
    }
    if (mode == 2) *rgen = send;
    else if (mode == 3) asm volatile("st.release.cluster.shared::cluster.u64 [%0], %1;" ::"r"(raddr), "l"(send) : "memory");
    else asm volatile("st.relaxed.cluster.shared::cluster.u64 [%0], %1;" ::"r"(raddr), "l"(send) : "memory");
    if (mode == 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
    if (me == 0) {
      long long x;
      do {
        if (mode == 3) asm volatile("ld.acquire.cluster.shared::cta.u64 %0, [%1];" : "=l"(x) : "r"(laddr) : "memory");
        else x = box;
      } while (x != send + 1);
    }
  }
  long long c1 = clock64();
  if (me == 0) *out = (c1 - c0) / iters;
  cl.sync();
}

int main() {
  long long* d; long long h;
  cudaMalloc(&d, 8);
  for (int mode = 0; mode < 4; ++mode) {
    k<<<2, 32>>>(mode, 2000, d);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(&h, d, 8, cudaMemcpyDeviceToHost);
    printf("mode %d: round trip %lld cycles (%s)\n", mode, h, cudaGetErrorString(e));
  }
  return 0;
}
