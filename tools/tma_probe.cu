// Probe: which TMA / bulk-copy forms are legal on this device (each mode in its own process).
// usage: tma_probe <mode>
//   0: 2D tensor fp64 box {16,96}, fence.mbarrier_init     1: same without the fence
//   2: 1D cp.async.bulk (non-tensor) of 4 KB                3: 2D tensor, dtype UINT64 instead of FLOAT64
//   4: 2D tensor fp64 with .shared::cta destination form    5: 2D tensor fp32 box {16,96}
#include <cuda.h>
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

__constant__ CUtensorMap c_tm;
__global__ void k(const __grid_constant__ CUtensorMap tm, int mode, const double* src, double* out, int nbytes,
                  const CUtensorMap* gtm) {
  const CUtensorMap* mp = mode == 6 ? gtm : mode == 7 ? &c_tm : &tm;
  extern __shared__ __align__(1024) unsigned char sm[];
  __shared__ __align__(8) unsigned long long bar;
  unsigned b = (unsigned)__cvta_generic_to_shared(&bar);
  unsigned dst = (unsigned)__cvta_generic_to_shared(sm);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(b));
    if (mode != 1) asm volatile("fence.mbarrier_init.release.cluster;");
    asm volatile("fence.proxy.async.shared::cta;");
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(b), "r"(nbytes));
    if (mode == 2) {
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                   ::"r"(dst), "l"(src), "r"(nbytes), "r"(b) : "memory");
    } else if (mode == 4) {
      asm volatile("cp.async.bulk.tensor.2d.shared::cta.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst), "l"(&tm), "r"(3), "r"(0), "r"(b) : "memory");
    } else {
      asm volatile("cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3}], [%4];"
                   ::"r"(dst), "l"(mp), "r"(3), "r"(0), "r"(b) : "memory");
    }
    unsigned done = 0;
    while (!done)
      asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(done) : "r"(b) : "memory");
    const double* d = reinterpret_cast<const double*>(sm);
    for (int i = 0; i < nbytes / 8; ++i) out[i] = d[i];
  }
}

typedef CUresult (*Enc)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*, const cuuint64_t*,
                        const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                        CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int mode = argc > 1 ? atoi(argv[1]) : 0;
  const long long ld = 1024;
  std::vector<double> h(ld * 208);
  for (size_t i = 0; i < h.size(); ++i) h[i] = (double)i;
  double *d, *o;
  cudaMalloc(&d, h.size() * 8);
  cudaMalloc(&o, 64 * 1024);
  cudaMemcpy(d, h.data(), h.size() * 8, cudaMemcpyHostToDevice);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  CUtensorMap tm;
  const int esz = mode == 5 ? 4 : 8;
  cuuint64_t gd[2] = {(cuuint64_t)ld, 208}, gs[1] = {(cuuint64_t)ld * esz};
  cuuint32_t box[2] = {16, 96}, es[2] = {1, 1};
  CUtensorMapDataType dt = mode == 3 ? CU_TENSOR_MAP_DATA_TYPE_UINT64
                           : mode == 5 ? CU_TENSOR_MAP_DATA_TYPE_FLOAT32 : CU_TENSOR_MAP_DATA_TYPE_FLOAT64;
  CUresult r = ((Enc)fn)(&tm, dt, 2, d, gd, gs, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                         CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  const int nbytes = mode == 2 ? 4096 : 16 * 96 * esz;
  CUtensorMap* gtm;
  cudaMalloc(&gtm, sizeof(CUtensorMap));
  cudaMemcpy(gtm, &tm, sizeof(tm), cudaMemcpyHostToDevice);
  cudaMemcpyToSymbol(c_tm, &tm, sizeof(tm));
  printf("host tm addr mod 64 = %d\n", (int)((size_t)&tm % 64));
  k<<<1, 32, 40 * 1024>>>(tm, mode, d, o, nbytes, gtm);
  cudaError_t l = cudaGetLastError();
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<double> ho(nbytes / 8);
  cudaMemcpy(ho.data(), o, nbytes, cudaMemcpyDeviceToHost);
  int bad = 0;
  if (mode == 2) { for (int i = 0; i < nbytes / 8; ++i) bad += ho[i] != (double)i; }
  else if (mode != 5) { for (int p = 0; p < 96; ++p) for (int c = 0; c < 16; ++c) bad += ho[p * 16 + c] != (double)(p * ld + 3 + c); }
  printf("mode %d: encode %d launch %s sync %s mismatches %d\n", mode, (int)r, cudaGetErrorString(l), cudaGetErrorString(e), bad);
  return 0;
}
