// K6 in 2D: the RAS/BILU(0) apply z = sum_i R_i^{0T} (L_i U_i)^{-1} R_i^delta r (reading R19)
// as a row-pipelined sweep instead of a level-synchronous one.
//
// Natural-order BILU(0) on the 13-point block pattern has dependency depth i + 2j (reading R21):
// point (i, j) needs y at (i-1,j), (i-2,j) [own row], (i-1,j-1), (i,j-1), (i+1,j-1) [row j-1] and
// (i,j-2).  Giving every box row a group of 4 threads (one per output field) and processing point
// i = t - 2j of row j at step t satisfies all of them with ONE CTA barrier per step, and keeps the
// working vector of the rows in shared memory (the backward sweep mirrors it: step t descending,
// rows j+1, j+2).  A box is split into CS stripes of consecutive rows, one CTA each, forming a
// thread-block cluster: the two boundary rows a stripe needs from its neighbour stripe are pushed
// into the neighbour's shared memory (DSMEM stores) as they are produced; the consumer spins on a
// signalling-NaN sentinel in the slot itself (each slot is written exactly once per apply, so no
// flags or fences are needed).
//
// The factor blocks a stripe needs at step t are repacked once per factorisation (k_ras2d_pack)
// into one contiguous chunk per (box, stripe, step) -- [column q = row - first active row][plane],
// plane = slot*16 + col*4 + row (blocks column-major so the 4 threads of a row read 4 consecutive
// doubles; row pitch padded for conflict-free shared-memory reads) -- and stream through an
// NS-deep shared-memory ring with one bulk copy per step (cp.async.bulk + mbarrier complete_tx,
// issued NS-1 steps ahead).  Source layout (precond.cu): plane p = slot*16 + row*4 + col,
// position-minor with leading dimension ld; slots 0..5 lower, 6 diagonal (inverted), 7..12 upper.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "nks_internal.cuh"

namespace cg = cooperative_groups;

namespace nks {

struct Box2Geo {
  int s0x, s0y;       // global coordinate of local (0,0) (may be negative: wraps)
  int ex, ey;         // extended box size
  int ox0, oy0;       // first owned local index (= delta)
  int ownx, owny;     // owned extent
  int lev_off;        // index into lev_ptr of this box's level 0
  int pad;
};

constexpr unsigned long long kSentinel = 0x7FF4DEADBEEF0001ull;   // signalling NaN: never produced by arithmetic
constexpr int kGR = 8;     // rows per warp group (4 lanes per row)
constexpr int kPF = 98;    // forward chunk row pitch (96 planes: 6 lower slots x 16); 784 B = 16 mod 128
constexpr int kPB = 114;   // backward chunk row pitch (112 planes: diagonal + 6 upper); 912 B = 16 mod 128

// slot offsets (ox, oy): lower slots 0..5 and upper 7..12 (build_slot_tables: natural key order)
// lower: (0,-2) (-1,-1) (0,-1) (1,-1) (-2,0) (-1,0); upper: (1,0) (2,0) (-1,1) (0,1) (1,1) (0,2)
__host__ __device__ constexpr int lo_dx(int a) { return a == 1 ? -1 : a == 3 ? 1 : a == 4 ? -2 : a == 5 ? -1 : 0; }
__host__ __device__ constexpr int lo_dy(int a) { return a == 0 ? -2 : a <= 3 ? -1 : 0; }
__host__ __device__ constexpr int up_dx(int a) { return a == 0 ? 1 : a == 1 ? 2 : a == 2 ? -1 : a == 4 ? 1 : 0; }
__host__ __device__ constexpr int up_dy(int a) { return a <= 1 ? 0 : a <= 4 ? 1 : 2; }

__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ double ld_spin(const double* p) {
  unsigned long long v;
  const unsigned a = smem_u32(p);
  unsigned spins = 0;
  do {
    asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(a) : "memory");
    if (++spins > (1u << 28)) __trap();      // a lost producer would otherwise hang the GPU
  } while (v == kSentinel);
  return __longlong_as_double((long long)v);
}

__device__ __forceinline__ void st_remote(double* local_equiv, unsigned rank, double v) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("st.relaxed.cluster.shared::cluster.f64 [%0], %1;" ::"r"(raddr), "d"(v) : "memory");
}

__device__ __forceinline__ void remote_flush(int mode) {
  if (mode == 1) asm volatile("fence.acq_rel.cluster;" ::: "memory");
  else if (mode == 2) asm volatile("fence.proxy.async.shared::cluster;" ::: "memory");
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  const unsigned a = smem_u32(bar);
  unsigned done = 0;
  while (!done) {
    asm volatile(
        "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
        : "=r"(done)
        : "r"(a), "r"(parity)
        : "memory");
  }
}

// one contiguous global -> shared bulk copy completing on an mbarrier (bytes: multiple of 16)
__device__ __forceinline__ void bulk_load(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

struct Ras2dArgs {
  const Box2Geo* boxes;
  const int* lev_ptr;
  const double* chunkF;   // [box][group][KG][8][kPF]
  const double* chunkB;   // [box][group][KG][8][kPB]
  long long N;
  int nx, ny;
  int CS, NGmax, KG, NSW, Wmax, rmaxC;
  int prof, dbg;
  const double* r;
  double* z;
};

// optional in-kernel cycle accounting (NKS_RAS2D_PROF): per warp [total, mbar wait, neighbour wait, steps]
__device__ unsigned long long g_ras2d_prof[4096 * 4];
__device__ long long g_ras2d_cta[2048 * 4];   // per CTA: start, after prologue, after sweeps, end (globaltimer ns)

__device__ __forceinline__ int jmin_of(int t, int ex) { return max(0, (t - ex + 2) >> 1); }

__device__ __forceinline__ int ld_vol(const int* p) {
  int v;
  asm volatile("ld.volatile.shared.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ int ld_acq_cluster(const int* p) {
  int v;
  asm volatile("ld.acquire.cluster.shared::cta.u32 %0, [%1];" : "=r"(v) : "r"(smem_u32(p)) : "memory");
  return v;
}
__device__ __forceinline__ void st_rel_cta(int* p, int v) {
  asm volatile("st.release.cta.shared::cta.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}
__device__ __forceinline__ void st_rel_remote(int* local_equiv, unsigned rank, int v) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("st.release.cluster.shared::cluster.u32 [%0], %1;" ::"r"(raddr), "r"(v) : "memory");
}
__device__ __forceinline__ void st_vol(int* p, int v) {
  asm volatile("st.volatile.shared.u32 [%0], %1;" ::"r"(smem_u32(p)), "r"(v) : "memory");
}

// ---------------------------------------------------------------------------------- repack
// One thread per (box point, plane): copies one factor entry from the SoA planes into the chunk of
// the point's 8-row group and step, at column q (forward: 6 lower blocks; backward: diag + 6 upper).
__global__ void k_ras2d_pack(Ras2dArgs A, const double* __restrict__ fac, long long ld, int nbox, long long work,
                             double* chunkF, double* chunkB) {
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < work;
       w += (long long)gridDim.x * blockDim.x) {
    long long rem = w;
    const int plane = (int)(rem % 208);
    rem /= 208;
    int b = 0;
    for (; b < nbox; ++b) {                 // boxes may differ in size (nbox is small)
      const long long npts = (long long)A.boxes[b].ex * A.boxes[b].ey;
      if (rem < npts) break;
      rem -= npts;
    }
    if (b >= nbox) continue;
    const Box2Geo G = A.boxes[b];
    const int j = (int)(rem / G.ex), i = (int)(rem % G.ex);
    const int t = i + 2 * j;
    const int pos = A.lev_ptr[G.lev_off + t] + (j - jmin_of(t, G.ex));
    const int g = j / kGR, R0 = g * kGR;
    const int q = j - R0;                  // chunk row = row within the 8-row group
    const int kk = t - 2 * R0;
    const int slot = plane >> 4;
    const double v = fac[(long long)plane * ld + pos];
    const long long row = (((long long)b * A.NGmax + g) * A.KG + kk) * kGR + q;
    if (slot < 6) chunkF[row * kPF + plane] = v;
    else chunkB[row * kPB + (plane - 96)] = v;
  }
}

// ---------------------------------------------------------------------------------- apply
// CTA s of box b owns the 8-row groups [g0, g1); warp w runs group g0 + w as an independent
// pipeline: its own bulk-copy ring (one step per stage, L2 prefetch further ahead), no CTA barrier
// inside the sweeps.  Lanes: 4 per row (output field f).
//
// Per step only the lag-1 neighbours (own row at t-1, row above at t-1) are on the loop-carried
// critical path; they arrive by warp shuffles of the previous step's outputs.  Older neighbours are
// register history (the vectors shuffled at earlier steps) -- the row two above comes from the row
// above's history -- so a step costs 12 f64 shuffles and 24 DFMA.  The first two rows of a group
// read the rows above from the stripe rows S (shared memory) after the group above has published
// its progress; that group is another warp of the CTA, or the last group of CTA s-1, which pushes
// its two boundary rows and its progress word into this CTA's shared memory (DSMEM).  The backward
// sweep mirrors all of it (rows below, descending steps).
constexpr int kPub = 4;    // progress published every kPub steps
constexpr int kDL2 = 12;   // L2 prefetch distance (steps); off by default (NKS_RAS2D_DBG bit 8 clear = off)

__device__ __forceinline__ void st_remote_u32(int* local_equiv, unsigned rank, int v) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("st.relaxed.cluster.shared::cluster.u32 [%0], %1;" ::"r"(raddr), "r"(v) : "memory");
}

__device__ __forceinline__ void l2_prefetch(const void* p, unsigned bytes) {
  asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}

__device__ __forceinline__ double2 lds2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// acc -= B(row f) . v   (B row = 4 consecutive doubles at p)
__device__ __forceinline__ void fms4(const double* p, const double (&v)[4], double& a0, double& a1) {
  const double2 b01 = lds2(p), b23 = lds2(p + 2);
  a0 = fma(-b01.x, v[0], a0);
  a1 = fma(-b01.y, v[1], a1);
  a0 = fma(-b23.x, v[2], a0);
  a1 = fma(-b23.y, v[3], a1);
}

__global__ void __launch_bounds__(256) k_ras2d(Ras2dArgs A) {
  extern __shared__ __align__(128) unsigned char smem[];
  long long T0;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(T0));
  cg::cluster_group cluster = cg::this_cluster();
  const int s = (int)cluster.block_rank();
  const int CS = A.CS;
  const int b = blockIdx.x / CS;
  const Box2Geo G = A.boxes[b];
  const int ex = G.ex, ey = G.ey;
  const int NG = (ey + kGR - 1) / kGR;
  const int g0 = (s * NG) / CS, g1 = ((s + 1) * NG) / CS;
  const int r0 = g0 * kGR, r1 = min(g1 * kGR, ey), R = r1 - r0;
  const int g0u = s > 0 ? ((s - 1) * NG) / CS : 0;
  const int Rup = r0 - g0u * kGR;                          // rows of CTA s-1
  const int NSW = A.NSW, Wmax = A.Wmax;
  const int tid = threadIdx.x, nthr = blockDim.x;
  const int w = tid >> 5, lane = tid & 31;
  const int rl = lane >> 2, f = lane & 3;

  // ---- shared memory carve
  const int stage_elems = kGR * kPB;
  double* stage = reinterpret_cast<double*>(smem);                                          // [Wmax][NSW][8][kPB]
  uint64_t* mbar = reinterpret_cast<uint64_t*>(stage + (size_t)Wmax * NSW * stage_elems);  // [Wmax][NSW] full
  uint64_t* ebar = mbar + Wmax * NSW;                                                       // [Wmax][NSW] empty
  int* prog = reinterpret_cast<int*>(ebar + Wmax * NSW);                                    // [Wmax][2]: fwd-in, bwd-in
  const int pitch = (ex + 4) * 4 + 2;       // doubles per S row: cells -2 .. ex+1 (2 zero pads each side) + bank spread
  double* S = reinterpret_cast<double*>(smem + ((((size_t)Wmax * NSW * stage_elems * 8 + (size_t)Wmax * NSW * 16 +
                                                  (size_t)Wmax * 8) + 15) & ~(size_t)15));  // rows -2 .. rmaxC+1
  auto Srow = [&](int rr) -> double* { return S + (size_t)(rr + 2) * pitch + 8; };   // cell 0 of row rr

  // ---- prologue: zero S (pads, halo rows), r gathered onto the stripe (R^delta), barriers, progress words
  for (int k = tid; k < (R + 4) * pitch; k += nthr) S[k] = 0.0;
  __syncthreads();
  for (int k = tid; k < R * ex * 4; k += nthr) {
    const int ff = k / (R * ex), rem = k % (R * ex), rr = rem / ex, i = rem % ex;
    int gx = (G.s0x + i) % A.nx; if (gx < 0) gx += A.nx;
    int gy = (G.s0y + r0 + rr) % A.ny; if (gy < 0) gy += A.ny;
    Srow(rr)[i * 4 + ff] = __ldg(A.r + (long long)ff * A.N + (long long)gy * A.nx + gx);
  }
  if (lane == 0 && w < Wmax) {
    for (int k = 0; k < NSW; ++k) {
      mbar_init(&mbar[w * NSW + k], 1);
      mbar_init(&ebar[w * NSW + k], 1);
    }
    prog[w * 2 + 0] = -(1 << 30);
    prog[w * 2 + 1] = 1 << 30;
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster.sync();      // halo rows and progress words of every CTA are initialised before neighbours write them
  long long T1;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(T1));

  // ---- producer warp (warp Wmax): streams every group's factor chunks into its stage ring, one bulk
  // copy per (group, step), as far ahead as the group's consumer has released stages (empty barriers)
  if (w == Wmax) {
    if (lane == 0) {
      int kiss[16];
      int ntot_w[16];
      const double* chF_w[16];
      const double* chB_w[16];
      const int ng = g1 - g0;
      for (int q = 0; q < ng; ++q) {
        const int gq = g0 + q;
        const int R0q = gq * kGR, R1q = min(R0q + kGR, ey);
        ntot_w[q] = 2 * (2 * (R1q - 1) + ex - 1 - 2 * R0q + 1);
        const long long cbq = ((long long)b * A.NGmax + gq) * A.KG;
        chF_w[q] = A.chunkF + cbq * kGR * kPF;
        chB_w[q] = A.chunkB + cbq * kGR * kPB;
        kiss[q] = 0;
      }
      const unsigned stage_sa0 = smem_u32(stage), bar_sa0 = smem_u32(mbar), ebar_sa0 = smem_u32(ebar);
      const unsigned fbytes = (unsigned)(kGR * kPF * 8), bbytes = (unsigned)(kGR * kPB * 8);
      int remaining = ng;
      while (remaining > 0) {
        bool issued = false;
        for (int q = 0; q < ng; ++q) {
          const int k = kiss[q];
          if (k >= ntot_w[q]) continue;
          const int st = k % NSW, use = k / NSW;
          if (use > 0) {      // the consumer must have released use-1 of this stage
            unsigned ok;
            asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                         : "=r"(ok) : "r"(ebar_sa0 + (q * NSW + st) * 8), "r"((unsigned)((use - 1) & 1)) : "memory");
            if (!ok) continue;
          }
          const int nF = ntot_w[q] / 2;
          const bool fw = k < nF;
          const double* src = fw ? chF_w[q] + (size_t)k * kGR * kPF : chB_w[q] + (size_t)(2 * nF - 1 - k) * kGR * kPB;
          const unsigned nb = fw ? fbytes : bbytes;
          const unsigned bar = bar_sa0 + (q * NSW + st) * 8;
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(nb) : "memory");
          asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                           stage_sa0 + (unsigned)((q * NSW + st) * stage_elems * 8)),
                       "l"(src), "r"(nb), "r"(bar)
                       : "memory");
          kiss[q] = k + 1;
          if (k + 1 >= ntot_w[q]) --remaining;
          issued = true;
        }
        if (!issued) __nanosleep(32);
      }
    }
  }

  const int g = g0 + w;
  if (w < Wmax && g < g1) {
    const int R0 = g * kGR, R1 = min(R0 + kGR, ey);
    const int lr0 = R0 - r0;                                  // local S row of the group's first row
    const int tf0 = 2 * R0, tf1 = 2 * (R1 - 1) + ex - 1;
    const int nF = tf1 - tf0 + 1, ntot = 2 * nF;
    const bool has_up = g > 0, has_dn = g + 1 < NG;
    const bool up_remote = g == g0 && s > 0, dn_remote = g + 1 == g1 && s < CS - 1;
    const int tf1_up = 2 * (R0 - 1) + ex - 1;               // last forward step of the group above
    const int tf0_dn = 2 * R1;                                // first step of the group below
    const long long cb = ((long long)b * A.NGmax + g) * A.KG;
    const double* chF = A.chunkF + cb * kGR * kPF;
    const double* chB = A.chunkB + cb * kGR * kPB;
    double* wstage = stage + (size_t)w * NSW * stage_elems;
    // 32-bit shared addresses, computed once (the loops never convert generic pointers)
    const unsigned bar_sa = smem_u32(mbar + w * NSW), ebar_sa = smem_u32(ebar + w * NSW);
    const unsigned stage_bytes = (unsigned)(stage_elems * 8);
    const unsigned fbytes = (unsigned)(kGR * kPF * 8), bbytes = (unsigned)(kGR * kPB * 8);
    auto test_stage = [&](int stg, unsigned par) -> unsigned {     // non-blocking probe, issued early
      unsigned ok;
      asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(bar_sa + stg * 8), "r"(par));
      return ok;
    };
    auto wait_stage = [&](int stg, unsigned par) {
      const unsigned a = bar_sa + stg * 8;
      unsigned done = 0;
      while (!done)
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(done) : "r"(a), "r"(par) : "memory");
    };
    const int j = R0 + rl;
    const int lr = lr0 + rl;
    const bool row_ok = j < R1;
    double* const Sown = Srow(lr);
    const double* const Sup1 = Srow(lr - 1);
    const double* const Sup2 = Srow(lr - 2);
    const double* const Sdn1 = Srow(lr + 1);
    const double* const Sdn2 = Srow(lr + 2);
    const int q4 = lane & ~3;                       // own quad
    const int qa = (lane - 4) & 31, qb = (lane + 4) & 31;     // same field, row above / below
    const int qa4 = qa & ~3, qb4 = qb & ~3;
    int* const pubF = dn_remote ? &prog[0 * 2 + 0] : &prog[(w + 1) * 2 + 0];                 // warp 0 of CTA s+1 if remote
    int* const pubB = up_remote ? &prog[(g0 - 1 - g0u) * 2 + 1] : &prog[(w - 1) * 2 + 1];   // last warp of CTA s-1
    const int* const myF = &prog[w * 2 + 0];
    const int* const myB = &prog[w * 2 + 1];
    const double* const tile0 = wstage + rl * kPF + f * 4;     // forward tile row of this lane in stage 0
    const double* const utile0 = wstage + rl * kPB + f * 4;    // backward
    long long c_start = A.prof ? clock64() : 0;
    int stg = 0;
    unsigned par = 0;
    int seen = -(1 << 30);

    // ================================================================ forward sweep
    {
      double h0 = 0.0;                                    // this lane's output at t-1
      double Yo1[4] = {0, 0, 0, 0}, Yo2[4] = {0, 0, 0, 0};                 // own row at t-1, t-2
      double Ya1[4] = {0, 0, 0, 0}, Ya2[4] = {0, 0, 0, 0}, Ya3[4] = {0, 0, 0, 0};   // row above at t-1..t-3
      int i = tf0 - 2 * j;
#pragma unroll 2
      for (int k = 0; k < nF; ++k, ++i) {
        const int t = tf0 + k;
        const bool active = row_ok && i >= 0 && i < ex;
        const int ic = min(max(i, 0), ex - 1);
        __syncwarp();
        const unsigned ready = test_stage(stg, par);
        // row two above at t-4 = the row above's Ya3 (before it shifts); lag-1 vectors at t-1
        double Yaa4[4], n_o1[4], n_a1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          Yaa4[c] = __shfl_sync(0xffffffffu, Ya3[c], qa);
          n_o1[c] = __shfl_sync(0xffffffffu, h0, q4 + c);
          n_a1[c] = __shfl_sync(0xffffffffu, h0, qa4 + c);
        }
        if (has_up) {
          const int need = min(t - 1, tf1_up);
          if (seen < need) {
            int v;
            do { v = ld_acq_cluster(myF); } while (__any_sync(0xffffffffu, v < need));
            seen = __shfl_sync(0xffffffffu, v, 0);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          Ya3[c] = Ya2[c]; Ya2[c] = Ya1[c]; Ya1[c] = n_a1[c];
          Yo2[c] = Yo1[c]; Yo1[c] = n_o1[c];
        }
        // the group's first rows take the rows above straight from S (the group above ran steps this
        // warp never executed, so there is no history to shift)
        {
          // uniform loads (valid rows for every lane), selected for the group's first rows: no branch
          const double2 p1 = lds2(Sup1 + (ic + 1) * 4), p2 = lds2(Sup1 + (ic + 1) * 4 + 2);
          const double2 q1 = lds2(Sup1 + ic * 4), q2 = lds2(Sup1 + ic * 4 + 2);
          const double2 r1 = lds2(Sup1 + (ic - 1) * 4), r2 = lds2(Sup1 + (ic - 1) * 4 + 2);
          const double2 s1 = lds2(Sup2 + ic * 4), s2 = lds2(Sup2 + ic * 4 + 2);
          const bool b0 = rl == 0, b01 = rl < 2;
          Ya1[0] = b0 ? p1.x : Ya1[0]; Ya1[1] = b0 ? p1.y : Ya1[1]; Ya1[2] = b0 ? p2.x : Ya1[2]; Ya1[3] = b0 ? p2.y : Ya1[3];
          Ya2[0] = b0 ? q1.x : Ya2[0]; Ya2[1] = b0 ? q1.y : Ya2[1]; Ya2[2] = b0 ? q2.x : Ya2[2]; Ya2[3] = b0 ? q2.y : Ya2[3];
          Ya3[0] = b0 ? r1.x : Ya3[0]; Ya3[1] = b0 ? r1.y : Ya3[1]; Ya3[2] = b0 ? r2.x : Ya3[2]; Ya3[3] = b0 ? r2.y : Ya3[3];
          Yaa4[0] = b01 ? s1.x : Yaa4[0]; Yaa4[1] = b01 ? s1.y : Yaa4[1];
          Yaa4[2] = b01 ? s2.x : Yaa4[2]; Yaa4[3] = b01 ? s2.y : Yaa4[3];
        }
        if (!ready) wait_stage(stg, par);
        const double* L = tile0 + (size_t)stg * stage_elems;
        double a0 = Sown[ic * 4 + f], a1 = 0.0;
        fms4(L + 0 * 16, Yaa4, a0, a1);      // (0,-2)
        fms4(L + 1 * 16, Ya3, a0, a1);       // (-1,-1)
        fms4(L + 2 * 16, Ya2, a0, a1);       // (0,-1)
        fms4(L + 4 * 16, Yo2, a0, a1);       // (-2,0)
        fms4(L + 3 * 16, Ya1, a0, a1);       // (1,-1)  lag 1
        fms4(L + 5 * 16, Yo1, a0, a1);       // (-1,0)  lag 1
        const double y = active ? a0 + a1 : 0.0;
        h0 = y;
        if (active) {
          Sown[i * 4 + f] = y;
          if (dn_remote && j >= R1 - 2) st_remote(Srow(j - r1) + i * 4 + f, (unsigned)(s + 1), y);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ebar_sa + stg * 8) : "memory");
        if (++stg == NSW) { stg = 0; par ^= 1u; }
        if (has_dn && ((k & (kPub - 1)) == kPub - 1 || k == nF - 1)) {
          __syncwarp();
          if (lane == 0) {
            if (dn_remote) st_rel_remote(pubF, (unsigned)(s + 1), t);   // release: cumulative over the warp's
            else st_rel_cta(pubF, t);                                   // stores ordered by __syncwarp
          }
        }
      }
    }
    // ================================================================ backward sweep
    seen = 1 << 30;
    {
      double h0 = 0.0;
      double Xo1[4] = {0, 0, 0, 0}, Xo2[4] = {0, 0, 0, 0};                 // own row at t+1, t+2 (i+1, i+2)
      double Xb1[4] = {0, 0, 0, 0}, Xb2[4] = {0, 0, 0, 0}, Xb3[4] = {0, 0, 0, 0};   // row below at t+1..t+3 (i-1, i, i+1)
      int i = tf1 - 2 * j;
#pragma unroll 2
      for (int kb = 0; kb < nF; ++kb, --i) {
        const int t = tf1 - kb;
        const bool active = row_ok && i >= 0 && i < ex;
        const int ic = min(max(i, 0), ex - 1);
        __syncwarp();
        const unsigned ready = test_stage(stg, par);
        double Xbb4[4], n_o1[4], n_b1[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          Xbb4[c] = __shfl_sync(0xffffffffu, Xb3[c], qb);
          n_o1[c] = __shfl_sync(0xffffffffu, h0, q4 + c);
          n_b1[c] = __shfl_sync(0xffffffffu, h0, qb4 + c);
        }
        if (has_dn) {
          const int need = max(t + 1, tf0_dn);
          if (seen > need) {
            int v;
            do { v = ld_acq_cluster(myB); } while (__any_sync(0xffffffffu, v > need));
            seen = __shfl_sync(0xffffffffu, v, 0);
          }
        }
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          Xb3[c] = Xb2[c]; Xb2[c] = Xb1[c]; Xb1[c] = n_b1[c];
          Xo2[c] = Xo1[c]; Xo1[c] = n_o1[c];
        }
        {
          // uniform loads; lanes of rows past the group's end read their own row (never selected)
          const bool last = row_ok && (rl == kGR - 1 || j == R1 - 1);
          const bool last2 = row_ok && (rl >= kGR - 2 || j >= R1 - 2);
          const double* d1 = row_ok ? Sdn1 : Sown;
          const double* d2 = row_ok ? Sdn2 : Sown;
          const double2 p1 = lds2(d1 + (ic - 1) * 4), p2 = lds2(d1 + (ic - 1) * 4 + 2);
          const double2 q1 = lds2(d1 + ic * 4), q2 = lds2(d1 + ic * 4 + 2);
          const double2 r1 = lds2(d1 + (ic + 1) * 4), r2 = lds2(d1 + (ic + 1) * 4 + 2);
          const double2 s1 = lds2(d2 + ic * 4), s2 = lds2(d2 + ic * 4 + 2);
          Xb1[0] = last ? p1.x : Xb1[0]; Xb1[1] = last ? p1.y : Xb1[1]; Xb1[2] = last ? p2.x : Xb1[2]; Xb1[3] = last ? p2.y : Xb1[3];
          Xb2[0] = last ? q1.x : Xb2[0]; Xb2[1] = last ? q1.y : Xb2[1]; Xb2[2] = last ? q2.x : Xb2[2]; Xb2[3] = last ? q2.y : Xb2[3];
          Xb3[0] = last ? r1.x : Xb3[0]; Xb3[1] = last ? r1.y : Xb3[1]; Xb3[2] = last ? r2.x : Xb3[2]; Xb3[3] = last ? r2.y : Xb3[3];
          Xbb4[0] = last2 ? s1.x : Xbb4[0]; Xbb4[1] = last2 ? s1.y : Xbb4[1];
          Xbb4[2] = last2 ? s2.x : Xbb4[2]; Xbb4[3] = last2 ? s2.y : Xbb4[3];
        }
        if (!ready) wait_stage(stg, par);
        const double* U = utile0 + (size_t)stg * stage_elems;
        double a0 = Sown[ic * 4 + f], a1 = 0.0;
        fms4(U + 6 * 16, Xbb4, a0, a1);      // (0,2)
        fms4(U + 5 * 16, Xb3, a0, a1);       // (1,1)
        fms4(U + 4 * 16, Xb2, a0, a1);       // (0,1)
        fms4(U + 2 * 16, Xo2, a0, a1);       // (2,0)
        fms4(U + 3 * 16, Xb1, a0, a1);       // (-1,1) lag 1
        fms4(U + 1 * 16, Xo1, a0, a1);       // (1,0)  lag 1
        const double sum = a0 + a1;
        const double v0 = __shfl_sync(0xffffffffu, sum, q4 + 0), v1 = __shfl_sync(0xffffffffu, sum, q4 + 1);
        const double v2 = __shfl_sync(0xffffffffu, sum, q4 + 2), v3 = __shfl_sync(0xffffffffu, sum, q4 + 3);
        const double2 d01 = lds2(U), d23 = lds2(U + 2);
        const double xr = fma(d01.x, v0, d01.y * v1) + fma(d23.x, v2, d23.y * v3);
        const double x = active ? xr : 0.0;
        h0 = x;
        if (active) {
          Sown[i * 4 + f] = x;
          if (up_remote && j < R0 + 2) st_remote(Srow(Rup + (j - r0)) + i * 4 + f, (unsigned)(s - 1), x);
        }
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(ebar_sa + stg * 8) : "memory");
        if (++stg == NSW) { stg = 0; par ^= 1u; }
        if (has_up && ((kb & (kPub - 1)) == kPub - 1 || kb == nF - 1)) {
          __syncwarp();
          if (lane == 0) {
            if (up_remote) st_rel_remote(pubB, (unsigned)(s - 1), t);
            else st_rel_cta(pubB, t);
          }
        }
      }
    }
    if (A.prof && lane == 0) {
      const int slotp = blockIdx.x * Wmax + w;
      g_ras2d_prof[slotp * 4 + 0] = clock64() - c_start;
      g_ras2d_prof[slotp * 4 + 1] = 0;
      g_ras2d_prof[slotp * 4 + 2] = 0;
      g_ras2d_prof[slotp * 4 + 3] = 2 * nF;
    }
  }
  __syncthreads();
  long long T2;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(T2));

  // ---- R_i^{0T}: owned points only
  for (int k = tid; k < R * ex * 4; k += nthr) {
    const int ff = k / (R * ex), rem = k % (R * ex), rr = rem / ex, i = rem % ex;
    const int jj = r0 + rr;
    if (i < G.ox0 || i >= G.ox0 + G.ownx || jj < G.oy0 || jj >= G.oy0 + G.owny) continue;
    int gx = (G.s0x + i) % A.nx; if (gx < 0) gx += A.nx;
    int gy = (G.s0y + jj) % A.ny; if (gy < 0) gy += A.ny;
    A.z[(long long)ff * A.N + (long long)gy * A.nx + gx] = Srow(rr)[i * 4 + ff];
  }
  cluster.sync();      // no CTA leaves while a neighbour may still address its shared memory
  if (A.prof && threadIdx.x == 0) {
    long long T3;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(T3));
    g_ras2d_cta[blockIdx.x * 4 + 0] = T0; g_ras2d_cta[blockIdx.x * 4 + 1] = T1;
    g_ras2d_cta[blockIdx.x * 4 + 2] = T2; g_ras2d_cta[blockIdx.x * 4 + 3] = T3;
  }
}

// ------------------------------------------------------------------------------------------ host
struct Ras2dPlan {
  int CS = 1, NSW = 4, Wmax = 1, NGmax = 1, KG = 1, threads = 32, nbox = 0, rmaxC = 8, max_clusters = 0;
  size_t smem = 0;
  long long npts_total = 0;
  Ras2dArgs A{};
};

static void split(int n, int nsub, std::vector<int>& st, std::vector<int>& ln) {
  const int base = n / nsub, rem = n % nsub;
  int s = 0;
  for (int b = 0; b < nsub; ++b) {
    const int l = base + (b < rem ? 1 : 0);
    st.push_back(s);
    ln.push_back(l);
    s += l;
  }
}

struct Ras2dGeom {
  int CS, NGmax, Wmax, KG, exmax, eymax, nbox;
};

static bool ras2d_geom(const nks_grid& g, Ras2dGeom& Gm, int cs_try = 0) {
  if (g.dim != 2) return false;
  std::vector<int> st[2], ln[2];
  for (int j = 0; j < 2; ++j) split(g.n[j], g.nsub[j], st[j], ln[j]);
  Gm.nbox = g.nsub[0] * g.nsub[1];
  Gm.exmax = *std::max_element(ln[0].begin(), ln[0].end()) + 2 * g.overlap;
  Gm.eymax = *std::max_element(ln[1].begin(), ln[1].end()) + 2 * g.overlap;
  const int eymin = *std::min_element(ln[1].begin(), ln[1].end()) + 2 * g.overlap;
  const int NGmin = (eymin + kGR - 1) / kGR;
  Gm.NGmax = (Gm.eymax + kGR - 1) / kGR;
  int CS = cs_try > 0 ? cs_try : std::max(1, std::min(8, 148 / Gm.nbox));
  if (const char* e = std::getenv("NKS_RAS2D_CS")) CS = std::max(1, std::min(8, std::atoi(e)));   // experiments
  CS = std::min(CS, NGmin);
  Gm.CS = CS;
  Gm.Wmax = (Gm.NGmax + CS - 1) / CS;
  Gm.KG = 2 * (kGR - 1) + Gm.exmax;
  return Gm.Wmax <= 7;      // 32 (Wmax + 1) threads <= 256 (launch bound)
}

// Workspace bytes for the packed chunks + geometry (0 when the pipelined path does not apply).
size_t ras2d_workspace_bytes(const nks_grid& g) {
  Ras2dGeom Gm;
  if (!ras2d_geom(g, Gm)) return 0;
  const size_t rows = (size_t)Gm.nbox * Gm.NGmax * Gm.KG * kGR;
  return rows * (kPF + kPB) * sizeof(double) + (size_t)Gm.nbox * sizeof(Box2Geo) + 1024;
}

// Plans the pipelined apply inside the given workspace slice; nullptr = use the level-synchronous kernel.
// Shared memory and co-residency of one launch configuration: returns NSW (0 = does not fit) and the
// number of clusters that can be resident at once.
static int ras2d_fit(const Ras2dGeom& Gm, size_t& smem, int& max_clusters) {
  const int rmaxC = Gm.Wmax * kGR;
  const int pitch = (Gm.exmax + 4) * 4 + 2;
  const size_t fixed = (size_t)(rmaxC + 4) * pitch * 8 + (size_t)Gm.Wmax * 8 + 64;
  const size_t per_stage = (size_t)Gm.Wmax * (kGR * kPB * 8 + 16);
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  int NSW = 6;
  if (const char* e = std::getenv("NKS_RAS2D_NSW")) NSW = std::max(2, std::atoi(e));
  while (NSW > 3 && fixed + NSW * per_stage > (size_t)maxsm) --NSW;
  if (fixed + NSW * per_stage > (size_t)maxsm) return 0;
  smem = fixed + NSW * per_stage;
  if (cudaFuncSetAttribute(k_ras2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) return 0;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(Gm.nbox * Gm.CS, 1, 1);
  cfg.blockDim = dim3(32 * (Gm.Wmax + 1), 1, 1);
  cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = Gm.CS; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  max_clusters = 0;
  if (cudaOccupancyMaxActiveClusters(&max_clusters, k_ras2d, &cfg) != cudaSuccess) max_clusters = 0;
  cudaGetLastError();
  return NSW;
}

// Plans the pipelined apply inside the given workspace slice; nullptr = use the level-synchronous kernel.
// The cluster size is the largest <= 8 whose clusters are all co-resident (one wave).
void* ras2d_plan(const nks_grid& g, const BoxSet& B, void* ws, size_t ws_bytes, cudaStream_t stream, std::string& why) {
  Ras2dGeom Gm;
  if (g.dim != 2 || !ras2d_geom(g, Gm)) { why = "not applicable (dim or box height)"; return nullptr; }
  if (B.nslots != 13 || B.diag != 6) { why = "unexpected slot table"; return nullptr; }
  if (ws_bytes < ras2d_workspace_bytes(g)) { why = "workspace"; return nullptr; }
  int NSW = 0, ncl = 0;
  size_t smem = 0;
  for (int cs = Gm.CS; cs >= 1; --cs) {
    Ras2dGeom T;
    if (!ras2d_geom(g, T, cs)) continue;
    size_t sm = 0;
    int mc = 0;
    const int nsw = ras2d_fit(T, sm, mc);
    if (nsw == 0) continue;
    if (NSW == 0 || mc >= T.nbox) { Gm = T; NSW = nsw; smem = sm; ncl = mc; }
    if (mc >= T.nbox) break;
  }
  if (NSW == 0) { why = "shared memory"; return nullptr; }
  std::vector<int> st[2], ln[2];
  for (int j = 0; j < 2; ++j) split(g.n[j], g.nsub[j], st[j], ln[j]);
  std::vector<Box2Geo> geo;
  long long npts = 0;
  for (int by = 0; by < g.nsub[1]; ++by)
    for (int bx = 0; bx < g.nsub[0]; ++bx) {
      Box2Geo q{};
      q.ex = ln[0][bx] + 2 * g.overlap;
      q.ey = ln[1][by] + 2 * g.overlap;
      q.s0x = st[0][bx] - g.overlap;
      q.s0y = st[1][by] - g.overlap;
      q.ox0 = g.overlap;
      q.oy0 = g.overlap;
      q.ownx = ln[0][bx];
      q.owny = ln[1][by];
      q.lev_off = B.h_box_lev_off[geo.size()];
      npts += (long long)q.ex * q.ey;
      geo.push_back(q);
    }
  Ras2dPlan* P = new Ras2dPlan();
  P->CS = Gm.CS; P->NSW = NSW; P->Wmax = Gm.Wmax; P->NGmax = Gm.NGmax; P->KG = Gm.KG; P->nbox = Gm.nbox;
  P->rmaxC = Gm.Wmax * kGR;
  P->threads = 32 * (Gm.Wmax + 1);      // + the producer warp
  P->smem = smem;
  P->npts_total = npts;
  P->max_clusters = ncl;
  char* w = (char*)ws;
  const size_t rows = (size_t)Gm.nbox * Gm.NGmax * Gm.KG * kGR;
  double* cF = (double*)w;
  double* cB = cF + rows * kPF;
  Box2Geo* gd = (Box2Geo*)(cB + rows * kPB);
  if (cudaMemcpyAsync(gd, geo.data(), geo.size() * sizeof(Box2Geo), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
      cudaMemsetAsync(w, 0, rows * (kPF + kPB) * sizeof(double), stream) != cudaSuccess) {
    why = "copy"; delete P; return nullptr;
  }
  P->A = Ras2dArgs{gd, B.lev_ptr, cF, cB, (long long)g.n[0] * g.n[1], g.n[0], g.n[1], Gm.CS, Gm.NGmax, Gm.KG, NSW,
                   Gm.Wmax, P->rmaxC, 0, 0, nullptr, nullptr};
  if (cudaFuncSetAttribute(k_ras2d, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem) != cudaSuccess) {
    why = "smem attribute"; delete P; return nullptr;
  }
  if (std::getenv("NKS_DEBUG"))
    std::fprintf(stderr, "[nks] ras2d: %d boxes, cluster %d, %d warps/CTA, NSW %d, smem %zu B, max active clusters %d\n",
                 P->nbox, P->CS, P->Wmax, P->NSW, P->smem, ncl);
  return P;
}

void ras2d_free(void* plan) { delete (Ras2dPlan*)plan; }

int ras2d_cluster(void* plan) { return plan ? ((Ras2dPlan*)plan)->CS : 0; }

// Repack the factors (after every factorisation).
void launch_ras2d_pack(void* plan, const double* fac, long long ld, cudaStream_t s) {
  Ras2dPlan* P = (Ras2dPlan*)plan;
  const long long work = P->npts_total * 208;
  const int blocks = (int)std::min<long long>((work + 255) / 256, 148 * 16);
  k_ras2d_pack<<<blocks, 256, 0, s>>>(P->A, fac, ld, P->nbox, work, const_cast<double*>(P->A.chunkF),
                                      const_cast<double*>(P->A.chunkB));
}

cudaError_t launch_ras2d(void* plan, const double* r, double* z, cudaStream_t s) {
  Ras2dPlan* P = (Ras2dPlan*)plan;
  Ras2dArgs A = P->A;
  A.r = r;
  A.z = z;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->nbox * P->CS, 1, 1);
  cfg.blockDim = dim3(P->threads, 1, 1);
  cfg.dynamicSmemBytes = P->smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P->CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
  static const bool prof = std::getenv("NKS_RAS2D_PROF") != nullptr;
  A.prof = prof ? 1 : 0;
  static const int dbg = std::getenv("NKS_RAS2D_DBG") ? std::atoi(std::getenv("NKS_RAS2D_DBG")) : 0;
  A.dbg = dbg;
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_ras2d, A);
  if (prof && e == cudaSuccess) {
    static int calls = 0;
    if (++calls % 10 == 0) {
      const int nw = P->nbox * P->CS * P->Wmax;
      std::vector<unsigned long long> h((size_t)nw * 4, 0);
      cudaStreamSynchronize(s);
      cudaMemcpyFromSymbol(h.data(), g_ras2d_prof, h.size() * 8);
      double tot = 0, mb = 0, wt = 0, st = 0, mx = 0, n = 0;
      for (int c = 0; c < nw; ++c) {
        if (!h[c * 4 + 3]) continue;
        tot += h[c * 4]; mb += h[c * 4 + 1]; wt += h[c * 4 + 2]; st += h[c * 4 + 3]; n += 1;
        mx = std::max(mx, (double)h[c * 4]);
      }
      std::vector<long long> hc((size_t)P->nbox * P->CS * 4);
      cudaMemcpyFromSymbol(hc.data(), g_ras2d_cta, hc.size() * 8);
      long long t0 = hc[0], t3 = 0;
      double pro = 0, swp = 0, epi = 0;
      for (int c = 0; c < P->nbox * P->CS; ++c) {
        t0 = std::min(t0, hc[c * 4]); t3 = std::max(t3, hc[c * 4 + 3]);
        pro += hc[c * 4 + 1] - hc[c * 4]; swp += hc[c * 4 + 2] - hc[c * 4 + 1]; epi += hc[c * 4 + 3] - hc[c * 4 + 2];
      }
      const double nc = P->nbox * P->CS;
      std::fprintf(stderr, "[ras2d prof] CTA avg ns: prologue %.0f sweeps %.0f epilogue %.0f | first start->last end %lld ns\n",
                   pro / nc, swp / nc, epi / nc, t3 - t0);
      std::fprintf(stderr, "[ras2d prof] CS %d Wmax %d NSW %d smem %zu | per warp: total %.0f cyc (max %.0f), mbar wait %.0f, "
                   "neighbour wait %.0f, steps %.0f -> %.0f cyc/step\n", P->CS, P->Wmax, P->NSW, P->smem, tot / n, mx,
                   mb / n, wt / n, st / n, tot / st);
    }
  }
  return e;
}

}  // namespace nks
