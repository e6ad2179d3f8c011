// K6 in 2D, second design: the RAS/BILU(0) apply z = sum_i R_i^{0T} (L_i U_i)^{-1} R_i^delta r
// (reading R19) as a row-pipelined sweep with ONE LANE PER BOX ROW.
//
// Natural-order BILU(0) on the 13-point block pattern has dependency depth t = i + 2j (reading
// R21): point (i, j) needs y at (i-1,j), (i-2,j) [own row], (i-1,j-1), (i,j-1), (i+1,j-1) [row
// above] and (i,j-2).  Lane rl of a warp owns box row j = r0 + rl and processes point
// i = k - 2 rl at step k, so every step of the warp is one wavefront t = 2 r0 + k.  All four field
// components of a point live in the lane's registers: the own-row neighbours are register history,
// the row-above neighbours arrive by one warp shuffle of the previous step's outputs, and the only
// loop-carried chain per step is shuffle -> 4 DFMA (-> 4 DFMA for the inverted diagonal block in the
// backward sweep).  Everything else -- 96 (forward) / 112 (backward) DFMA of the older neighbours --
// is independent work, so a step costs about its instruction issue instead of a chain of latencies
// (the first design, ras2d.cu, spread a point over 4 lanes and paid ~900 cycles per step in
// shuffle/shared-memory latencies).
//
// Geometry: a box of ey rows is split into CS stripes, one CTA each (one consumer warp, one producer
// warp), the stripes of a box forming a thread-block cluster.  The two rows a stripe needs from the
// stripe above (forward) or below (backward) are stored into its halo rows in shared memory by the
// neighbour CTA (DSMEM) as they are produced; the consumer polls the cells themselves (sentinel
// initialised, written once per apply), so the sweeps contain no fence.  The factor blocks are repacked once per factorisation into one
// chunk per (box, stripe, step) -- [row][plane], blocks row-major (lane = row reads its 16 doubles
// with 16-byte loads; row pitch = 16 mod 128 bytes) -- and streamed by the producer warp through an
// NSW-deep shared-memory ring with one 1D bulk copy (cp.async.bulk + mbarrier complete_tx) of the
// step's active rows.  r is gathered from global memory with a register prefetch kPD steps ahead;
// the forward result y goes to a per-step scratch (coalesced, L2-resident) that the backward sweep
// prefetches back; x is stored straight to z at the box's owned points (R_i^{0T}).
// Source factor layout (precond.cu): plane p = slot*16 + row*4 + col, position-minor with leading
// dimension ld; slots 0..5 lower, 6 diagonal (inverted), 7..12 upper.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "nks_internal.cuh"

namespace cg = cooperative_groups;

namespace nks {
namespace r2 {

constexpr int kRPC = 32;   // rows per CTA at most (one lane per row)
constexpr int kPF = 98;    // forward chunk row pitch: 6 lower blocks = 96 doubles; 784 B = 16 mod 128
constexpr int kPB = 114;   // backward chunk row pitch: diagonal + 6 upper = 112 doubles; 912 B = 16 mod 128

struct Geo {
  int s0x, s0y;       // global coordinate of local (0,0) (may be negative: wraps)
  int ex, ey;         // extended box size
  int ox0, oy0;       // first owned local index (= delta)
  int ownx, owny;     // owned extent
  int lev_off;        // index into lev_ptr of this box's level 0
  int pad;
};

struct Args {
  const Geo* boxes;
  const int* lev_ptr;
  const double* chunkF;   // [box][stripe][KG][RPC][kPF]
  const double* chunkB;   // [box][stripe][KG][RPC][kPB]
  double* yscr;           // [box][stripe][KG][32][4]
  long long N;
  int nx, ny;
  int CS, RPC, KG, NSW;
  int prof;               // NKS_RAS2D_PROF: per-CTA cycle accounting into g_prof
  int dbg;                // NKS_RAS2D_DBG bits (timing experiments only; results are wrong when set)
  const double* r;
  double* z;
};

// per CTA: [fwd cycles, bwd cycles, halo-wait cycles, stage-wait cycles, start clock (globaltimer), end, 0, 0]
__device__ long long g_prof[1024 * 8];

__device__ __forceinline__ int jmin_of(int t, int ex) { return max(0, (t - ex + 2) >> 1); }
__device__ __forceinline__ unsigned smem_u32(const void* p) { return (unsigned)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_wait(unsigned bar, unsigned parity) {
  unsigned done = 0;
  while (!done)
    asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(done) : "r"(bar), "r"(parity) : "memory");
}
// Halo cells written by a neighbour CTA start as a signalling-NaN sentinel that arithmetic never
// produces; each cell is written exactly once per apply, so the consumer polls the data itself and
// needs no flag, fence or acquire (a cluster-scope release/acquire compiles to MEMBAR.ALL.GPU +
// L1 invalidation, which would wait on this warp's in-flight prefetch loads every time).
constexpr unsigned long long kSentinel = 0x7FF4DEADBEEF0001ull;
__device__ __forceinline__ bool ld_vol4(const double* p, double (&v)[4]) {
  unsigned long long a, b, c, d;
  const unsigned sa = smem_u32(p);
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(sa) : "memory");
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(c), "=l"(d) : "r"(sa + 16) : "memory");
  v[0] = __longlong_as_double((long long)a); v[1] = __longlong_as_double((long long)b);
  v[2] = __longlong_as_double((long long)c); v[3] = __longlong_as_double((long long)d);
  return a != kSentinel && b != kSentinel && c != kSentinel && d != kSentinel;
}
__device__ __forceinline__ void st_remote4(double* local_equiv, unsigned rank, const double (&v)[4]) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("st.relaxed.cluster.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(raddr), "d"(v[0]), "d"(v[1]) : "memory");
  asm volatile("st.relaxed.cluster.shared::cluster.v2.f64 [%0], {%1, %2};" ::"r"(raddr + 16), "d"(v[2]), "d"(v[3])
               : "memory");
}
// predicated variants (no branch in the sweeps)
__device__ __forceinline__ void st_remote4_if(bool pred, double* local_equiv, unsigned rank, const double (&v)[4]) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n"
               " @p st.relaxed.cluster.shared::cluster.v2.f64 [%1], {%2, %3};\n"
               " @p st.relaxed.cluster.shared::cluster.v2.f64 [%4], {%5, %6};\n}\n"
               ::"r"((int)pred), "r"(raddr), "d"(v[0]), "d"(v[1]), "r"(raddr + 16), "d"(v[2]), "d"(v[3])
               : "memory");
}
__device__ __forceinline__ void st_remote4_weak_if(bool pred, double* local_equiv, unsigned rank, const double (&v)[4]) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n"
               " @p st.shared::cluster.v2.f64 [%1], {%2, %3};\n"
               " @p st.shared::cluster.v2.f64 [%4], {%5, %6};\n}\n"
               ::"r"((int)pred), "r"(raddr), "d"(v[0]), "d"(v[1]), "r"(raddr + 16), "d"(v[2]), "d"(v[3])
               : "memory");
}
__device__ __forceinline__ void st_global_if(bool pred, double* p, double v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.global.f64 [%1], %2;\n}\n" ::"r"((int)pred), "l"(p),
               "d"(v)
               : "memory");
}
__device__ __forceinline__ bool ready4(const double* p) {      // no sentinel in the cell (volatile)
  double v[4];
  return ld_vol4(p, v);
}
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}

// acc[c] -= B[c][:] . v  for a row-major 4x4 block B in shared memory.  The 16 entries are loaded
// first and the FMAs issued input-component-outer, so every round is 4 independent DFMAs (chain
// depth 4 per block instead of a serial 16-FMA walk).
__device__ __forceinline__ void blk_sub(const double* B, const double (&v)[4], double (&acc)[4]) {
  double b[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double2 p = *reinterpret_cast<const double2*>(B + c * 4);
    const double2 q = *reinterpret_cast<const double2*>(B + c * 4 + 2);
    b[c][0] = p.x; b[c][1] = p.y; b[c][2] = q.x; b[c][3] = q.y;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < 4; ++c) acc[c] = fma(-b[c][k], v[k], acc[c]);
}

// two blocks into two accumulator sets, interleaved round by round (8 independent DFMAs per round)
__device__ __forceinline__ void blk_sub2(const double* B1, const double (&v1)[4], double (&a1)[4], const double* B2,
                                         const double (&v2)[4], double (&a2)[4]) {
  double b[4][4], e[4][4];
#pragma unroll
  for (int c = 0; c < 4; ++c) {
    const double2 p = *reinterpret_cast<const double2*>(B1 + c * 4);
    const double2 q = *reinterpret_cast<const double2*>(B1 + c * 4 + 2);
    const double2 r = *reinterpret_cast<const double2*>(B2 + c * 4);
    const double2 t = *reinterpret_cast<const double2*>(B2 + c * 4 + 2);
    b[c][0] = p.x; b[c][1] = p.y; b[c][2] = q.x; b[c][3] = q.y;
    e[c][0] = r.x; e[c][1] = r.y; e[c][2] = t.x; e[c][3] = t.y;
  }
#pragma unroll
  for (int k = 0; k < 4; ++k)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      a1[c] = fma(-b[c][k], v1[k], a1[c]);
      a2[c] = fma(-e[c][k], v2[k], a2[c]);
    }
}

// ---------------------------------------------------------------------------------- repack
__global__ void k_pack(Args A, const double* __restrict__ fac, long long ld, int nbox, long long work, double* chunkF,
                       double* chunkB) {
  for (long long w = blockIdx.x * (long long)blockDim.x + threadIdx.x; w < work; w += (long long)gridDim.x * blockDim.x) {
    long long rem = w;
    const int plane = (int)(rem % 208);
    rem /= 208;
    int b = 0;
    for (; b < nbox; ++b) {
      const long long npts = (long long)A.boxes[b].ex * A.boxes[b].ey;
      if (rem < npts) break;
      rem -= npts;
    }
    if (b >= nbox) continue;
    const Geo G = A.boxes[b];
    const int j = (int)(rem / G.ex), i = (int)(rem % G.ex);
    const int t = i + 2 * j;
    const int pos = A.lev_ptr[G.lev_off + t] + (j - jmin_of(t, G.ex));
    int s = 0;
    while (s < A.CS - 1 && j >= ((s + 1) * G.ey) / A.CS) ++s;
    const int rl = j - (s * G.ey) / A.CS;
    const int k = i + 2 * rl;
    const long long row = (((long long)b * A.CS + s) * A.KG + k) * A.RPC + rl;
    const double v = fac[(long long)plane * ld + pos];
    if (plane < 96) chunkF[row * kPF + plane] = v;
    else chunkB[row * kPB + (plane - 96)] = v;
  }
}

// ---------------------------------------------------------------------------------- apply
__global__ void __launch_bounds__(64, 1) k_apply(Args A) {
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int s = (int)cluster.block_rank();
  const int CS = A.CS;
  const int b = blockIdx.x / CS;
  const Geo G = A.boxes[b];
  const int ex = G.ex, ey = G.ey;
  const int r0 = (s * ey) / CS, r1 = ((s + 1) * ey) / CS, R = r1 - r0;
  const int NSW = A.NSW, RPC = A.RPC;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nF = ex + 2 * (R - 1);            // steps per sweep of this stripe
  const int nFp = (nF + 3) & ~3;              // padded to the unroll (the extra steps have no active row)
  const long long cbase = ((long long)b * CS + s) * A.KG;

  // ---- shared memory: [NSW][RPC][kPB] stages | full[NSW] | empty[NSW] | pad[4] | halo rows [4][(ex+4)*4]
  const size_t stage_elems = (size_t)RPC * kPB;
  double* stage = reinterpret_cast<double*>(smem);
  uint64_t* fullb = reinterpret_cast<uint64_t*>(stage + (size_t)NSW * stage_elems);
  uint64_t* emptyb = fullb + NSW;
  const int pitch = (ex + 4) * 4;                      // cells -2 .. ex+1, zero pads
  double* H = reinterpret_cast<double*>(emptyb + NSW) + 2;   // halo rows: 0 = r0-2, 1 = r0-1, 2 = r1, 3 = r1+1
  auto hcell = [&](int q, int i) -> double* { return H + (size_t)q * pitch + (i + 2) * 4; };
  const bool up_remote = s > 0, dn_remote = s < CS - 1;

  // halo rows a neighbour will write start as the sentinel; rows past the box edge (and pads) are 0
  for (int k = tid; k < 4 * pitch; k += blockDim.x) {
    const int q = k / pitch, cell = (k % pitch) / 4 - 2;
    const bool remote = (q < 2 ? up_remote : dn_remote) && cell >= 0 && cell < ex;
    H[k] = remote ? __longlong_as_double((long long)kSentinel) : 0.0;
  }
  if (tid == 0) {
    for (int k = 0; k < NSW; ++k) {
      mbar_init(&fullb[k], 1);
      mbar_init(&emptyb[k], 1);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  cluster.sync();      // halo rows and progress words of every CTA are initialised before neighbours write them

  if (w == 1) {
    // ---- producer: one bulk copy of the active rows of every step, forward then backward
    if (lane == 0) {
      const unsigned full0 = smem_u32(fullb), empty0 = smem_u32(emptyb), stage0 = smem_u32(stage);
      // 2 nFp chunks, then one dummy (the consumer's look-ahead wait past the last step)
      for (int q = 0; q <= 2 * nFp; ++q) {
        const int st = q % NSW, use = q / NSW;
        if (use > 0) mbar_wait(empty0 + st * 8, (unsigned)((use - 1) & 1));
        const bool fw = q < nFp;
        const int k = q == 2 * nFp ? 0 : (fw ? q : 2 * nFp - 1 - q);
        // rows with 0 <= k - 2 rl < ex (one dummy row on the padding steps; KG covers them)
        const int lo = min(R - 1, max(0, (k - ex + 2) / 2)), hi = max(lo, min(R - 1, k / 2));
        const int pf = fw ? kPF : kPB;
        const double* src = (fw ? A.chunkF + (cbase + k) * RPC * kPF : A.chunkB + (cbase + k) * RPC * kPB) + (size_t)lo * pf;
        const unsigned dst = stage0 + (unsigned)((st * stage_elems + (size_t)lo * pf) * 8);
        const unsigned bytes = (unsigned)((hi - lo + 1) * pf * 8);
        const unsigned bar = full0 + st * 8;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
        asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                     "l"(src), "r"(bytes), "r"(bar)
                     : "memory");
      }
    }
  } else {
    // ---- consumer: lane rl = box row r0 + rl
    const int rl = lane;
    const bool row_ok = rl < R;
    const int j = r0 + rl;
    int gy = (G.s0y + j) % A.ny;
    if (gy < 0) gy += A.ny;
    const bool own_row = row_ok && j >= G.oy0 && j < G.oy0 + G.owny;
    const long long N = A.N;
    const double* rrow = A.r + (long long)gy * A.nx;
    double* zrow = A.z + (long long)gy * A.nx;
    double* ybuf = A.yscr + cbase * 128 + rl * 4;    // + k * 128
    const unsigned full0 = smem_u32(fullb);
    int stg = 0;
    unsigned par = 0;
    const unsigned FULL = 0xffffffffu;

    auto gx_of = [&](int i) {          // s0x + i lies in [-delta, nx + delta): one wrap at most
      int gx = G.s0x + i;
      gx += gx < 0 ? A.nx : 0;
      return gx >= A.nx ? gx - A.nx : gx;
    };
    auto load_r = [&](int k, double (&o)[4]) {
      const int i = k - 2 * rl;
      if (row_ok && i >= 0 && i < ex && k < nF && !(A.dbg & 1)) {
        const int gx = gx_of(i);
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = __ldg(rrow + c * N + gx);
      } else {
#pragma unroll
        for (int c = 0; c < 4; ++c) o[c] = 0.0;
      }
    };
    auto hclamp = [&](int q, int cell) -> const double* { return hcell(q, min(max(cell, -2), ex + 1)); };
    long long t_halo = 0, t_stage = 0;
    // poll two halo cells until a neighbour has written both (pads and rows past the box are 0)
    auto poll2 = [&](const double* pa, const double* pb, double (&a)[4], double (&b)[4]) {
      unsigned spins = 0;
      const long long c0 = A.prof ? clock64() : 0;
      while (!(ld_vol4(pa, a) & ld_vol4(pb, b)))
        if (++spins > (1u << 28)) __trap();      // a lost neighbour would otherwise hang the GPU
      if (A.prof) t_halo += clock64() - c0;
    };
    auto wait_stage = [&](int stg_, unsigned par_) {
      const long long c0 = A.prof ? clock64() : 0;
      mbar_wait(full0 + stg_ * 8, par_);
      if (A.prof) t_stage += clock64() - c0;
    };
    const double* const stage_row0 = stage + (size_t)min(rl, RPC - 1) * kPB;   // pitch applied below
    const int rowc = min(rl, RPC - 1);
    // Software pipeline: iteration k finishes step k (only the two lag-1 blocks, the loop-carried
    // chain) and accumulates the four older-neighbour blocks of step k+1, so the issue of one
    // step's bulk work overlaps the latency of the other's chain.
    int stn = 1 % NSW;                 // stage / parity of the next step
    unsigned parn = NSW == 1 ? 1u : 0u;
    auto advance = [&]() {
      stg = stn; par = parn;
      if (++stn == NSW) { stn = 0; parn ^= 1u; }
    };
    (void)stage_row0;
    // wait for the stages of the next four steps (stn and the three after it)
    auto wait_next4 = [&]() {
      int st_ = stn;
      unsigned pa_ = parn;
      const long long c0 = A.prof ? clock64() : 0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        mbar_wait(full0 + st_ * 8, pa_);
        if (++st_ == NSW) { st_ = 0; pa_ ^= 1u; }
      }
      if (A.prof) t_stage += clock64() - c0;
    };
    // release the four stages used by a group (from s0 on)
    auto release4 = [&](int s0) {
      __syncwarp();
      if (lane == 0) {
        int st_ = s0;
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          // relaxed: the stage's shared-memory reads all fed DFMAs issued before (no release fence needed)
          asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(smem_u32(emptyb) + st_ * 8) : "memory");
          if (++st_ == NSW) st_ = 0;
        }
      }
    };

    const long long cf0 = clock64();
    long long gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    // ================================================================ forward sweep (L y = r)
    {
      const bool top = rl == 0;
      double Ya2[4], Ya3[4] = {0, 0, 0, 0}, yp[4] = {0, 0, 0, 0}, pre[4], hA[4];
      double q0[4], q1[4], q2[4], q3[4];                                         // r prefetch ring
      load_r(0, q0); load_r(1, q1); load_r(2, q2); load_r(3, q3);
      {
        // step 0: lane 0's rows above at cells 0 (row r0-1, Ya2) and 0 (row r0-2, aa4); Ya1 = cell 1
        double h0[4], h4[4];
        poll2(hclamp(1, 0), hclamp(0, 0), h0, h4);
        poll2(hclamp(1, 1), hclamp(1, 1), hA, hA);
        double aa4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) { Ya2[c] = top ? h0[c] : 0.0; aa4[c] = top ? h4[c] : 0.0; }
        wait_stage(stg, par);
        const double* L = stage + (size_t)stg * stage_elems + (size_t)rowc * kPF;
        double b0[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) pre[c] = q0[c];
        blk_sub(L + 0 * 16, aa4, pre);   // (0,-2)
        blk_sub(L + 2 * 16, Ya2, b0);    // (0,-1)   [(-1,-1) and (-2,0) are zero at step 0]
#pragma unroll
        for (int c = 0; c < 4; ++c) pre[c] += b0[c];
        load_r(4, q0);
      }
      auto fiter = [&](int k, const double (&rn)[4]) {
        const int i = k - 2 * rl;
        const bool active = row_ok && i >= 0 && i < ex;
        double hAn[4], hBn[4];
        ld4(hclamp(1, k + 2), hAn);        // lane 0's cells for step k+1 (written: checked per group)
        ld4(hclamp(0, k + 1), hBn);
        double Ya1[4], aa4n[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double u = __shfl_up_sync(FULL, yp[c], 1);       // row above, step k-1: (i+1, j-1)
          const double w = __shfl_up_sync(FULL, Ya3[c], 1);      // row j-2 for step k+1
          Ya1[c] = top ? hA[c] : u;
          aa4n[c] = top ? hBn[c] : w;
        }
        // ---- step k: the lag-1 blocks
        const double* L = stage + (size_t)stg * stage_elems + (size_t)rowc * kPF;
        double a0[4], a1[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) a0[c] = pre[c];
        if (!(A.dbg & 16)) blk_sub2(L + 3 * 16, Ya1, a0, L + 5 * 16, yp, a1);   // (1,-1), (-1,0)
        // ---- step k+1: the older blocks (aa4 (0,-2), Ya3 = Ya2_k (-1,-1), Ya2 = Ya1_k (0,-1), Yo2 = y_{k-1} (-2,0))
        const double* Ln = stage + (size_t)stn * stage_elems + (size_t)rowc * kPF;
        double p0[4], p1[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) p0[c] = rn[c];
        if (!(A.dbg & 8)) {
          blk_sub2(Ln + 0 * 16, aa4n, p0, Ln + 1 * 16, Ya2, p1);
          blk_sub2(Ln + 2 * 16, Ya1, p0, Ln + 4 * 16, yp, p1);
        }
        double y[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          y[c] = active ? a0[c] + a1[c] : 0.0;
          pre[c] = p0[c] + p1[c];
          Ya3[c] = Ya2[c]; Ya2[c] = Ya1[c]; yp[c] = y[c]; hA[c] = hAn[c];
        }
        advance();
        if (!(A.dbg & 2)) {
          *reinterpret_cast<double2*>(ybuf + (size_t)k * 128) = make_double2(y[0], y[1]);
          *reinterpret_cast<double2*>(ybuf + (size_t)k * 128 + 2) = make_double2(y[2], y[3]);
        }
        if (A.dbg & 64) st_remote4_weak_if(!(A.dbg & 4) && dn_remote && active && rl >= R - 2,
                      hcell(min(max(rl - (R - 2), 0), 1), min(max(i, 0), ex - 1)), (unsigned)min(s + 1, CS - 1), y);
        else st_remote4_if(!(A.dbg & 4) && dn_remote && active && rl >= R - 2, hcell(min(max(rl - (R - 2), 0), 1), min(max(i, 0), ex - 1)),
                      (unsigned)min(s + 1, CS - 1), y);
      };
      for (int k0 = 0; k0 < nFp; k0 += 4) {
        // once per 4 steps: the stages of steps k0+1..k0+4 are resident and lane 0's halo cells for
        // them are written (one uniform poll loop), so the four steps below are branch-free
        wait_next4();
        {
          unsigned spins = 0;
          const long long c0 = A.prof ? clock64() : 0;
          while (!(A.dbg & 32) && !(ready4(hclamp(1, k0 + 2)) & ready4(hclamp(1, k0 + 3)) & ready4(hclamp(1, k0 + 4)) &
                   ready4(hclamp(1, k0 + 5)) & ready4(hclamp(0, k0 + 1)) & ready4(hclamp(0, k0 + 2)) &
                   ready4(hclamp(0, k0 + 3)) & ready4(hclamp(0, k0 + 4))))
            if (++spins > (1u << 28)) __trap();      // a lost neighbour would otherwise hang the GPU
          if (A.prof) t_halo += clock64() - c0;
        }
        const int s0 = stg;
        fiter(k0, q1); load_r(k0 + 5, q1);
        fiter(k0 + 1, q2); load_r(k0 + 6, q2);
        fiter(k0 + 2, q3); load_r(k0 + 7, q3);
        fiter(k0 + 3, q0); load_r(k0 + 8, q0);
        release4(s0);
      }
    }

    const long long cf1 = clock64();
    // ================================================================ backward sweep (U x = y)
    {
      const bool bot = rl == R - 1;
      const int dR = 2 * (R - 1);       // lane R-1 processes i = k - dR
      double Xb2[4], Xb3[4], xp[4] = {0, 0, 0, 0}, pre[4], hA[4];
      double q0[4], q1[4], q2[4], q3[4];                                         // y prefetch ring
      auto load_y = [&](int k, double (&o)[4]) {
        if (k >= 0) ld4(ybuf + (size_t)k * 128, o);
        else { o[0] = o[1] = o[2] = o[3] = 0.0; }
      };
      load_y(nFp - 1, q0); load_y(nFp - 2, q1); load_y(nFp - 3, q2); load_y(nFp - 4, q3);
      {
        // first step k = nFp-1: lane R-1's rows below at cells i-1 (Xb1), i (Xb2), i+1 (Xb3), row r1+1 cell i
        const int i0 = nFp - 1 - dR;
        double h2[4], h3[4], h4[4];
        poll2(hclamp(2, i0), hclamp(2, i0 + 1), h2, h3);
        poll2(hclamp(3, i0), hclamp(2, i0 - 1), h4, hA);
        double bb4[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) { Xb2[c] = bot ? h2[c] : 0.0; Xb3[c] = bot ? h3[c] : 0.0; bb4[c] = bot ? h4[c] : 0.0; }
        wait_stage(stg, par);
        const double* U = stage + (size_t)stg * stage_elems + (size_t)rowc * kPB;
        double b0[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) pre[c] = q0[c];
        blk_sub(U + 6 * 16, bb4, pre);   // (0,2)
        blk_sub(U + 5 * 16, Xb3, b0);    // (1,1)
        blk_sub(U + 4 * 16, Xb2, pre);   // (0,1)    [(2,0) is zero at the first step]
#pragma unroll
        for (int c = 0; c < 4; ++c) pre[c] += b0[c];
        load_y(nFp - 5, q0);
      }
      auto biter = [&](int k, const double (&yn)[4]) {
        const int i = k - 2 * rl;
        const bool active = row_ok && i >= 0 && i < ex;
        const int iR = k - dR;            // lane R-1's point at step k
        double hAn[4], hBn[4];
        ld4(hclamp(2, iR - 2), hAn);      // lane R-1's cells for step k-1 (written: checked per group)
        ld4(hclamp(3, iR - 1), hBn);
        double Xb1[4], bb4n[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double u = __shfl_down_sync(FULL, xp[c], 1);     // row below, step k+1: (i-1, j+1)
          const double w = __shfl_down_sync(FULL, Xb3[c], 1);    // row j+2 for step k-1
          Xb1[c] = bot ? hA[c] : u;
          bb4n[c] = bot ? hBn[c] : w;
        }
        // ---- step k: the lag-1 blocks, then the inverted diagonal block
        const double* U = stage + (size_t)stg * stage_elems + (size_t)rowc * kPB;
        double a0[4], a1[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) a0[c] = pre[c];
        blk_sub2(U + 3 * 16, Xb1, a0, U + 1 * 16, xp, a1);   // (-1,1), (1,0)
        double v[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) v[c] = a0[c] + a1[c];
        double x[4];
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          const double2 p = *reinterpret_cast<const double2*>(U + c * 4);
          const double2 q = *reinterpret_cast<const double2*>(U + c * 4 + 2);
          x[c] = fma(p.x, v[0], p.y * v[1]) + fma(q.x, v[2], q.y * v[3]);
        }
        // ---- step k-1: the older blocks (bb4 (0,2), Xb3 = Xb2_k (1,1), Xb2 = Xb1_k (0,1), Xo2 = x_{k+1} (2,0))
        const double* Un = stage + (size_t)stn * stage_elems + (size_t)rowc * kPB;
        double p0[4], p1[4] = {0, 0, 0, 0};
#pragma unroll
        for (int c = 0; c < 4; ++c) p0[c] = yn[c];
        blk_sub2(Un + 6 * 16, bb4n, p0, Un + 5 * 16, Xb2, p1);
        blk_sub2(Un + 4 * 16, Xb1, p0, Un + 2 * 16, xp, p1);
#pragma unroll
        for (int c = 0; c < 4; ++c) {
          x[c] = active ? x[c] : 0.0;
          pre[c] = p0[c] + p1[c];
          Xb3[c] = Xb2[c]; Xb2[c] = Xb1[c]; xp[c] = x[c]; hA[c] = hAn[c];
        }
        advance();
        {
          const bool own = active && own_row && i >= G.ox0 && i < G.ox0 + G.ownx;
          double* zp = zrow + gx_of(min(max(i, 0), ex - 1));
#pragma unroll
          for (int c = 0; c < 4; ++c) st_global_if(own, zp + c * N, x[c]);
        }
        st_remote4_if(up_remote && active && rl < 2, hcell(2 + min(rl, 1), min(max(i, 0), ex - 1)), (unsigned)max(s - 1, 0), x);
      };
      // iteration for step k uses y_{k-1}: k = nFp-1-kb; ring q1, q2, q3, q0 holds y_{nFp-2-kb}
      for (int kb0 = 0; kb0 < nFp; kb0 += 4) {
        const int k0 = nFp - 1 - kb0;
        wait_next4();
        {
          const int iR = k0 - dR;
          unsigned spins = 0;
          const long long c0 = A.prof ? clock64() : 0;
          while (!(A.dbg & 32) && !(ready4(hclamp(2, iR - 2)) & ready4(hclamp(2, iR - 3)) & ready4(hclamp(2, iR - 4)) &
                   ready4(hclamp(2, iR - 5)) & ready4(hclamp(3, iR - 1)) & ready4(hclamp(3, iR - 2)) &
                   ready4(hclamp(3, iR - 3)) & ready4(hclamp(3, iR - 4))))
            if (++spins > (1u << 28)) __trap();
          if (A.prof) t_halo += clock64() - c0;
        }
        const int s0 = stg;
        biter(k0, q1); load_y(k0 - 5, q1);
        biter(k0 - 1, q2); load_y(k0 - 6, q2);
        biter(k0 - 2, q3); load_y(k0 - 7, q3);
        biter(k0 - 3, q0); load_y(k0 - 8, q0);
        release4(s0);
      }
    }
    if (A.prof && lane == 0) {
      long long gt1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
      long long* q = g_prof + blockIdx.x * 8;
      q[0] = cf1 - cf0; q[1] = clock64() - cf1; q[2] = t_halo; q[3] = t_stage; q[4] = gt0; q[5] = gt1;
    }
  }
  cluster.sync();      // no CTA leaves while a neighbour may still address its shared memory
}

// ------------------------------------------------------------------------------------------ host
struct Plan {
  int CS = 1, RPC = 32, KG = 1, NSW = 4, nbox = 0, max_clusters = 0;
  size_t smem = 0;
  long long npts_total = 0;
  Args A{};
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

struct Dims {
  int nbox, exmax, eymax, eymin;
};

static bool dims_of(const nks_grid& g, Dims& D) {
  if (g.dim != 2) return false;
  std::vector<int> st[2], ln[2];
  for (int j = 0; j < 2; ++j) split(g.n[j], g.nsub[j], st[j], ln[j]);
  D.nbox = g.nsub[0] * g.nsub[1];
  D.exmax = *std::max_element(ln[0].begin(), ln[0].end()) + 2 * g.overlap;
  D.eymax = *std::max_element(ln[1].begin(), ln[1].end()) + 2 * g.overlap;
  D.eymin = *std::min_element(ln[1].begin(), ln[1].end()) + 2 * g.overlap;
  return true;
}

static int cs_min(const Dims& D) { return (D.eymax + kRPC - 1) / kRPC; }

// cluster sizes this grid admits: every stripe <= 32 rows and >= 2 rows, portable cluster size <= 8
static bool cs_ok(const Dims& D, int CS) { return CS >= cs_min(D) && CS <= 8 && D.eymin / CS >= 2; }

static size_t chunk_bytes(const Dims& D, int CS) {
  const int RPC = (D.eymax + CS - 1) / CS;
  const int KG = D.exmax + 2 * (RPC - 1) + 3;
  const size_t rows = (size_t)D.nbox * CS * KG * RPC;
  const size_t yscr = (size_t)D.nbox * CS * KG * 128;
  return (rows * (kPF + kPB) + yscr) * sizeof(double);
}

size_t workspace_bytes(const nks_grid& g) {
  Dims D;
  if (!dims_of(g, D)) return 0;
  size_t m = 0;
  for (int cs = 1; cs <= 8; ++cs)
    if (cs_ok(D, cs)) m = std::max(m, chunk_bytes(D, cs));
  return m ? m + (size_t)D.nbox * sizeof(Geo) + 1024 : 0;
}

static size_t smem_for(const Dims& D, int RPC, int NSW) {
  return (size_t)NSW * RPC * kPB * 8 + 2 * (size_t)NSW * 8 + 16 + (size_t)4 * (D.exmax + 4) * 4 * 8;
}

void* plan(const nks_grid& g, const BoxSet& B, void* ws, size_t ws_bytes, cudaStream_t stream, std::string& why) {
  Dims D;
  if (!dims_of(g, D)) { why = "not 2D"; return nullptr; }
  if (B.nslots != 13 || B.diag != 6) { why = "unexpected slot table"; return nullptr; }
  if (ws_bytes < workspace_bytes(g) || workspace_bytes(g) == 0) { why = "workspace / geometry"; return nullptr; }
  int dev = 0, maxsm = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&maxsm, cudaDevAttrMaxSharedMemoryPerBlockOptin, dev);
  // The sweep time is the wavefront span (about ex + 2 ey steps) whatever the stripe count, as long
  // as every cluster is resident at once: take the largest admissible CS (<= 8, 2..32 rows per
  // stripe) whose nbox clusters fit in one wave, else the one with the most resident clusters.
  int CS = 0, NSW = 0, ncl = 0;
  size_t smem = 0;
  const char* cs_env = std::getenv("NKS_RAS2D_CS");
  for (int cs = 8; cs >= 1; --cs) {
    if (!cs_ok(D, cs) || (cs_env && cs != std::atoi(cs_env))) continue;
    const int rpc = (D.eymax + cs - 1) / cs;
    int nsw = 12;   // >= 6: a group of 4 steps holds 5 stages
    if (const char* e = std::getenv("NKS_RAS2D_NSW")) nsw = std::max(2, std::atoi(e));
    while (nsw > 6 && smem_for(D, rpc, nsw) > (size_t)maxsm) --nsw;
    const size_t sm = smem_for(D, rpc, nsw);
    if (sm > (size_t)maxsm) continue;
    if (cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.nbox * cs, 1, 1);
    cfg.blockDim = dim3(64, 1, 1);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, k_apply, &cfg) != cudaSuccess) mc = 0;
    cudaGetLastError();
    if (mc < 1) continue;
    if (CS == 0 || (mc >= D.nbox && ncl < D.nbox) || (ncl < D.nbox && mc > ncl)) { CS = cs; NSW = nsw; smem = sm; ncl = mc; }
    if (ncl >= D.nbox) break;
  }
  if (CS == 0) { why = "box height / shared memory / cluster residency"; return nullptr; }
  const int RPC = (D.eymax + CS - 1) / CS;
  Plan* P = new Plan();
  P->CS = CS; P->RPC = RPC; P->KG = D.exmax + 2 * (RPC - 1) + 3; P->NSW = NSW; P->nbox = D.nbox;
  P->smem = smem;
  P->max_clusters = ncl;
  if (cudaFuncSetAttribute(k_apply, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem) != cudaSuccess) {
    cudaGetLastError();
    why = "smem attribute"; delete P; return nullptr;
  }
  std::vector<int> st[2], ln[2];
  for (int j = 0; j < 2; ++j) split(g.n[j], g.nsub[j], st[j], ln[j]);
  std::vector<Geo> geo;
  long long npts = 0;
  for (int by = 0; by < g.nsub[1]; ++by)
    for (int bx = 0; bx < g.nsub[0]; ++bx) {
      Geo q{};
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
  P->npts_total = npts;
  char* w = (char*)ws;
  const size_t rows = (size_t)D.nbox * CS * P->KG * RPC;
  double* cF = (double*)w;
  double* cB = cF + rows * kPF;
  double* ys = cB + rows * kPB;
  Geo* gd = (Geo*)(ys + (size_t)D.nbox * CS * P->KG * 128);
  if (cudaMemcpyAsync(gd, geo.data(), geo.size() * sizeof(Geo), cudaMemcpyHostToDevice, stream) != cudaSuccess) {
    why = "copy"; delete P; return nullptr;
  }
  P->A = Args{gd, B.lev_ptr, cF, cB, ys, (long long)g.n[0] * g.n[1], g.n[0], g.n[1], CS, RPC, P->KG, NSW, 0, 0, nullptr, nullptr};
  if (std::getenv("NKS_DEBUG"))
    std::fprintf(stderr, "[nks] ras2d rows: %d boxes, cluster %d, %d rows/CTA, NSW %d, smem %zu B, max active clusters %d\n",
                 P->nbox, CS, RPC, NSW, P->smem, P->max_clusters);
  return P;
}

void free_plan(void* p) { delete (Plan*)p; }
int cluster_of(void* p) { return p ? ((Plan*)p)->CS : 0; }

void launch_pack(void* plan, const double* fac, long long ld, cudaStream_t s) {
  Plan* P = (Plan*)plan;
  const long long work = P->npts_total * 208;
  const int blocks = (int)std::min<long long>((work + 255) / 256, 148 * 16);
  k_pack<<<blocks, 256, 0, s>>>(P->A, fac, ld, P->nbox, work, const_cast<double*>(P->A.chunkF),
                                const_cast<double*>(P->A.chunkB));
}

cudaError_t launch_apply(void* plan, const double* r, double* z, cudaStream_t s) {
  Plan* P = (Plan*)plan;
  Args A = P->A;
  A.r = r;
  A.z = z;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->nbox * P->CS, 1, 1);
  cfg.blockDim = dim3(64, 1, 1);
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
  cudaError_t e = cudaLaunchKernelEx(&cfg, k_apply, A);
  if (prof && e == cudaSuccess) {
    static int calls = 0;
    if (++calls % 10 == 0) {
      const int nc = P->nbox * P->CS;
      std::vector<long long> h((size_t)nc * 8);
      cudaStreamSynchronize(s);
      cudaMemcpyFromSymbol(h.data(), g_prof, h.size() * 8);
      long long tmin = h[4], tmax = 0;
      for (int c = 0; c < nc; ++c) { tmin = std::min(tmin, h[c * 8 + 4]); tmax = std::max(tmax, h[c * 8 + 5]); }
      std::fprintf(stderr, "[ras2d rows prof] CS %d RPC %d NSW %d, span %lld ns\n", P->CS, P->RPC, P->NSW, tmax - tmin);
      for (int c = 0; c < std::min(nc, 2 * P->CS); ++c)
        std::fprintf(stderr, "  cta %2d (stripe %d): fwd %lld cyc, bwd %lld cyc, halo wait %lld, stage wait %lld, start +%lld ns, "
                     "end +%lld ns\n", c, c % P->CS, h[c * 8], h[c * 8 + 1], h[c * 8 + 2], h[c * 8 + 3], h[c * 8 + 4] - tmin,
                     h[c * 8 + 5] - tmin);
    }
  }
  return e;
}

}  // namespace r2
}  // namespace nks
