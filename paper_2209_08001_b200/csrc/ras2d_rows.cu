// K6 in 2D, second design: the RAS/BILU(0) apply z = sum_i R_i^{0T} (L_i U_i)^{-1} R_i^delta r
// (reading R19) as a row-pipelined wavefront sweep, one lane per box row and one warp per
// field component.
//
// Natural-order BILU(0) on the 13-point block pattern has dependency depth t = i + 2j (reading
// R21): point (i, j) needs y at (i-1,j), (i-2,j) [own row], (i-1,j-1), (i,j-1), (i+1,j-1) [row
// above] and (i,j-2).  Lane rl owns box row j = r0 + rl and processes point i = k - 2 rl at step k,
// so every step of the CTA is one wavefront t = 2 r0 + k.  Warp c computes output component c of
// every row (a quarter of the arithmetic per step: 24 DFMA and 12 16-byte loads of its block rows);
// the four warps exchange each step's 4-vectors through a shared ring E (two planes [4][32][2]) with one named
// barrier per step (the inverted diagonal block is folded into the upper blocks at pack time, so the
// backward sweep has the same shape).
// Only the two lag-1 blocks are on the loop-carried chain: iteration k finishes step k with them and
// accumulates the four older-neighbour blocks of step k+1 (software pipeline).
//
// A box of ey rows is split into CS stripes of <= 32 rows, one CTA each (4 consumer warps + 1
// producer warp), forming a thread-block cluster.  The two rows a stripe needs from the stripe above
// (forward) or below (backward) are stored into its halo rows by the neighbour CTA (DSMEM,
// relaxed); the consumer polls the cells themselves (sentinel-initialised, written once per apply),
// so the sweeps contain no fence.
//
// Factor streaming.  Measured on B200: 1D bulk copies (cp.async.bulk) issued by one SM complete
// one after another with ~540 cycles of fixed cost each (20 KB: 38 B/cycle, 64 KB: 110 B/cycle per
// SM; tools/bulk_probe.cu), so one copy per step would cap the step rate.  The factors are therefore
// repacked once per factorisation into a COMPACT per-stripe stream -- the active rows of step 0, then
// of step 1, ... ([row][plane], blocks row-major, row pitch = 16 mod 128 bytes) -- and the producer
// moves one group of kG = 2 steps per bulk copy into a ring of NS = 4 buffers, off the consumers' step
// barrier (they wait on each group's full mbarrier and release buffers through named barriers); off[k]
// (rows before step k) is a small host-built table.  r is gathered with a register prefetch 4 steps ahead; the forward result
// y goes to a per-step scratch the backward sweep prefetches back; x goes straight to z at the box's
// owned points (R_i^{0T}).  Source factor layout (precond.cu): plane p = slot*16 + row*4 + col,
// position-minor with leading dimension ld; slots 0..5 lower, 6 diagonal (inverted), 7..12 upper.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <ctime>
#include <cstdio>
#include <cstdlib>
#include <string>
#include <vector>

#include "nks_internal.cuh"

namespace cg = cooperative_groups;

namespace nks {
namespace r2 {

constexpr int kRPC = 32;   // rows per CTA at most (one lane per row)
// Stream element type: fp64 factors (default) or fp32 copies (factor_fp32: preconditioner only).
// Row pitches are odd multiples of 16 bytes, so the 16-byte loads of 8 lanes hit distinct banks.
template <bool F32> struct Strm {
  using T = double;
  static constexpr int PF = 98;    // forward: 6 lower blocks = 96 doubles, 784 B
  static constexpr int PB = 114;   // backward: diagonal + 6 upper = 112 doubles, 912 B
#ifndef NKS_R2_G
#define NKS_R2_G 2
#endif
// factor stream transport: 1 = 16-byte cp.async by the producer warp's 32 lanes (requests of one SM overlap),
// 0 = one 1D bulk copy per group (cp.async.bulk; the copies of one SM complete one after another)
#ifndef NKS_R2_LDGSTS
#define NKS_R2_LDGSTS 0      // measured: 1 is 1.5x slower at config 2 (the producer's issue loop sits on the step path)
#endif
#ifndef NKS_R2_NS
#define NKS_R2_NS 4
#endif
// ring release: 1 = named barriers (the consumers' bar.arrive of group g wakes the producer's bar.sync
// on barrier 4 + g % NS: no spinning producer), 0 = empty mbarriers polled by the producer
#ifndef NKS_R2_NBREL
#define NKS_R2_NBREL 1
#endif
#ifndef NKS_R2_UNROLL
#define NKS_R2_UNROLL 4      // steps per loop trip of the sweeps (4 or 8)
#endif
#ifndef NKS_R2_PSLEEP
#define NKS_R2_PSLEEP 256    // producer back-off (ns) while the ring is full
#endif
  static constexpr int G = NKS_R2_G;     // steps per group (one bulk copy)
  static constexpr int NS = NKS_R2_NS;   // group buffers
};
template <> struct Strm<true> {
  using T = float;
  static constexpr int PF = 100;   // 400 B
  static constexpr int PB = 116;   // 464 B
  static constexpr int G = 4;
  static constexpr int NS = 4;
};
constexpr int kGmax = Strm<false>::G > 4 ? Strm<false>::G : 4;

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
  const int* offt;        // [box][stripe][KGp]: rows of the compact stream before step k
  const void* chunkF;     // [box][stripe][RPC*exmax rows][PF] of Strm<F32>::T
  const void* chunkB;     // [box][stripe][RPC*exmax rows][PB]
  double* yscr;           // [box][stripe][KGp][32][4]
  long long N;
  int nx, ny;
  int CS, RPC, KGp, exmax;
  int prof;               // NKS_RAS2D_PROF: per-CTA cycle accounting into g_prof
  int dbg;                // NKS_RAS2D_DBG bits: timing ablations only (results are wrong when set)
  const double* r;
  double* z;
};

// per CTA: [fwd cycles, bwd cycles, halo-wait cycles, stage-wait cycles, start (globaltimer), end, bar wait, 0]
// Ablation switches (NKS_RAS2D_DBG) and clock instrumentation (NKS_RAS2D_PROF) of the apply kernel are
// compiled in only with -DNKS_R2_ABLATE (python -m paper_2209_08001_b200.build with NKS_BUILD_DEFS); the
// production kernel tests constant zeros, which removes their per-step instructions.
#ifdef NKS_R2_ABLATE
#define R2_DBG(A) ((A).dbg)
#define R2_PROF(A) ((A).prof)
#else
#define R2_DBG(A) 0
#define R2_PROF(A) 0
#endif
__device__ long long g_prof[1024 * 8];
__device__ long long g_gt[72 * 8];
__device__ long long g_st[2][5][32][2];   // NKS_RAS2D_PROF: CTA 0, sweep, warp (4 = producer), steps 40..71: barrier arrive / release clocks
__device__ long long g_cp[64 * 4];   // NKS_RAS2D_PROF: CTA 0 producer, groups 8..71: issue / first test / ready clocks   // NKS_RAS2D_PROF: CTA 0, warp 0, forward groups 8..15: per-phase clocks

__device__ __forceinline__ int jmin_of(int t, int ex) { return max(0, (t - ex + 2) >> 1); }
__host__ __device__ __forceinline__ int lo_of(int k, int ex, int R) { return min(R, max(0, (k - ex + 2) / 2)); }
__host__ __device__ __forceinline__ int hi_of(int k, int R) { return min(R - 1, k / 2); }
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
__device__ __forceinline__ bool ready4(const double* p) {
  unsigned long long a, b, c, d;
  const unsigned sa = smem_u32(p);
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(a), "=l"(b) : "r"(sa) : "memory");
  asm volatile("ld.volatile.shared.v2.u64 {%0, %1}, [%2];" : "=l"(c), "=l"(d) : "r"(sa + 16) : "memory");
  return a != kSentinel && b != kSentinel && c != kSentinel && d != kSentinel;
}
__device__ __forceinline__ void ld4(const float* p, double (&v)[4]) {
  const float4 a = *reinterpret_cast<const float4*>(p);
  v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
}
// v <- p[0..3] (shared memory) when on, else unchanged; predicated, so it needs no divergent branch
__device__ __forceinline__ void ld4_shared_if(bool on, const double* p, double (&v)[4]) {
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n @q ld.shared.v2.f64 {%0, %1}, [%5];\n"
               " @q ld.shared.v2.f64 {%2, %3}, [%5+16];\n}\n"
               : "+d"(v[0]), "+d"(v[1]), "+d"(v[2]), "+d"(v[3])
               : "r"((int)on), "r"(smem_u32(p)));
}
__device__ __forceinline__ void ld4_shared_if(bool on, const float* p, double (&v)[4]) {
  float a = 0.f, b = 0.f, c = 0.f, d = 0.f;
  asm volatile("{\n .reg .pred q;\n setp.ne.b32 q, %4, 0;\n @q ld.shared.v4.f32 {%0, %1, %2, %3}, [%5];\n}\n"
               : "+f"(a), "+f"(b), "+f"(c), "+f"(d)
               : "r"((int)on), "r"(smem_u32(p)));
  if (on) { v[0] = a; v[1] = b; v[2] = c; v[3] = d; }
}
__device__ __forceinline__ void ld4(const double* p, double (&v)[4]) {
  const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + 2);
  v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
}
// acc - B[0..3] . v  (one block row, 16-byte aligned)
__device__ __forceinline__ double dot_sub(const double* B, const double (&v)[4], double acc) {
  const double2 p = *reinterpret_cast<const double2*>(B);
  const double2 q = *reinterpret_cast<const double2*>(B + 2);
  acc = fma(-p.x, v[0], acc);
  acc = fma(-p.y, v[1], acc);
  acc = fma(-q.x, v[2], acc);
  return fma(-q.y, v[3], acc);
}
__device__ __forceinline__ void bar_consumers() { asm volatile("bar.sync 1, 128;" ::: "memory"); }
// predicated stores (no branch in the sweeps)
__device__ __forceinline__ void st_remote1_if(bool pred, double* local_equiv, unsigned rank, double v) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.relaxed.cluster.shared::cluster.f64 [%1], %2;\n}\n"
               ::"r"((int)pred), "r"(raddr), "d"(v)
               : "memory");
}
__device__ __forceinline__ unsigned mapa_u32(const void* local_equiv, unsigned rank) {
  unsigned raddr;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(raddr) : "r"(smem_u32(local_equiv)), "r"(rank));
  return raddr;
}
__device__ __forceinline__ void st_cluster_if(bool pred, unsigned raddr, double v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.relaxed.cluster.shared::cluster.f64 [%1], %2;\n}\n"
               ::"r"((int)pred), "r"(raddr), "d"(v)
               : "memory");
}
__device__ __forceinline__ void st_global_if(bool pred, double* p, double v) {
  asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %0, 0;\n @p st.global.f64 [%1], %2;\n}\n" ::"r"((int)pred), "l"(p),
               "d"(v)
               : "memory");
}

// ---------------------------------------------------------------------------------- repack
// One thread per (box point, plane): the point's row in its stripe's compact stream is
// off[k] + (rl - lo(k)), k = i + 2 rl.
template <bool F32>
__global__ void k_pack(Args A, const double* __restrict__ fac, long long ld, int nbox, long long work) {
  using S = Strm<F32>;
  using T = typename S::T;
  T* chunkF = (T*)A.chunkF;
  T* chunkB = (T*)A.chunkB;
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
    const int r0 = (s * G.ey) / A.CS, R = ((s + 1) * G.ey) / A.CS - r0;
    const int rl = j - r0;
    const int k = i + 2 * rl;
    const long long sb = (long long)b * A.CS + s;
    const long long row = sb * A.RPC * A.exmax + A.offt[sb * A.KGp + k] + (rl - lo_of(k, G.ex, R));
    double v;
    if (plane < 112) {
      v = fac[(long long)plane * ld + pos];            // lower blocks; inverted diagonal block D^-1
    } else {
      // upper block U_j folded with the inverted diagonal: (D^-1 U_j)[r][cc] = sum_m D^-1[r][m] U_j[m][cc]
      // (backward sweep x = D^-1 y - sum_j (D^-1 U_j) x_j: one exchange per step, no diagonal solve)
      const int jb = (plane - 96) >> 4, r = (plane >> 2) & 3, cc = plane & 3;
      v = 0.0;
#pragma unroll
      for (int m = 0; m < 4; ++m)
        v = fma(fac[(long long)(96 + r * 4 + m) * ld + pos], fac[(long long)(96 + jb * 16 + m * 4 + cc) * ld + pos], v);
    }
    if (plane < 96) chunkF[row * S::PF + plane] = (T)v;
    else chunkB[row * S::PB + (plane - 96)] = (T)v;
  }
}

// ---------------------------------------------------------------------------------- apply
// (Two alternatives measured in round 1 and removed: block rows read straight from global memory with
// an L2 prefetch by the producer, 0.62 ms; one warp computing all four components with shuffles,
// 0.61 ms -- against 0.337 ms for this kernel at config 2.)
template <bool F32>
__global__ void __launch_bounds__(160, 1) k_apply(Args A) {
  using S = Strm<F32>;
  using T = typename S::T;
  constexpr int kPF = S::PF, kPB = S::PB, kG = S::G, kNSW = S::NS;
  constexpr int NCW = 4;                      // consumer warps; the producer is warp NCW
  extern __shared__ __align__(128) unsigned char smem[];
  cg::cluster_group cluster = cg::this_cluster();
  const int s = (int)cluster.block_rank();
  const int CS = A.CS;
  const int b = blockIdx.x / CS;
  const Geo G = A.boxes[b];
  const int ex = G.ex, ey = G.ey;
  const int r0 = (s * ey) / CS, r1 = ((s + 1) * ey) / CS, R = r1 - r0;
  const int RPC = A.RPC;
  const int tid = threadIdx.x, w = tid >> 5, lane = tid & 31;
  const int nF = ex + 2 * (R - 1);            // steps per sweep of this stripe
  const int nFp = (nF + 4 * kG - 1) / (4 * kG) * (4 * kG);   // whole groups and whole 4-step unrolls
                                                              // (the padding steps have no active row)
  const int nGr = nFp / kG;                   // groups per sweep
  const long long sb = (long long)b * CS + s;
  const int* off_g = A.offt + sb * A.KGp;     // off[0 .. nFp] in global memory (copied to shared below)
  const size_t stage_elems = (size_t)kG * RPC * kPB;
  T* stage = reinterpret_cast<T*>(smem);                               // [kNSW][kG*RPC rows][pitch]
  uint64_t* fullb = reinterpret_cast<uint64_t*>(stage + kNSW * stage_elems);
  uint64_t* emptyb = fullb + kNSW;
  const int pitch = (ex + 4) * 4;
  double* H = reinterpret_cast<double*>(emptyb + kNSW);               // 4 halo rows (16-byte aligned)
  double* E = H + 4 * (size_t)pitch;                                  // [8][32][4] exchange ring
  double* V = E + 8 * 128;                                            // [32][4] (unused since the diagonal fold)
  int4* tb = reinterpret_cast<int4*>(V + 128);                        // per processing step p: stage element
                                                                      // offset of row 0, active rows [lo, hi]
  int* off = reinterpret_cast<int*>(tb + 2 * A.KGp + 8);              // off[] in shared memory: the stage
                                                                      // addresses are on the step's chain
  auto hcell = [&](int q, int i) -> double* { return H + (size_t)q * pitch + (min(max(i, -2), ex + 1) + 2) * 4; };
  const bool up_remote = s > 0, dn_remote = s < CS - 1;

  // halo rows a neighbour will write start as the sentinel; rows past the box edge (and pads) are 0
  for (int k = tid; k < 4 * pitch; k += blockDim.x) {
    const int q = k / pitch, cell = (k % pitch) / 4 - 2;
    const bool remote = (q < 2 ? up_remote : dn_remote) && cell >= 0 && cell < ex;
    H[k] = remote ? __longlong_as_double((long long)kSentinel) : 0.0;
  }
  for (int k = tid; k < 9 * 128; k += blockDim.x) E[k] = 0.0;
  for (int k = tid; k <= nFp; k += blockDim.x) off[k] = off_g[k];
  if (tid == 0) {
    for (int k = 0; k < kNSW; ++k) {
      mbar_init(&fullb[k], NKS_R2_LDGSTS ? 32 : 1);   // LDGSTS: one arrive.noinc per producer lane
      mbar_init(&emptyb[k], NCW);     // one arrive per consumer warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  // Row table: lane rl's block row at processing step p (forward k = p, backward k = 2 nFp - 1 - p) is
  // stage + tb[e].x + rl * pitch when tb[e].y <= rl <= tb[e].z, e = p (forward) or p + 3 (backward), so
  // the per-step preload needs one broadcast shared load instead of the group/offset arithmetic and two
  // off[] loads per row.  Three empty entries after each sweep let the look-ahead (rows of steps k+1..k+3
  // loaded in iteration k) run past its end without range checks.
  for (int e = tid; e < 2 * nFp + 6; e += blockDim.x) {
    const bool pad = (e >= nFp && e < nFp + 3) || e >= 2 * nFp + 3;
    if (pad) { tb[e] = make_int4(0, 1, 0, 0); continue; }
    const int p = e < nFp ? e : e - 3;
    const int k = p < nFp ? p : 2 * nFp - 1 - p;
    const int q = p / kG;
    const int kb = q < nGr ? q * kG : nFp - kG * (q - nGr + 1);
    const int lo = lo_of(k, ex, R), hi = hi_of(k, R);
    const int pf = p < nFp ? kPF : kPB;
    tb[e] = make_int4((int)((q % kNSW) * stage_elems) + (off[k] - off[kb] - lo) * pf, lo, hi, 0);
  }
  __syncthreads();
  cluster.sync();

  // group q (0 .. 2 nGr - 1: forward groups, then backward groups in descending k) covers steps
  // [klo(q), klo(q) + kG); one extra dummy group lets the consumer look one group past the end
  auto klo = [&](int q) { return q < nGr ? q * kG : nFp - kG * (q - nGr + 1); };

  // Step barrier: the 4 consumer warps meet once per step (named barrier 1, 128 threads).  The producer
  // is not on it: each consumer warp waits on a group's full mbarrier itself (probed one step early) and
  // polls the neighbour's halo cells itself (one step ahead), and releases ring buffers with bar.arrive on
  // barrier 4 + g mod NS, on which the producer sleeps.  (Until round 2 the producer was a gatekeeper on
  // every step barrier -- it checked copies and halo cells before arriving -- and arrived last: the step
  // took ~840 cycles, now ~690.)  Barrier 3 (128) orders the E reset between sweeps.
  auto gof = [&](int p) { return p / kG; };   // group of processing step p (forward k = p, backward k = 2 nFp - 1 - p)

  if (w == NCW) {
    // ================================================================ producer (off the step path)
    // The consumers synchronise among themselves (barrier 1, 128 threads), wait on a group's full
    // mbarrier once per group and poll the halo cells themselves one step ahead; the producer only
    // refills the ring: group q goes out as soon as the consumers have released group q - kNSW.
    const unsigned full0 = smem_u32(fullb), empty0 = smem_u32(emptyb), stage0 = smem_u32(stage);
    const long long base = sb * RPC * A.exmax;
    auto issue_one = [&](int q) {
      const bool fw = q < nGr;
      const int k0 = klo(q);
      const int r_lo = off[k0];
      const int nrows = max(1, off[k0 + kG] - r_lo);
      const int pf = fw ? kPF : kPB;
      const int r_src = (R2_DBG(A) & 512) ? 0 : r_lo;     // ablation: every group copies the stream's first rows (L2-resident)
      const T* src = fw ? (const T*)A.chunkF + (base + r_src) * kPF : (const T*)A.chunkB + (base + r_src) * kPB;
      const unsigned bytes = (unsigned)(nrows * pf * sizeof(T));
      const unsigned bar = full0 + (q % kNSW) * 8;
      if (R2_PROF(A) && blockIdx.x == 0 && lane == 0 && q >= 8 && q < 72) g_cp[(q - 8) * 4] = clock64();
      const unsigned dst = stage0 + (unsigned)((q % kNSW) * stage_elems * sizeof(T));
#if NKS_R2_LDGSTS
      // all 32 lanes: 16-byte cp.async (LDGSTS) over the group's contiguous bytes, then one
      // arrive.noinc each, so the full barrier (count 32) completes when every lane's copies have landed
      const char* s8 = reinterpret_cast<const char*>(src);
#pragma unroll 4
      for (unsigned o = (unsigned)lane * 16u; o < bytes; o += 512u)
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(dst + o), "l"(s8 + o) : "memory");
      asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];" ::"r"(bar) : "memory");
#else
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(bar), "r"(bytes) : "memory");
      asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
                   "l"(src), "r"(bytes), "r"(bar)
                   : "memory");
#endif
    };
    // blocking wait on an mbarrier phase (try_wait suspends the thread between checks, so the
    // producer takes few issue slots from consumer warp 0, which shares its sub-partition)
    auto wait_bar = [&](unsigned bar, unsigned par) {
      unsigned sp = 0;
      while (true) {
        unsigned ok;
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2, %3;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(bar), "r"(par), "r"(2000u) : "memory");
        if (__all_sync(0xffffffffu, ok)) break;
        // measured: without a sleep this loop issued ~4x the instructions of a consumer warp on the
        // sub-partition it shares with consumer warp 0 (the try_wait suspend hint does not hold it)
        __nanosleep(NKS_R2_PSLEEP);
        if (++sp > (1u << 24)) __trap();          // a lost consumer would otherwise hang the GPU
      }
    };
    // groups 0 .. 2 nGr - 1 (forward groups, then backward groups in descending k), in order; group q
    // reuses the buffer of group q - kNSW once all four consumer warps have released it
    for (int q = 0; q < 2 * nGr; ++q) {
      if ((R2_DBG(A) & 128) && q >= kNSW) break;   // ablation: no copy management after the first groups
      const int use = q / kNSW;
#if NKS_R2_NBREL
      // Named barrier 4 + (q - NS) % NS completes when the four consumer warps have arrived for group
      // q - NS (bar.arrive: prior shared reads performed) and this warp syncs: the warp sleeps in the
      // barrier instead of polling.  At most NS releases are outstanding (a consumer cannot pass group
      // q - 1 before group q is issued), so NS barrier ids never see two releases at once.
      if (use > 0) {
        asm volatile("bar.sync %0, %1;" ::"r"(4 + (q - kNSW) % kNSW), "n"(32 * (NCW + 1)) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before async-proxy writes
      }
      (void)wait_bar;
#else
      if (use > 0) wait_bar(empty0 + (q % kNSW) * 8, (unsigned)((use - 1) & 1));
#endif
      if (NKS_R2_LDGSTS || lane == 0) issue_one(q);
      __syncwarp();
    }
    (void)full0;
  } else {
    // ================================================================ consumers
    const int c = w;                  // output component of this warp
    const int rl = lane;
    const bool row_ok = rl < R;
    const int j = r0 + rl;
    int gy = (G.s0y + j) % A.ny;
    if (gy < 0) gy += A.ny;
    const bool own_row = row_ok && j >= G.oy0 && j < G.oy0 + G.owny;
    const long long N = A.N;
    const double* rrow = A.r + (long long)c * N + (long long)gy * A.nx;
    double* zrow = A.z + (long long)c * N + (long long)gy * A.nx;
    double* ybuf = A.yscr + sb * A.KGp * 128 + rl * 4 + c;    // + k * 128
    const unsigned empty0 = smem_u32(emptyb);
    auto gx_of = [&](int i) {          // s0x + i lies in [-delta, nx + delta): one wrap at most
      int gx = G.s0x + i;
      gx += gx < 0 ? A.nx : 0;
      return gx >= A.nx ? gx - A.nx : gx;
    };
    // r at (row, i = k - 2 rl): global x = s0x + i wraps at most once; 32-bit index arithmetic and a
    // predicated load keep this off the per-step issue budget
    const int gx0 = G.s0x - 2 * rl, nxg = A.nx;
    const int nFr = row_ok ? nF : 0;              // rows past the stripe load nothing
    auto load_r = [&](int k) -> double {
      const int i = k - 2 * rl;
      if (R2_DBG(A) & 64) return 1e-3 * i;            // ablation: no global loads on the step chain
      const int gi = gx0 + k;
      const int gx = gi < 0 ? gi + nxg : (gi >= nxg ? gi - nxg : gi);
      double v = 0.0;
      if ((unsigned)i < (unsigned)ex && k < nFr) v = __ldg(rrow + gx);
      return v;
    };
    auto release_group = [&](int q) {
      __syncwarp();
#if NKS_R2_NBREL
      // whole warp (bar.arrive is .aligned); the producer syncs on the release of groups
      // 0 .. 2 nGr - 1 - NS only (later groups have no successor in the ring), so the last NS releases
      // are not signalled.  bar.arrive orders this warp's shared reads of the group before the refill.
      (void)empty0;
      if (q < 2 * nGr - kNSW) asm volatile("bar.arrive %0, %1;" ::"r"(4 + q % kNSW), "n"(32 * (NCW + 1)) : "memory");
#else
      // release semantics: this warp's shared-memory reads of the group are ordered before the
      // producer's refill of the buffer (it acquires the empty barrier, then issues the bulk copy)
      if (lane == 0)
        asm volatile("mbarrier.arrive.release.cta.shared::cta.b64 _, [%0];" ::"r"(empty0 + (q % kNSW) * 8) : "memory");
#endif
    };
    const unsigned full0c = smem_u32(fullb);
    // group q's bulk copy has landed (waited once per group by every consumer warp, before the first
    // preload that reads it); try_wait returns at once when the producer is ahead
    auto wait_full = [&](int q) {
      if ((R2_DBG(A) & 128) && q >= kNSW) return;
      const unsigned bar = full0c + (q % kNSW) * 8, par = (unsigned)((q / kNSW) & 1);
      unsigned sp = 0;
      while (true) {
        unsigned ok;
        asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                     : "=r"(ok) : "r"(bar), "r"(par) : "memory");
        if (__all_sync(0xffffffffu, ok)) break;
        if (++sp > (1u << 24)) __trap();
      }
    };
    // Halo polls, one step ahead: lanes 0-3 / 4-7 / 8-31 watch component lane & 3 of the three halo
    // cells the NEXT iteration reads (forward: (1,k+1) (0,k+2) (1,k); backward: (2,iR-1) (2,iR)
    // (3,iR-2)).  A plain load at the end of an iteration, checked by one vote after the next step
    // barrier (slow path: volatile re-reads), so its latency is off the step chain; the stripe pipeline
    // settles one step further behind its neighbour.
    const int pwhich = min(lane >> 2, 2);
    const int pqf = pwhich == 1 ? 0 : 1, pdf = pwhich == 0 ? 1 : (pwhich == 1 ? 2 : 0);
    const int pqb = pwhich == 2 ? 3 : 2, pdb = pwhich == 0 ? -1 : (pwhich == 1 ? 0 : -2);
    auto pload = [&](int q, int i) -> unsigned long long {
      unsigned long long v;
      asm volatile("ld.volatile.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(hcell(q, i) + (lane & 3))) : "memory");
      return v;
    };
    // the speculative poll load at the end of a step is a plain shared load: a volatile one is ordered
    // after this warp's outstanding block-row preloads and waited for them (measured, ncu source page)
    auto pload_plain = [&](int q, int i) -> unsigned long long {
      unsigned long long v;
      asm volatile("ld.shared.u64 %0, [%1];" : "=l"(v) : "r"(smem_u32(hcell(q, i) + (lane & 3))));
      return v;
    };
    // non-blocking probe of a group's full barrier, issued one step before the group is needed (the
    // SYNCS phase check has a long latency; its predicate is consumed after the next step barrier)
    auto test_full = [&](int q) -> bool {
      if ((R2_DBG(A) & 128) && q >= kNSW) return true;
      unsigned ok;
      asm volatile("{\n .reg .pred p;\n mbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
                   : "=r"(ok) : "r"(full0c + (q % kNSW) * 8), "r"((unsigned)((q / kNSW) & 1)));
      return ok != 0;
    };
    auto pcheck = [&](unsigned long long v, int q, int i) {
      unsigned sp = 0;
      while (!__all_sync(0xffffffffu, v != kSentinel)) {
        v = pload(q, i);
        if (++sp > (1u << 26)) __trap();          // a lost neighbour would otherwise hang the GPU
      }
    };
    auto poll3c = [&](int q0_, int c0_, int q1_, int c1_, int q2_, int c2_) {   // blocking, prologues only
      const int qq = pwhich == 0 ? q0_ : (pwhich == 1 ? q1_ : q2_);
      const int cc = pwhich == 0 ? c0_ : (pwhich == 1 ? c1_ : c2_);
      pcheck(pload(qq, cc), qq, cc);
    };
    auto step_bar = [&]() { asm volatile("bar.sync 1, 128;" ::: "memory"); };
    auto step_bar_c = [&](int sw, int k) {        // NKS_RAS2D_PROF: barrier arrive / release clocks
      if (R2_PROF(A) && blockIdx.x == 0 && k >= 40 && k < 72) {
        const long long a = clock64();
        step_bar();
        const long long r = clock64();
        if (lane == 0) { g_st[sw][w][k - 40][0] = a; g_st[sw][w][k - 40][1] = r; }
      } else {
        step_bar();
      }
    };
    auto e_bar = [&]() { asm volatile("bar.sync 3, 128;" ::: "memory"); };
    // this lane's block row c of step k (processing step p) in its group's buffer; nullptr-safe row 0
    auto rowp = [&](int k, int p, int pf) -> const T* {
      const int q = gof(p);
      const int kb = klo(q);
      const int kc = min(max(k, 0), nFp);
      const int lo = lo_of(kc, ex, R), hi = hi_of(kc, R);
      const int rr = (k >= 0 && k < nFp && rl >= lo && rl <= hi) ? off[kc] - off[kb] + (rl - lo) : 0;
      return stage + (size_t)(q % kNSW) * stage_elems + (size_t)rr * pf + c * 4;
    };
    auto ldrow = [&](const T* p, double (&v)[4]) { ld4(p, v); };
    auto zero4 = [&](double (&v)[4]) { v[0] = v[1] = v[2] = v[3] = 0.0; };
    // the block rows of processing step p (0 <= p < 2 nFp) from the row table: lanes without a row at
    // that step skip the shared loads (their outputs of that step are discarded)
    struct RowRef { const T* ptr; bool on; };
    auto rowt = [&](int e, int pf) -> RowRef {      // e: row-table entry (forward p, backward p + 3)
      const int4 t = tb[e];
      return RowRef{stage + t.x + rl * pf + c * 4, rl >= t.y && rl <= t.z};
    };
    // lanes without a row at that step keep stale (finite) values: every output of such a (lane, step)
    // is discarded (y = active ? ... : 0), and no zeroing keeps ~60 selects and moves per step off the
    // issue path
    auto ldrow_if = [&](const RowRef& r, int blk, double (&v)[4]) {
      ld4_shared_if(r.on, r.ptr + blk * 16, v);       // predicated loads: no divergent branch per row
    };
    auto dot4 = [&](const double (&m)[4], const double (&v)[4], double acc) {
      acc = fma(-m[0], v[0], acc);
      acc = fma(-m[1], v[1], acc);
      acc = fma(-m[2], v[2], acc);
      return fma(-m[3], v[3], acc);
    };
    // E holds components (0,1) and (2,3) in two planes [8][32][2] 512 doubles apart, so a lane's two
    // 16-byte loads of a neighbour's 4-vector hit consecutive 16-byte slots (4 wavefronts per warp
    // load instead of 8 with the interleaved [8][32][4] layout); halo cells keep 4 contiguous doubles
    // exchange ring depth: step k's values are written in iteration k and read in iterations k+1, k+2
    // (backward: k-1, k-2), and every warp passes the step barrier of k+1 only after all wrote step k, so
    // 4 slots suffice; with the 4-step unroll the slot of every unrolled iteration is then a compile-time
    // constant (one add from a per-lane base instead of the ring arithmetic)
#ifndef NKS_R2_ESLOTS
#define NKS_R2_ESLOTS 4
#endif
    constexpr int kES = NKS_R2_ESLOTS;
    auto Erow = [&](int k, int row) -> const double* { return E + ((k & (kES - 1)) * 32 + row) * 2; };
    constexpr int kEP = kES * 64;     // plane offset of components (2,3)
    auto ld4s = [&](const double* p, int off2, double (&v)[4]) {
      const double2 a = *reinterpret_cast<const double2*>(p), b = *reinterpret_cast<const double2*>(p + off2);
      v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
    };
    auto Est = [&](int k, double val) { E[(c >> 1) * kEP + ((k & (kES - 1)) * 32 + rl) * 2 + (c & 1)] = val; };
    // the same loads on 32-bit shared addresses: per-lane ring bases, one select between the ring and the
    // halo cell for the boundary lanes (no divergent branch)
    const unsigned sE = smem_u32(E), sH = smem_u32(H);
    // exchange loads: ptxas otherwise sinks some of them below the twelve block-row preloads (register
    // pressure), where they queue behind the preloads and the last DFMAs of the step wait on them (ncu source
    // page); a volatile load stays in program order
#ifndef NKS_R2_VOLX
#define NKS_R2_VOLX 1
#endif
    auto ld4a = [&](unsigned a, unsigned off2, double (&v)[4]) {
#if NKS_R2_VOLX
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a) : "memory");
      asm volatile("ld.volatile.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + off2) : "memory");
#else
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[0]), "=d"(v[1]) : "r"(a) : "memory");
      asm volatile("ld.shared.v2.f64 {%0, %1}, [%2];" : "=d"(v[2]), "=d"(v[3]) : "r"(a + off2) : "memory");
#endif
    };
    auto ering = [&](int k, int row) { return sE + (unsigned)(((k & (kES - 1)) * 32 + row) * 16); };
    auto hcella = [&](int q, int i) { return sH + (unsigned)(q * pitch * 8 + (min(max(i, -2), ex + 1) + 2) * 32); };
    constexpr unsigned kEPB = kEP * 8;    // plane offset in bytes
    long long t_bar = 0, t_stage = 0, t_poll = 0;
    (void)t_bar;

    const long long cf0 = clock64();
    long long gt0;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt0));
    // Two-step look-ahead.  After the barrier of step k, every input of three block pairs is known:
    //   y(k)      = pre(k)    - L3(k).Ya1(k) - L5(k).y(k-1)            (the loop-carried chain)
    //   pre(k+1)  = half(k+1) - L2(k+1).Ya1(k) - L4(k+1).y(k-1)        (Ya2(k+1) = Ya1(k), Yo2(k+1) = y(k-1))
    //   half(k+2) = r(k+2)    - L0(k+2).aa4(k+2) - L1(k+2).Ya1(k)      (Ya3(k+2) = Ya1(k), aa4(k+2) = row j-2 at k-2)
    // The six block rows are loaded into registers during the previous step.
    // ================================================================ forward sweep (L y = r)
    {
      double pre, half;
      // two register sets of block rows: iteration k computes with one while the loads of iteration
      // k + 1's rows into the other are in flight (issued right after its exchange loads, so the next
      // step's exchange loads do not queue behind them)
      struct FRows { double L3[4], L5[4], N2[4], N4[4], M0[4], M1[4]; };
      FRows SA, SB;
      auto preload = [&](FRows& S, int k) {      // rows for iteration k (steps past the sweep: none)
        if (R2_DBG(A) & 32) return;
        { const RowRef r = rowt(k, kPF); ldrow_if(r, 3, S.L3); ldrow_if(r, 5, S.L5); }
        { const RowRef r = rowt(k + 1, kPF); ldrow_if(r, 2, S.N2); ldrow_if(r, 4, S.N4); }
        { const RowRef r = rowt(k + 2, kPF); ldrow_if(r, 0, S.M0); ldrow_if(r, 1, S.M1); }
      };
      for (FRows* S : {&SA, &SB}) { zero4(S->L3); zero4(S->L5); zero4(S->N2); zero4(S->N4); zero4(S->M0); zero4(S->M1); }
      double q0, q1, q2, q3;                       // r prefetch ring: r(k+2) is used at iteration k
      q0 = load_r(2); q1 = load_r(3); q2 = load_r(4); q3 = load_r(5);
      const double r0v = load_r(0), r1v = load_r(1);
      for (int q = 0; q <= gof(2); ++q) wait_full(q);        // groups of steps 0..2 resident
      if (up_remote && !(R2_DBG(A) & 16)) {
        poll3c(1, 0, 0, 0, 0, 1);                            // cells (1,0), (0,0), (0,1) of the prologue
        poll3c(pqf, pdf, pqf, pdf, pqf, pdf);                // cells of iteration 0
      }
      step_bar();
      {
        const bool top = rl == 0;
        double h10[4], h00[4], h01[4], a[4], bb[4];
        ld4(hcell(1, 0), h10);
        ld4(hcell(0, 0), h00);
        ld4(hcell(0, 1), h01);
#pragma unroll
        for (int u = 0; u < 4; ++u) { h10[u] = top ? h10[u] : 0.0; h00[u] = top ? h00[u] : 0.0; h01[u] = top ? h01[u] : 0.0; }
        ldrow(rowp(0, 0, kPF) + 0 * 16, a); ldrow(rowp(0, 0, kPF) + 2 * 16, bb);
        pre = dot4(bb, h10, dot4(a, h00, r0v));        // (0,-2), (0,-1) of step 0
        ldrow(rowp(1, 1, kPF) + 0 * 16, a); ldrow(rowp(1, 1, kPF) + 1 * 16, bb);
        half = dot4(bb, h10, dot4(a, h01, r1v));       // (0,-2), (-1,-1) of step 1
        preload(SA, 0);
      }
      // lanes R-2, R-1 push y into the next stripe's halo rows 0, 1 (cluster address of cell 0, + 32 B per i)
      const bool dn_push = dn_remote && rl >= R - 2 && rl < R;
      const unsigned dn_base = mapa_u32(hcell(min(max(rl - (R - 2), 0), 1), 0) + c, (unsigned)min(s + 1, CS - 1));
      // Control flow inside a step makes the compiler wait for every outstanding load at the branch
      // (the block-row preloads share its few scoreboards), so the step's two checks -- this iteration's
      // halo cells (loaded by the previous iteration) and the full barrier of the group the preload
      // will read -- sit right after the step barrier, where those loads are needed anyway.
      const bool pol = up_remote && !(R2_DBG(A) & 16);
      unsigned long long pvn = 0ull;                 // iteration 0's cells were checked in the prologue
      // half(k+2)'s last two terms (M0[2..3] . aa4[2..3]) are finished after the next step barrier: ptxas
      // sinks the second half of the aa4 load below the block-row preloads, and the step would otherwise
      // end waiting for it (ncu source page); half(k+2) is first read in iteration k+1's pre(k+2)
      double dm2 = 0.0, dm3 = 0.0, da2 = 0.0, da3 = 0.0;
      auto finish_half = [&]() { half = fma(-dm3, da3, fma(-dm2, da2, half)); };
      auto fneed = [&](int k) { return (k + 3) % kG == 0 && k + 3 < nFp; };   // preload of k reads steps k+1..k+3
      bool fok = !fneed(0) || test_full(gof(3));
      auto fiter = [&](int k, double r2, FRows& cur, FRows& nxt) {
        const int i = k - 2 * rl;
        const bool active = row_ok && (unsigned)i < (unsigned)ex;
        step_bar_c(0, k);                                             // E[k-1] complete; stages/cells ready
        // fast path: one vote on the probes issued during the previous step; slow path: blocking waits
        if (!__all_sync(0xffffffffu, fok && (!pol || pvn != kSentinel))) {
          if (pol) pcheck(pvn, pqf, k + pdf);
          if (fneed(k)) wait_full(gof(k + 3));
        }
        double Ya1[4], yp[4], aa4[4];
        ld4a(rl >= 1 ? ering(k - 1, rl - 1) : hcella(1, k + 1), rl >= 1 ? kEPB : 16u, Ya1);   // (i+1, j-1) at step k-1
        ld4a(ering(k - 1, rl), kEPB, yp);                                                     // own row at step k-1
        ld4a(rl >= 2 ? ering(k - 2, rl - 2) : hcella(rl == 1 ? 1 : 0, rl == 1 ? k : k + 2), rl >= 2 ? kEPB : 16u, aa4);
        preload(nxt, k + 1);
        const double a0 = dot4(cur.L3, Ya1, pre);                     // (1,-1)
        const double a1 = dot4(cur.L5, yp, 0.0);                      // (-1,0)
        const double y = active ? a0 + a1 : 0.0;
        Est(k, y);
        finish_half();                                                // half(k+1) complete
        const double b0 = dot4(cur.N2, Ya1, half);                    // pre(k+1): (0,-1)
        const double b1 = dot4(cur.N4, yp, 0.0);                      //           (-2,0)
        const double c0 = fma(-cur.M0[1], aa4[1], fma(-cur.M0[0], aa4[0], r2));   // half(k+2): (0,-2), first half
        const double c1 = dot4(cur.M1, Ya1, 0.0);                     //            (-1,-1)
        pre = b0 + b1;
        half = c0 + c1;
        dm2 = cur.M0[2]; dm3 = cur.M0[3]; da2 = aa4[2]; da3 = aa4[3];
        if (!(R2_DBG(A) & 260)) ybuf[(size_t)k * 128] = y;
        st_cluster_if(!(R2_DBG(A) & 4) && dn_push && active, dn_base + (unsigned)(i * 32), y);
        if (k % kG == kG - 2) release_group(gof(k));   // the group's last rows are in registers now
        if (pol) pvn = pload_plain(pqf, k + 1 + pdf);  // the next iteration's cells (checked after its barrier)
        fok = !fneed(k + 1) || test_full(gof(k + 4));
      };
#if NKS_R2_UNROLL == 8
      // 8 steps per loop trip (nFp is a multiple of 8 with kG = 2): the exchange-ring slots k mod 8 become
      // compile-time offsets
      for (int k0 = 0; k0 < nFp; k0 += 8) {
        fiter(k0, q0, SA, SB); q0 = load_r(k0 + 6);
        fiter(k0 + 1, q1, SB, SA); q1 = load_r(k0 + 7);
        fiter(k0 + 2, q2, SA, SB); q2 = load_r(k0 + 8);
        fiter(k0 + 3, q3, SB, SA); q3 = load_r(k0 + 9);
        fiter(k0 + 4, q0, SA, SB); q0 = load_r(k0 + 10);
        fiter(k0 + 5, q1, SB, SA); q1 = load_r(k0 + 11);
        fiter(k0 + 6, q2, SA, SB); q2 = load_r(k0 + 12);
        fiter(k0 + 7, q3, SB, SA); q3 = load_r(k0 + 13);
      }
#else
      for (int k0 = 0; k0 < nFp; k0 += 4) {
        fiter(k0, q0, SA, SB); q0 = load_r(k0 + 6);
        fiter(k0 + 1, q1, SB, SA); q1 = load_r(k0 + 7);
        fiter(k0 + 2, q2, SA, SB); q2 = load_r(k0 + 8);
        fiter(k0 + 3, q3, SB, SA); q3 = load_r(k0 + 9);
      }
#endif
    }
    const long long cf1 = clock64();
    e_bar();                          // every forward read of E is done: clear it for the backward sweep
    for (int k = tid; k < 8 * 128; k += 128) E[k] = 0.0;
    e_bar();

    // ================================================================ backward sweep (U x = y)
    // With the inverted diagonal folded into the upper blocks at pack time (U'_j = D^-1 U_j,
    // y' = D^-1 y), x = y' - sum_j U'_j x_j has the forward sweep's shape: one exchange per step.
    //   x(k)      = pre(k)    - U'3(k).Xb1(k) - U'1(k).x(k+1)           (chain)
    //   pre(k-1)  = half(k-1) - U'4(k-1).Xb1(k) - U'2(k-1).x(k+1)    (Xb2(k-1) = Xb1(k), Xo2(k-1) = x(k+1))
    //   half(k-2) = y'(k-2)   - U'6(k-2).bb4(k-2) - U'5(k-2).Xb1(k)  (Xb3(k-2) = Xb1(k), bb4(k-2) = row j+2 at k+2)
    // y'(k)_c = (D^-1(k) row c) . y(k), from the forward sweep's y of all four components.
    {
      const int dR = 2 * (R - 1);     // lane R-1 processes i = k - dR
      const int K = nFp - 1;
      auto pofk = [&](int k) { return 2 * nFp - 1 - k; };
      double pre, half;
      struct BRows { double U3[4], U1[4], N4[4], N2[4], M6[4], M5[4], DM[4]; };
      BRows SA, SB;
      auto preload = [&](BRows& S, int k) {      // rows for iteration k (steps past the sweep: none)
        { const RowRef r = rowt(pofk(k) + 3, kPB); ldrow_if(r, 3, S.U3); ldrow_if(r, 1, S.U1); }
        { const RowRef r = rowt(pofk(k - 1) + 3, kPB); ldrow_if(r, 4, S.N4); ldrow_if(r, 2, S.N2); }
        { const RowRef r = rowt(pofk(k - 2) + 3, kPB); ldrow_if(r, 6, S.M6); ldrow_if(r, 5, S.M5); ldrow_if(r, 0, S.DM); }
      };
      for (BRows* S : {&SA, &SB}) { zero4(S->U3); zero4(S->U1); zero4(S->N4); zero4(S->N2); zero4(S->M6); zero4(S->M5); zero4(S->DM); }
      const double* yrow = A.yscr + sb * A.KGp * 128 + rl * 4;    // y(k) of this row: yrow[k * 128 + 0..3]
      auto load_y4 = [&](int k, double (&v)[4]) {
        if (R2_DBG(A) & 64) { v[0] = v[1] = v[2] = v[3] = 1e-3 * k; return; }
        if (k >= 0) {
          const double2 a = *reinterpret_cast<const double2*>(yrow + (size_t)k * 128);
          const double2 b = *reinterpret_cast<const double2*>(yrow + (size_t)k * 128 + 2);
          v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
        } else { zero4(v); }
      };
      auto ydot = [&](const double (&d)[4], const double (&y4)[4]) {   // (D^-1 row c) . y
        return fma(d[3], y4[3], fma(d[2], y4[2], fma(d[1], y4[1], d[0] * y4[0])));
      };
      double q0[4], q1[4], q2[4], q3[4];   // y prefetch ring: y(k-2) is used at iteration k
      load_y4(K - 2, q0); load_y4(K - 3, q1); load_y4(K - 4, q2); load_y4(K - 5, q3);
      double yK[4], yK1[4];
      load_y4(K, yK); load_y4(K - 1, yK1);
      for (int q = gof(nFp); q <= gof(nFp + 2); ++q) wait_full(q);   // first backward groups resident
      if (dn_remote && !(R2_DBG(A) & 16)) {
        const int iR = K - dR;
        poll3c(2, iR, 2, iR + 1, 2, iR + 2);                  // cells of the prologue
        poll3c(3, iR, 3, iR - 1, 2, iR - 1);
        poll3c(pqb, iR + pdb, pqb, iR + pdb, pqb, iR + pdb);   // cells of iteration K
      }
      step_bar();
      {
        const int iR = K - dR;
        const bool bot = rl == R - 1, bot2 = rl == R - 2;
        double h2a[4], h2b[4], h2c[4], h3a[4], h3b[4];
        ld4(hcell(2, iR), h2a);       // Xb2(K) for lane R-1; Xb3(K-1) for lane R-1
        ld4(hcell(2, iR + 1), h2b);   // Xb3(K) for lane R-1; bb4(K-1) for lane R-2
        ld4(hcell(2, iR + 2), h2c);   // bb4(K) for lane R-2
        ld4(hcell(3, iR), h3a);       // bb4(K) for lane R-1
        ld4(hcell(3, iR - 1), h3b);   // bb4(K-1) for lane R-1
        double Xb2[4], Xb3[4], bb4[4], bb4n[4], a[4], bb[4], cc[4], dd[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          Xb2[u] = bot ? h2a[u] : 0.0;
          Xb3[u] = bot ? h2b[u] : 0.0;
          bb4[u] = bot ? h3a[u] : (bot2 ? h2c[u] : 0.0);
          bb4n[u] = bot ? h3b[u] : (bot2 ? h2b[u] : 0.0);
        }
        const T* u = rowp(K, pofk(K), kPB);
        ldrow(u + 6 * 16, a); ldrow(u + 5 * 16, bb); ldrow(u + 4 * 16, cc); ldrow(u, dd);
        pre = dot4(cc, Xb2, dot4(bb, Xb3, dot4(a, bb4, ydot(dd, yK))));     // (0,2), (1,1), (0,1)
        const T* un = rowp(K - 1, pofk(K - 1), kPB);
        ldrow(un + 6 * 16, a); ldrow(un + 5 * 16, bb); ldrow(un, dd);
        half = dot4(bb, Xb2, dot4(a, bb4n, ydot(dd, yK1)));                 // (0,2), (1,1) of step K-1 (Xb3(K-1) = Xb2(K))
        preload(SA, K);
      }
      const int gz0 = G.s0x - 2 * rl;
      // lanes 0, 1 push x into the previous stripe's halo rows 2, 3
      const bool up_push = up_remote && rl < 2;
      const unsigned up_base = mapa_u32(hcell(2 + min(rl, 1), 0) + c, (unsigned)max(s - 1, 0));
      const bool pol = dn_remote && !(R2_DBG(A) & 16);
      unsigned long long pvn = 0ull;                 // iteration K's cells were checked in the prologue
      double dm2 = 0.0, dm3 = 0.0, da2 = 0.0, da3 = 0.0;   // half(k-2)'s deferred terms (see the forward sweep)
      auto finish_half = [&]() { half = fma(-dm3, da3, fma(-dm2, da2, half)); };
      auto bneed = [&](int k) { const int pp = pofk(k) + 3; return pp % kG == 0 && pp < 2 * nFp; };
      bool fok = !bneed(K) || test_full(gof(pofk(K) + 3));
      auto biter = [&](int k, const double (&y2)[4], BRows& cur, BRows& nxt) {
        const int i = k - 2 * rl;
        const bool active = row_ok && (unsigned)i < (unsigned)ex;
        const int iR = k - dR;
        step_bar_c(1, nFp - 1 - k);                                   // E[k+1] complete; stages/cells ready
        if (!__all_sync(0xffffffffu, fok && (!pol || pvn != kSentinel))) {
          if (pol) pcheck(pvn, pqb, iR + pdb);
          if (bneed(k)) wait_full(gof(pofk(k) + 3));                // preload reads pofk(k)+1 .. pofk(k)+3
        }
        double Xb1[4], xp[4], bb4[4];
        ld4a(rl <= R - 2 ? ering(k + 1, rl + 1) : hcella(2, iR - 1), rl <= R - 2 ? kEPB : 16u, Xb1);   // (i-1, j+1) at step k+1
        ld4a(ering(k + 1, rl), kEPB, xp);                                                              // own row at step k+1
        ld4a(rl <= R - 3 ? ering(k + 2, rl + 2) : hcella(rl == R - 2 ? 2 : 3, rl == R - 2 ? iR : iR - 2), rl <= R - 3 ? kEPB : 16u, bb4);
        preload(nxt, k - 1);
        const double a0 = dot4(cur.U3, Xb1, pre);                     // (-1,1)
        const double a1 = dot4(cur.U1, xp, 0.0);                      // (1,0)
        const double x = active ? a0 + a1 : 0.0;
        Est(k, x);
        finish_half();                                                // half(k-1) complete
        const double b0 = dot4(cur.N4, Xb1, half);                    // pre(k-1): (0,1)
        const double b1 = dot4(cur.N2, xp, 0.0);                      //           (2,0)
        const double c0 = fma(-cur.M6[1], bb4[1], fma(-cur.M6[0], bb4[0], ydot(cur.DM, y2)));   // half(k-2): (0,2)
        const double c1 = dot4(cur.M5, Xb1, 0.0);                     //            (1,1)
        pre = b0 + b1;
        half = c0 + c1;
        dm2 = cur.M6[2]; dm3 = cur.M6[3]; da2 = bb4[2]; da3 = bb4[3];
        {
          const int gi = gz0 + k;                  // s0x + i, wraps at most once
          const int gx = gi < 0 ? gi + A.nx : (gi >= A.nx ? gi - A.nx : gi);
          st_global_if(!(R2_DBG(A) & 256) && active && own_row && (unsigned)(i - G.ox0) < (unsigned)G.ownx, zrow + gx, x);
        }
        st_cluster_if(up_push && active, up_base + (unsigned)(i * 32), x);
        const int p = pofk(k);
        if (p % kG == kG - 2) release_group(gof(p));
        if (pol) pvn = pload_plain(pqb, iR - 1 + pdb);  // the next iteration's cells
        fok = !bneed(k - 1) || test_full(gof(pofk(k - 1) + 3));
      };
#if NKS_R2_UNROLL == 8
      for (int kb0 = 0; kb0 < nFp; kb0 += 8) {
        const int k0 = K - kb0;
        biter(k0, q0, SA, SB); load_y4(k0 - 6, q0);
        biter(k0 - 1, q1, SB, SA); load_y4(k0 - 7, q1);
        biter(k0 - 2, q2, SA, SB); load_y4(k0 - 8, q2);
        biter(k0 - 3, q3, SB, SA); load_y4(k0 - 9, q3);
        biter(k0 - 4, q0, SA, SB); load_y4(k0 - 10, q0);
        biter(k0 - 5, q1, SB, SA); load_y4(k0 - 11, q1);
        biter(k0 - 6, q2, SA, SB); load_y4(k0 - 12, q2);
        biter(k0 - 7, q3, SB, SA); load_y4(k0 - 13, q3);
      }
#else
      for (int kb0 = 0; kb0 < nFp; kb0 += 4) {
        const int k0 = K - kb0;
        biter(k0, q0, SA, SB); load_y4(k0 - 6, q0);
        biter(k0 - 1, q1, SB, SA); load_y4(k0 - 7, q1);
        biter(k0 - 2, q2, SA, SB); load_y4(k0 - 8, q2);
        biter(k0 - 3, q3, SB, SA); load_y4(k0 - 9, q3);
      }
#endif
    }
    if (R2_PROF(A) && tid == 0) {
      long long gt1;
      asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(gt1));
      long long* pq = g_prof + blockIdx.x * 8;
      pq[0] = cf1 - cf0; pq[1] = clock64() - cf1; pq[2] = t_poll; pq[3] = t_stage; pq[4] = gt0; pq[5] = gt1; pq[6] = 0;
    }
  }
  // No closing cluster barrier is needed: every DSMEM store targets a halo cell its CTA polls before
  // it can finish, so no CTA exits while a neighbour may still address its shared memory.
  
}


// ------------------------------------------------------------------------------------------ host
struct Plan {
  int CS = 1, RPC = 32, KGp = 1, nbox = 0, max_clusters = 0;
  bool f32 = false;         // fp32 factor stream (factor_fp32)
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

}  // namespace r2
void box_axis(const nks_grid& g, int j, int start, int len, int dl, int& s0, int& e, int& d0);   // precond.cu
namespace r2 {

static bool dims_of(const nks_grid& g, Dims& D) {
  if (g.dim != 2) return false;
  std::vector<int> st[2], ln[2];
  for (int j = 0; j < 2; ++j) split(g.n[j], g.nsub[j], st[j], ln[j]);
  D.nbox = g.nsub[0] * g.nsub[1];
  D.exmax = D.eymax = 0;
  D.eymin = 1 << 30;
  for (int b = 0; b < g.nsub[0]; ++b) {
    int s0, e, d0;
    box_axis(g, 0, st[0][b], ln[0][b], g.overlap, s0, e, d0);
    D.exmax = std::max(D.exmax, e);
  }
  for (int b = 0; b < g.nsub[1]; ++b) {
    int s0, e, d0;
    box_axis(g, 1, st[1][b], ln[1][b], g.overlap, s0, e, d0);
    D.eymax = std::max(D.eymax, e);
    D.eymin = std::min(D.eymin, e);
  }
  return true;
}

static int cs_min(const Dims& D) { return (D.eymax + kRPC - 1) / kRPC; }

// cluster sizes this grid admits: every stripe <= 32 rows and >= 2 rows, portable cluster size <= 8
static int cs_max() {
#ifdef NKS_R2_ABLATE
  // ablation build only (tools/ras2d_step_cost.py): cap the stripes per box
  if (const char* e = std::getenv("NKS_RAS2D_CSMAX")) return std::max(1, std::min(8, std::atoi(e)));
#endif
  return 8;
}
static bool cs_ok(const Dims& D, int CS) { return CS >= cs_min(D) && CS <= cs_max() && D.eymin / CS >= 2; }

static int kgp_of(const Dims& D, int RPC) { return D.exmax + 2 * (RPC - 1) + 4 * kGmax + 1; }

static size_t chunk_bytes(const Dims& D, int CS) {
  const int RPC = (D.eymax + CS - 1) / CS;
  const size_t nsb = (size_t)D.nbox * CS;
  const size_t rows = nsb * RPC * D.exmax;
  const size_t yscr = nsb * kgp_of(D, RPC) * 128;
  return (rows * (Strm<false>::PF + Strm<false>::PB) + yscr) * sizeof(double) + nsb * kgp_of(D, RPC) * sizeof(int) + 256;
}

size_t workspace_bytes(const nks_grid& g) {
  Dims D;
  if (!dims_of(g, D)) return 0;
  size_t m = 0;
  for (int cs = 1; cs <= 16; ++cs)
    if (cs_ok(D, cs)) m = std::max(m, chunk_bytes(D, cs));
  return m ? m + (size_t)D.nbox * sizeof(Geo) + 1024 : 0;
}

static size_t smem_for(const Dims& D, int RPC, bool f32) {
  const size_t stage = f32 ? (size_t)Strm<true>::NS * Strm<true>::G * RPC * Strm<true>::PB * sizeof(float)
                           : (size_t)Strm<false>::NS * Strm<false>::G * RPC * Strm<false>::PB * sizeof(double);
  const int ns = f32 ? Strm<true>::NS : Strm<false>::NS;
  return stage + 2 * (size_t)ns * 8 + (size_t)4 * (D.exmax + 4) * 4 * 8 + (size_t)9 * 128 * 8 + (size_t)kgp_of(D, RPC) * 4 +
         ((size_t)2 * kgp_of(D, RPC) + 8) * 16;
}
// (A per-lane cp.async variant of the apply -- every consumer lane fetching its own block rows with
// LDGSTS, no bulk copies -- measured 0.75 ms against the bulk-copy kernel's 0.52 ms and was removed.)
static const void* apply_fn(bool f32) { return f32 ? (const void*)k_apply<true> : (const void*)k_apply<false>; }
static int apply_threads() { return 160; }
void* plan(const nks_grid& g, const BoxSet& B, void* ws, size_t ws_bytes, cudaStream_t stream, std::string& why, bool f32) {
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
  int CS = 0, ncl = 0;
  size_t smem = 0;
  for (int cs = cs_max(); cs >= 1; --cs) {
    if (!cs_ok(D, cs)) continue;
    if (cs > 8 && cudaFuncSetAttribute(apply_fn(f32), cudaFuncAttributeNonPortableClusterSizeAllowed, 1) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    const int rpc = (D.eymax + cs - 1) / cs;
    const size_t sm = smem_for(D, rpc, f32);
    if (sm > (size_t)maxsm) continue;
    if (cudaFuncSetAttribute(apply_fn(f32), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm) != cudaSuccess) {
      cudaGetLastError();
      continue;
    }
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(D.nbox * cs, 1, 1);
    cfg.blockDim = dim3(apply_threads(), 1, 1);
    cfg.dynamicSmemBytes = sm;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = cs; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
    cfg.attrs = at; cfg.numAttrs = 1;
    int mc = 0;
    if (cudaOccupancyMaxActiveClusters(&mc, apply_fn(f32), &cfg) != cudaSuccess) mc = 0;
    cudaGetLastError();
    if (mc < 1) continue;
    if (CS == 0 || (mc >= D.nbox && ncl < D.nbox) || (ncl < D.nbox && mc > ncl)) { CS = cs; smem = sm; ncl = mc; }
    if (ncl >= D.nbox) break;
  }
  if (CS == 0) { why = "box height / shared memory / cluster residency"; return nullptr; }
  const int RPC = (D.eymax + CS - 1) / CS;
  const int KGp = kgp_of(D, RPC);
  Plan* P = new Plan();
  P->CS = CS; P->RPC = RPC; P->KGp = KGp; P->nbox = D.nbox;
  P->smem = smem;
  P->max_clusters = ncl;
  P->f32 = f32;
  if (cudaFuncSetAttribute(apply_fn(f32), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem) != cudaSuccess) {
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
      box_axis(g, 0, st[0][bx], ln[0][bx], g.overlap, q.s0x, q.ex, q.ox0);
      box_axis(g, 1, st[1][by], ln[1][by], g.overlap, q.s0y, q.ey, q.oy0);
      q.ownx = ln[0][bx];
      q.owny = ln[1][by];
      q.lev_off = B.h_box_lev_off[geo.size()];
      npts += (long long)q.ex * q.ey;
      geo.push_back(q);
    }
  // off[k]: rows of the compact stream before step k, per (box, stripe)
  std::vector<int> offt((size_t)D.nbox * CS * KGp, 0);
  for (int b = 0; b < D.nbox; ++b)
    for (int s = 0; s < CS; ++s) {
      const int ey = geo[b].ey, ex = geo[b].ex;
      const int r0 = (s * ey) / CS, R = ((s + 1) * ey) / CS - r0;
      int* o = &offt[((size_t)b * CS + s) * KGp];
      for (int k = 0; k + 1 < KGp; ++k) o[k + 1] = o[k] + std::max(0, hi_of(k, R) - lo_of(k, ex, R) + 1);
    }
  P->npts_total = npts;
  char* w = (char*)ws;
  const size_t nsb = (size_t)D.nbox * CS;
  const size_t rows = nsb * RPC * D.exmax;
  double* cF = (double*)w;
  double* cB = cF + rows * Strm<false>::PF;     // fp64-sized slots; an fp32 stream uses half of each
  double* ys = cB + rows * Strm<false>::PB;
  int* ot = (int*)(ys + nsb * KGp * 128);
  Geo* gd = (Geo*)((char*)ot + ((nsb * KGp * sizeof(int) + 255) & ~(size_t)255));
  if (cudaMemcpyAsync(gd, geo.data(), geo.size() * sizeof(Geo), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
      cudaMemcpyAsync(ot, offt.data(), offt.size() * sizeof(int), cudaMemcpyHostToDevice, stream) != cudaSuccess ||
      cudaStreamSynchronize(stream) != cudaSuccess) {
    why = "copy"; delete P; return nullptr;
  }
  P->A = Args{gd, B.lev_ptr, ot, cF, cB, ys, (long long)g.n[0] * g.n[1], g.n[0], g.n[1], CS, RPC, KGp, D.exmax, 0, 0,
              nullptr, nullptr};
  if (std::getenv("NKS_DEBUG"))
    std::fprintf(stderr, "[nks] ras2d rows: %d boxes, cluster %d, %d rows/CTA, %s stream, smem %zu B, max active clusters %d\n",
                 P->nbox, CS, RPC, f32 ? "fp32" : "fp64", P->smem, P->max_clusters);
  return P;
}

void free_plan(void* p) { delete (Plan*)p; }
int cluster_of(void* p) { return p ? ((Plan*)p)->CS : 0; }

void launch_pack(void* plan, const double* fac, long long ld, cudaStream_t s) {
  Plan* P = (Plan*)plan;
  const long long work = P->npts_total * 208;
  const int blocks = (int)std::min<long long>((work + 255) / 256, 148 * 16);
  if (P->f32) k_pack<true><<<blocks, 256, 0, s>>>(P->A, fac, ld, P->nbox, work);
  else k_pack<false><<<blocks, 256, 0, s>>>(P->A, fac, ld, P->nbox, work);
}

cudaError_t launch_apply(void* plan, const double* r, double* z, cudaStream_t s) {
  Plan* P = (Plan*)plan;
  Args A = P->A;
  A.r = r;
  A.z = z;
  // The dynamic shared memory limit is an attribute of the kernel function, not of the plan: another
  // state's plan may have lowered it since this plan was made, so it is set before every launch.
  cudaError_t e = cudaFuncSetAttribute(apply_fn(P->f32), cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P->smem);
  if (e != cudaSuccess) return e;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(P->nbox * P->CS, 1, 1);
  cfg.blockDim = dim3(apply_threads(), 1, 1);
  cfg.dynamicSmemBytes = P->smem;
  cfg.stream = s;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension;
  at[0].val.clusterDim.x = P->CS;
  at[0].val.clusterDim.y = 1;
  at[0].val.clusterDim.z = 1;
  cfg.attrs = at;
  cfg.numAttrs = 1;
#ifdef NKS_R2_ABLATE
  // ablation / clock-instrumentation build only (tools/, -DNKS_R2_ABLATE)
  static const bool prof = std::getenv("NKS_RAS2D_PROF") != nullptr;
  A.prof = prof ? 1 : 0;
  A.dbg = std::getenv("NKS_RAS2D_DBG") ? std::atoi(std::getenv("NKS_RAS2D_DBG")) : 0;
#else
  const bool prof = false;
#endif
  e = P->f32 ? cudaLaunchKernelEx(&cfg, k_apply<true>, A) : cudaLaunchKernelEx(&cfg, k_apply<false>, A);
  if (prof && e == cudaSuccess) {
    static int calls = 0;
    if (++calls % 10 == 0) {
      const int nc = P->nbox * P->CS;
      std::vector<long long> h((size_t)nc * 8);
      cudaStreamSynchronize(s);
      cudaMemcpyFromSymbol(h.data(), g_prof, h.size() * 8);
      long long tmin = h[4], tmax = 0;
      for (int c = 0; c < nc; ++c) { tmin = std::min(tmin, h[c * 8 + 4]); tmax = std::max(tmax, h[c * 8 + 5]); }
      std::fprintf(stderr, "[ras2d rows prof] CS %d RPC %d, span %lld ns\n", P->CS, P->RPC, tmax - tmin);
      for (int c = 0; c < std::min(nc, 2 * P->CS); ++c)
        std::fprintf(stderr, "  cta %2d (stripe %d): fwd %lld cyc, bwd %lld cyc, start +%lld ns, end +%lld ns\n", c,
                     c % P->CS, h[c * 8], h[c * 8 + 1], h[c * 8 + 4] - tmin, h[c * 8 + 5] - tmin);
      // CTA 0, steps 40..71 of each sweep: per warp, work = arrive(k) - release(k-1), wait = release(k) - arrive(k)
      std::vector<long long> st(2 * 5 * 32 * 2);
      cudaMemcpyFromSymbol(st.data(), g_st, st.size() * 8);
      auto S = [&](int sw, int w, int k, int x) { return st[((sw * 5 + w) * 32 + k) * 2 + x]; };
      for (int sw = 0; sw < 2; ++sw) {
        std::fprintf(stderr, "  cta 0 %s steps 41..71, cycles per step (mean): ", sw ? "bwd" : "fwd");
        for (int w = 0; w < 5; ++w) {
          double work = 0, wait = 0;
          for (int k = 1; k < 32; ++k) { work += S(sw, w, k, 0) - S(sw, w, k - 1, 1); wait += S(sw, w, k, 1) - S(sw, w, k, 0); }
          std::fprintf(stderr, "%s work %.0f wait %.0f; ", w == 4 ? "producer" : ("warp " + std::to_string(w)).c_str(), work / 31, wait / 31);
        }
        std::fprintf(stderr, "period %.0f\n", (double)(S(sw, 0, 31, 1) - S(sw, 0, 0, 1)) / 31);
        for (int k = 8; k < 12; ++k) {
          std::fprintf(stderr, "    step %d:", 40 + k);
          for (int w = 0; w < 5; ++w)
            std::fprintf(stderr, " w%d arrive %+lld", w, S(sw, w, k, 0) - S(sw, 0, k - 1, 1));
          std::fprintf(stderr, " release %+lld\n", S(sw, 0, k, 1) - S(sw, 0, k - 1, 1));
        }
      }
    }
  }
  return e;
}

}  // namespace r2
}  // namespace nks
