// Internal declarations of the B200 NKS library (not part of the ABI; see include/nks.h).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <array>
#include <string>
#include <vector>

#include "../../include/nks.h"

namespace nks {

constexpr int kMaxDim = 3;
constexpr int kMaxNf = 5;          // 2 + d
constexpr int kMaxSlots = 25;      // |o|_1 <= 2 block footprint in 3D
constexpr int kMaxS = 16;
constexpr int kRedBlocks = 592;    // 4 x 148 SMs: blocks of every reduction first stage
constexpr int kRedThreads = 256;
constexpr int kMaxRanks = 64;      // ranks of one sharded run (all-gather area of the fixed-order reductions)

// Parameters passed by value to every kernel (fp64 model constants derived on the host).
struct DevParams {
  int dim, nx, ny, nz;
  int zg;               // z ghost planes per side (0: periodic in z; >= 2: slab of a z-sharded grid, no z wrap)
  int zoff;             // slab: global z of the first own plane (parity classes of the gauge)
  int nzg;              // slab: global number of planes (0 when not a slab)
  int yg;               // pencil: y ghost rows per side (0: periodic in y, no y split)
  int yoff;             // pencil: global y of the first own row
  int nyg;              // pencil: global number of rows
  int bc;               // 0 periodic, 1 homogeneous Neumann (mirror ghosts, reading R38)
  long long N;          // points
  double h, inv_h2, inv_2h, inv_4h2;
  double dt, inv_dt;
  double theta, gamma_c, gamma_eta, kappa, eps0, C11, C12, C44, Ls, w_c;
  // App. B, derived from L0..L3, U1, U4, dE0:
  // M1(phi) = m1a + m1b phi^2, M2(phi) = m2a + m2b phi^2 + m2c phi^3, M5(c) = m5a c^2 + m5b c^3,
  // M6(c) = m6 c^3.
  double M0, m1a, m1b, m2a, m2b, m2c, M3, M4, m5a, m5b, m6;
  int S;
  double pcoef[kMaxS];  // pcoef[k-1] = 1/(2k(2k+1)), k = 1..S-1 (odd-order Taylor terms)
  double K;             // Ls*(C11 + (d-1) C12): T = K (sum_J D^_J u_J - d eps0 (c - cbar0))
  double cbar0;
};

// Geometry of the RAS boxes (host-built, device-resident).
struct BoxSet {
  int nbox = 0;
  int nslots = 0;            // 13 or 25
  long long P = 0;           // total box positions over all boxes
  long long ld = 0;          // leading dimension of the factor planes (P rounded up to 32)
  int max_levels = 0;
  int max_level_width = 0;
  // device arrays
  int* gidx = nullptr;       // [P] global point index, negative-1-encoded when not owned: ~gidx
  int* nbr = nullptr;        // [nslots][P] neighbour position or -1
  int* box_lev_off = nullptr;   // [nbox+1] offset into lev_ptr
  int* lev_ptr = nullptr;       // concatenated per-box level pointers (absolute positions)
  int* box_pos_off = nullptr;   // [nbox+1]
  int* cover_off = nullptr;     // AS / RRAS: [N+1] CSR of the box positions covering each grid point
  int* cover_pos = nullptr;     // [P] positions, increasing (fixed summation order)
  int variant = 0;              // 0 RAS, 1 AS, 2 RRAS
  int cta_per_box = 0;          // level-synchronous apply: 0 auto, 1, 2, 4 (nks_params.ras_cta_per_box)
  // host copies
  std::vector<int> h_box_lev_off, h_box_pos_off;
  // slot tables (host, copied into kernel params)
  int off[kMaxSlots][3];
  int lower[kMaxSlots];   int nlower = 0;   // lower slots in ascending natural order
  int upper[kMaxSlots];   int nupper = 0;   // strictly upper slots
  int diag = 0;
  // update pairs for the IKJ factorisation: for lower slot index a: pairs (sb, st)
  int npairs[kMaxSlots];
  int pair_b[kMaxSlots][kMaxSlots];
  int pair_t[kMaxSlots][kMaxSlots];
  // level-k ILU (ilu_level != 0): slot tables in device memory (precond_iluk.cuh)
  bool gen = false;
  int g_nlower = 0, g_nupper = 0;
  int* g_off = nullptr;       // [nslots][3]
  int* g_lower = nullptr;
  int* g_upper = nullptr;
  int* g_pair_ptr = nullptr;
  int* g_pair_b = nullptr;
  int* g_pair_t = nullptr;
};

// Level-k ILU pattern (precond_iluk.cuh): slot offsets, lower/upper split, IKJ pairs, wavefront level
// function lx + la ly + lb lz, and per distinct box extent the presence of every (row, slot) entry.
struct IlukPattern {
  int nslots = 0, diag = 0, la = 2, lb = 3;
  std::vector<std::array<int, 3>> off;
  std::vector<int> lower, upper, pair_ptr, pair_b, pair_t;
  std::vector<std::array<int, 3>> ext;                 // distinct box extents
  std::vector<std::vector<unsigned char>> present;     // [extent][local natural index * nslots + slot]
};
IlukPattern build_iluk_pattern(const nks_grid& g, int level);

// Slot tables passed by value to the factor / solve kernels.
struct SlotTables {
  int nslots, nf, diag, nlower, nupper;
  int off[kMaxSlots][3];
  int lower[kMaxSlots];
  int upper[kMaxSlots];
  int npairs[kMaxSlots];
  int pair_b[kMaxSlots][kMaxSlots];
  int pair_t[kMaxSlots][kMaxSlots];
};

// Host-side box tables before upload (precond.cu).
struct HostBoxes {
  std::vector<int> gidx, nbr, box_lev_off, lev_ptr, box_pos_off;
  long long P = 0;
  int max_levels = 0, max_width = 0;
};

}  // namespace nks

struct nks_state {
  nks_grid grid;
  nks_params prm;
  nks::DevParams dp;
  cudaStream_t stream = nullptr;
  int d = 2, nf = 4;
  long long N = 0;          // points
  long long nvec = 0;       // nf * N
  // workspace carve
  char* ws = nullptr;
  size_t ws_bytes = 0;
  double* Xn = nullptr;     // X^n
  double* Xprev = nullptr;  // X^{n-1}
  double* Xb = nullptr;     // Newton iterate
  double* Xt = nullptr;     // line-search trial
  double* S = nullptr;      // Newton direction
  double* F = nullptr;
  double* Ft = nullptr;
  double* Ta = nullptr;     // T^n = tr sigma^el(u^n, c^n)
  double* jac4 = nullptr;   // a11, a12, a21, a22 pointwise partials (4N)
  double* V = nullptr;      // Krylov basis (m+1) * nvec
  double* Z = nullptr;      // preconditioned vector / scratch (nvec)
  double* W2 = nullptr;     // scratch (nvec)
  double* red_part = nullptr;   // reduction partials [kRedBlocks * 64]
  double* red_out = nullptr;    // reduction results [64]
  unsigned* red_cnt = nullptr;  // last-block-done counter of the CGS2 reductions (inside red_out's tail)
  double* h_red = nullptr;      // pinned host mirror [64]
  double* h_ring = nullptr;     // pinned [4][128]: GMRES dot products, one slot per in-flight iteration
  cudaEvent_t gm_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  // preconditioner
  nks::BoxSet boxes;
  double* fac = nullptr;    // [nslots][nf][nf][P]
  float* fac32 = nullptr;   // fp32 copy of fac (factor_fp32), read by the level-synchronous apply
  double* ybox = nullptr;   // [nf][P]
  bool pc_valid = false;
  void* ras2d = nullptr;    // plan of the row-pipelined 2D RAS apply (ras2d_rows.cu), or null
  void* spec = nullptr;     // cuFFT plans of the spectral preconditioner (spectral.cu), or null
  void* specbuf = nullptr;  // [nf][Nh] complex scratch (workspace)
  void* pinv = nullptr;     // [nf*nf][Nh] per-wave-number inverse (workspace)
  double* tl1 = nullptr;    // two-level preconditioner scratch (NKS_PC_RAS_SPECTRAL), or null
  double* tl2 = nullptr;
  double pc_dt = 0.0;
  // history / controller
  double time = 0.0;
  double dt_prev = 0.0;
  double zeta = 0.0;
  bool have_fields = false;
  bool have_prev = false;
  bool debug = false;          // NKS_DEBUG set: per-cycle GMRES trace on stderr
  // z-slab communication (nks_set_comm): null callbacks = not attached
  int rank = 0, nranks = 1;
  nks_allreduce_fn comm_allreduce = nullptr;
  nks_halo_fn comm_halo = nullptr;
  void* comm_user = nullptr;
  bool comm_set = false;
  void* nccl = nullptr;         // library-owned NCCL communicator (comm.cu), or null (callbacks / one state)
  double* gather = nullptr;     // [kMaxRanks][256] all-gather area
  double* ystage = nullptr;     // pencil: packed y blocks of one halo exchange
  // counters
  long long launches = 0;
  long long syncs = 0;
  long long reductions = 0;
  int u0_cg_its = 0;            // CG iterations of the last u^0 solve (0: FFT or given)     // global reductions issued (GMRES: one per Arnoldi step + one per restart)
  // phase profiling (CUDA events on this stream)
  bool profile = false;
  double phase_ms[8] = {0};
  long long phase_cnt[8] = {0};
  std::vector<cudaEvent_t> ev_pool;          // free events
  std::vector<int> pend_phase;                // pending (phase, start, end)
  std::vector<cudaEvent_t> pend_ev;
  int cur_phase = -1;
  cudaEvent_t cur_ev = nullptr;
  std::string err;
};
