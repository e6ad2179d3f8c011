// Host controller and C ABI of the B200 NKS library (include/nks.h).
//
// Newton with the line search of reading R17, restarted right-preconditioned
// GMRES (reading R18) with CGS2 and one host read of <= 2(m+1)+1 doubles per
// iteration, left-RAS/BILU(0) preconditioner, the adaptive controller of
// Eq. (sencondt).  Every arithmetic step runs in the device kernels of stencil.cu,
// krylov.cu, precond.cu and init_fft.cu; this file only sequences them and does O(m^2) Givens
// arithmetic on the <= 64 Hessenberg entries.
#include <cuda_runtime.h>

#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "nks_internal.cuh"

namespace nks {
// stencil.cu
void launch_level_prep(const DevParams& P, const double* X, double* T, cudaStream_t s);
void launch_residual_tiled(const DevParams& P, const double* Xa, const double* Xb, const double* Ta, double* F,
                           cudaStream_t s);
void launch_pointwise_jac(const DevParams& P, const double* Xa, const double* Xb, double* jac4, cudaStream_t s);
void launch_jv_tiled(const DevParams& P, const double* Xa, const double* jac4, const double* v, double* out,
                     cudaStream_t s);
void launch_norm_admissible(long long N, int nf, const double* F, const double* X, double* part, double* out, cudaStream_t s);
void launch_energy(const DevParams& P, const double* X, double* part, double* out, cudaStream_t s);
void launch_gauge(const DevParams& P, double* X, double* part, double* out, cudaStream_t s);
int launch_gauge_sums(const DevParams& P, const double* X, double* part, double* out, cudaStream_t s);
void launch_gauge_apply(const DevParams& P, double* X, const double* out, cudaStream_t s);
void launch_zero_ghosts(const DevParams& P, int nf, double* v, cudaStream_t s);
// krylov.cu
void launch_dcgs_dot(long long n, int nk, const double* V, long long ld, double* part, double* out, unsigned* counter,
                     cudaStream_t s);
void launch_dcgs_dot_u(long long n, int nk, const double* V, long long ld, double* part, double* out, unsigned* counter,
                       cudaStream_t s);
void launch_dcgs_update(long long n, int nk, double* V, long long ld, const double* hv, cudaStream_t s);
void launch_lincomb(long long n, int nk, const double* V, long long ld, const double* y, double* out, cudaStream_t s);
void launch_dot(long long n, const double* a, const double* b, double* part, double* out, cudaStream_t s);
void launch_axpby(long long n, double a, const double* x, double b, double* y, cudaStream_t s);
void launch_xpay(long long n, const double* x, double a, const double* y, double* z, cudaStream_t s);
// precond.cu
void build_slot_tables(int dim, BoxSet& B);
long long box_positions(const nks_grid& g);
HostBoxes build_boxes_host(const nks_grid& g, const BoxSet& B, const IlukPattern* K);
void launch_assemble_gen(const DevParams& P, const BoxSet& B, int nf, const double* Xa, const double* jac4, double* fac,
                         cudaStream_t s);
void launch_factor_gen(const BoxSet& B, int nf, double* fac, cudaStream_t s);
void launch_ras_apply_gen(const BoxSet& B, int nf, long long N, const double* fac, const double* r, double* y,
                          double* z, cudaStream_t s);
void launch_assemble(const DevParams& P, const BoxSet& B, int nf, const double* Xa, const double* jac4, double* fac,
                     cudaStream_t s);
void launch_factor(const BoxSet& B, int nf, double* fac, cudaStream_t s);
void launch_probe_vector(const DevParams& P, int nf, int q0, int q1, int q2, int f, double* v, cudaStream_t s);
void launch_probe_scatter(const DevParams& P, const BoxSet& B, int nf, int q0, int q1, int q2, int f, int first,
                          const double* Jv, double* fac, cudaStream_t s);
namespace r2 {
size_t workspace_bytes(const nks_grid& g);
void* plan(const nks_grid& g, const BoxSet& B, void* ws, size_t ws_bytes, cudaStream_t stream, std::string& why, bool f32);
void free_plan(void* p);
int cluster_of(void* p);
void launch_pack(void* plan, const double* fac, long long ld, cudaStream_t s);
cudaError_t launch_apply(void* plan, const double* r, double* z, cudaStream_t s);
}  // namespace r2
void launch_ras_apply(const BoxSet& B, int nf, long long N, const double* fac, const float* fac32, const double* r,
                      double* y, double* z, cudaStream_t s);
void launch_fac_to_fp32(const BoxSet& B, int nf, const double* fac, float* fac32, cudaStream_t s);
// spectral.cu
long long spectral_half(const nks_grid& g);
void* spectral_plan(const nks_grid& g, int nf, cudaStream_t s, std::string& err);
void spectral_free(void* p);
void launch_spectral_setup(void* plan, const DevParams& dp, int nf, const double* Xa, const double* jac4, double* part,
                           double* means, void* pinv, cudaStream_t s);
int launch_spectral_apply(void* plan, int nf, const double* r, double* z, const void* pinv, void* spec, cudaStream_t s);
// stencil_neumann.cu
void launch_residual_neumann(const DevParams& P, const double* Xa, const double* Xb, const double* Ta, double* F,
                             cudaStream_t s);
void launch_jv_neumann(const DevParams& P, const double* Xa, const double* jac4, const double* v, double* out,
                       cudaStream_t s);
void launch_gauge_neumann(const DevParams& P, double* X, double* part, double* out, cudaStream_t s);
// comm.cu
int slab_decompose(const nks_grid& global, int pc_type, int rank, int nranks, nks_grid& local, int& z_offset);
int nccl_unique_id(uint8_t id[128]);
void halo_plan(int rank, int nranks, int nf, long long fstride, int nzl, long long nxy, int zg,
               std::vector<nks_halo_msg>& out);
void* nccl_create(const uint8_t id[128], int rank, int nranks, std::string& err);
void nccl_destroy(void* c);
int nccl_halo(void* c, double* vec, int nf, long long fstride, int nzl, long long nxy, int zg, cudaStream_t s);
int nccl_allreduce_fixed(void* c, double* buf, long long n, double* gather, cudaStream_t s);
int pencil_decompose(const nks_grid& global, int pc_type, int rank, int pz, int py, nks_grid& local);
void pencil_halo_plan(const nks_grid& g, int rank, int nf, std::vector<nks_halo_msg>& out);
int nccl_halo_pencil(void* c, const nks_grid& g, double* vec, int nf, double* stage, cudaStream_t s);
// init_fft.cu
int init_displacement_fft(const DevParams& P, const double* c, double* u, void* scratch, cudaStream_t s, std::string& err);
}  // namespace nks

using namespace nks;

namespace {

enum Phase { PH_F = 0, PH_JV = 1, PH_RAS = 2, PH_ASM = 3, PH_FACT = 4, PH_VEC = 5, PH_RED = 6, PH_OTHER = 7 };

struct CommError {};   // a communication callback returned non-zero

struct CudaError {
  cudaError_t e;
};

#define CK(call)                                   \
  do {                                             \
    cudaError_t _e = (call);                       \
    if (_e != cudaSuccess) throw CudaError{_e};    \
  } while (0)

struct Layout {
  size_t off_X[7];
  size_t off_Ta, off_jac4, off_V, off_Z, off_W2, off_part, off_out;
  size_t off_fac, off_fac32, off_ybox, off_gidx, off_nbr, off_levoff, off_levptr, off_posoff, off_geo;
  size_t off_cover_off, off_cover_pos;
  size_t off_gather;        // z-slab: [kMaxRanks][256] all-gather area of the fixed-order reductions
  size_t off_ystage;        // pencil: packed y blocks of one halo exchange (4 per field)
  size_t off_gtab;          // level-k ILU slot tables (off, lower, upper, pair_ptr, pair_b, pair_t)
  size_t off_spec, off_pinv;  // spectral preconditioner: [nf][Nh] complex scratch, [nf*nf][Nh] inverse
  size_t off_tl;              // two-level RAS + spectral: 2 scratch vectors
  size_t total;
  long long P, ld;
  size_t geo_bytes;
  int nslots, nbox, nlevptr;
};

size_t align256(size_t x) { return (x + 255) & ~(size_t)255; }

const char* validate(const nks_grid* g, const nks_params* p) {
  if (!g || !p) return "NULL grid or params";
  if (g->dim != 2 && g->dim != 3) return "dim must be 2 or 3";
  for (int j = 0; j < g->dim; ++j)
    if (g->n[j] < 5) return "every n[j] must be >= 5";
  if (g->dim == 2 && g->n[2] != 1) return "n[2] must be 1 in 2D";
  if (!(g->h > 0)) return "h must be > 0";
  if (p->S < 1 || p->S > kMaxS) return "S must be in 1..16";
  if (p->gmres_restart < 1 || p->gmres_restart > 31) return "gmres_restart must be in 1..31";
  if (p->newton_maxit < 0 || p->gmres_maxit < 1 || p->gmres_stall_cycles < 0) return "bad iteration limits";
  if (p->pc_type != NKS_PC_NONE && p->pc_type != NKS_PC_RAS_BILU0 && p->pc_type != NKS_PC_AS_BILU0 &&
      p->pc_type != NKS_PC_RRAS_BILU0 && p->pc_type != NKS_PC_SPECTRAL && p->pc_type != NKS_PC_RAS_SPECTRAL)
    return "unknown pc_type";
  if ((p->pc_type == NKS_PC_SPECTRAL || p->pc_type == NKS_PC_RAS_SPECTRAL) && g->zghost > 0)
    return "the spectral preconditioner needs the whole periodic grid";
  if (g->zghost > 0 && (p->pc_type == NKS_PC_AS_BILU0 || p->pc_type == NKS_PC_RRAS_BILU0))
    return "z-slab states support pc_type NONE or RAS (AS / RRAS need a reverse halo exchange)";
  if (g->zghost != 0 && (g->zghost < 2 || g->zghost > 8)) return "zghost must be 0 or 2..8";
  if (g->bc != 0 && g->bc != 1) return "bc must be 0 (periodic) or 1 (Neumann)";
  if (g->bc == 1 && g->zghost > 0) return "Neumann boundaries: single-GPU states only";
  if (g->bc == 1 && (p->pc_type == NKS_PC_RAS_SPECTRAL || p->ilu_level != 0))
    return "Neumann boundaries: pc_type NONE, SPECTRAL or the Schwarz family with BILU(0) boxes";
  if (g->yghost != 0) {
    if (g->yghost < 2 || g->yghost > 8) return "yghost must be 0 or 2..8";
    if (g->zghost < 2) return "a pencil (yghost > 0) also carries z ghost planes (zghost >= 2)";
    if (p->pc_type != NKS_PC_NONE && p->pc_type != NKS_PC_RAS_BILU0) return "pencil states: pc_type NONE or RAS";
    if (p->pc_type != NKS_PC_NONE && p->ilu_level != 0) return "pencil states: BILU(0) boxes";
    const int owny = g->n[1] - 2 * g->yghost;
    if (owny < 2) return "a pencil must own at least 2 rows";
    if (p->pc_type != NKS_PC_NONE && g->overlap + 1 > g->yghost) return "pencil with RAS needs yghost >= overlap + 1";
    if (p->pc_type != NKS_PC_NONE && (g->nsub[1] < 1 || g->nsub[1] > owny)) return "pencil: nsub[1] must be in 1..own rows";
    if (g->ny_global < 5 || g->y_offset < 0 || g->y_offset + owny > g->ny_global)
      return "pencil: y_offset / ny_global do not place the own rows in the global grid";
    if (g->pz < 1 || g->py < 1) return "pencil: pz, py >= 1";
  }
  if (g->zghost > 0) {
    if (g->dim != 3) return "z-slab states (zghost > 0) are 3D";
    const int own = g->n[2] - 2 * g->zghost;
    if (g->nz_global < 5 || g->z_offset < 0 || g->z_offset + own > g->nz_global)
      return "z-slab: z_offset / nz_global do not place the own planes in the global grid";
    if (g->n[2] - 2 * g->zghost < 2) return "a z-slab must own at least 2 planes";
    if (p->pc_type != NKS_PC_NONE && g->overlap + 1 > g->zghost)
      return "z-slab with RAS needs zghost >= overlap + 1 (assembly reads one cell beyond the box)";
    if (p->pc_type != NKS_PC_NONE && (g->nsub[2] < 1 || g->nsub[2] > g->n[2] - 2 * g->zghost))
      return "z-slab: nsub[2] must be in 1..own planes";
  }
  if (p->pc_type != NKS_PC_NONE && p->pc_type != NKS_PC_SPECTRAL) {
    for (int j = 0; j < 3; ++j)
      if (g->nsub[j] < 1 || g->nsub[j] > g->n[j]) return "nsub[j] must be in 1..n[j]";
    if (g->dim == 2 && g->nsub[2] != 1) return "nsub[2] must be 1 in 2D";
    if (g->overlap < 0 || g->overlap > 8) return "overlap must be in 0..8";
  }
  if (!(p->kappa > 0) || !(p->theta >= 0)) return "kappa must be > 0, theta >= 0";
  if (p->ilu_level < -1 || p->ilu_level > 8) return "ilu_level must be -1 (exact LU) or 0..8";
  if (p->ras_cta_per_box != 0 && p->ras_cta_per_box != 1 && p->ras_cta_per_box != 2 && p->ras_cta_per_box != 4)
    return "ras_cta_per_box must be 0 (auto), 1, 2 or 4";
  if (p->ilu_level != 0 && p->factor_fp32) return "factor_fp32 is available for ILU(0) only";
  if (p->pc_type == NKS_PC_RAS_SPECTRAL && p->ilu_level != 0) return "the two-level preconditioner uses BILU(0) boxes";
  return nullptr;
}

// K: the level-k ILU pattern when p.ilu_level != 0 (built here, handed back to nks_create).
Layout make_layout(const nks_grid& g, const nks_params& p, IlukPattern* K = nullptr) {
  Layout L{};
  IlukPattern Kloc;
  if (p.pc_type != NKS_PC_NONE && p.ilu_level != 0) {
    if (!K) K = &Kloc;
    *K = build_iluk_pattern(g, p.ilu_level);
  }
  const int d = g.dim, nf = 2 + d;
  const long long N = (long long)g.n[0] * g.n[1] * g.n[2];
  const size_t vec = (size_t)nf * N * sizeof(double);
  size_t o = 0;
  for (int k = 0; k < 7; ++k) { L.off_X[k] = o; o = align256(o + vec); }
  L.off_Ta = o; o = align256(o + N * sizeof(double));
  L.off_jac4 = o; o = align256(o + 4 * N * sizeof(double));
  L.off_V = o; o = align256(o + (size_t)(p.gmres_restart + 1) * vec);
  L.off_Z = o; o = align256(o + vec);
  L.off_W2 = o; o = align256(o + vec);
  L.off_part = o; o = align256(o + (size_t)kRedBlocks * 80 * sizeof(double));
  L.off_out = o; o = align256(o + 256 * sizeof(double));
  L.off_gather = o; o = align256(o + (g.zghost > 0 ? (size_t)kMaxRanks * 256 * sizeof(double) : 0));
  L.off_ystage = o;
  if (g.yghost > 0) o = align256(o + (size_t)4 * nf * g.yghost * g.n[0] * (g.n[2] - 2 * g.zghost) * sizeof(double));
  L.P = 0;
  if (p.pc_type == NKS_PC_SPECTRAL || p.pc_type == NKS_PC_RAS_SPECTRAL) {
    const long long Nh = spectral_half(g);
    L.off_spec = o; o = align256(o + (size_t)nf * Nh * 16);
    L.off_pinv = o; o = align256(o + (size_t)nf * nf * Nh * 16);
    if (p.pc_type == NKS_PC_RAS_SPECTRAL) {   // two scratch vectors of the two-level apply
      L.off_tl = o; o = align256(o + 2 * vec);
    }
  }
  if (p.pc_type != NKS_PC_NONE && p.pc_type != NKS_PC_SPECTRAL) {
    const bool gen = p.ilu_level != 0;
    const int nslots = gen ? K->nslots : (d == 2 ? 13 : 25);
    const int la = gen ? K->la : 2, lb = gen ? K->lb : 3;
    L.nslots = nslots;
    L.nbox = g.nsub[0] * g.nsub[1] * g.nsub[2];
    L.P = box_positions(g);
    // upper bound of level pointers: sum over boxes of (nlev + 1)
    long long nl = 0;
    {
      // every box has at most (e0-1)+la(e1-1)+lb(e2-1)+2 entries
      const int ez = d == 3 ? g.overlap * 2 : 0;
      const int e0 = g.n[0] / g.nsub[0] + 1 + 2 * g.overlap, e1 = g.n[1] / g.nsub[1] + 1 + 2 * g.overlap,
                e2 = g.n[2] / g.nsub[2] + 1 + ez;
      nl = (long long)L.nbox * ((e0 - 1) + (long long)la * (e1 - 1) + (long long)lb * (e2 - 1) + 2);
    }
    L.nlevptr = (int)nl;
    L.ld = (L.P + 31) / 32 * 32;
    L.off_fac = o; o = align256(o + (size_t)nslots * nf * nf * L.ld * sizeof(double));
    L.off_fac32 = o; o = align256(o + (p.factor_fp32 ? (size_t)nslots * nf * nf * L.ld * sizeof(float) : 0));
    L.off_ybox = o; o = align256(o + (size_t)nf * L.P * sizeof(double));
    L.off_gidx = o; o = align256(o + (size_t)L.P * sizeof(int));
    L.off_nbr = o; o = align256(o + (size_t)nslots * L.P * sizeof(int));
    L.off_levoff = o; o = align256(o + (size_t)(L.nbox + 1) * sizeof(int));
    L.off_levptr = o; o = align256(o + (size_t)nl * sizeof(int));
    L.off_posoff = o; o = align256(o + (size_t)(L.nbox + 1) * sizeof(int));
    const bool cover = p.pc_type == NKS_PC_AS_BILU0 || p.pc_type == NKS_PC_RRAS_BILU0;
    L.off_cover_off = o; o = align256(o + (cover ? (size_t)(N + 1) * sizeof(int) : 0));
    L.off_cover_pos = o; o = align256(o + (cover ? (size_t)L.P * sizeof(int) : 0));
    // the pipelined 2D apply (ras2d_rows.cu) uses this slice
    L.geo_bytes = (d == 2 && !gen) ? r2::workspace_bytes(g) : 0;
    L.off_geo = o; o = align256(o + L.geo_bytes);
    L.off_gtab = o;
    if (gen) o = align256(o + sizeof(int) * (3 * (size_t)nslots + K->lower.size() + K->upper.size() + K->pair_ptr.size() +
                                             K->pair_b.size() + K->pair_t.size()));
  }
  L.total = o;
  return L;
}

DevParams make_devparams(const nks_grid& g, const nks_params& p) {
  DevParams P{};
  P.dim = g.dim;
  P.nx = g.n[0]; P.ny = g.n[1]; P.nz = g.n[2];
  P.zg = g.zghost;
  P.yg = g.yghost;
  P.bc = g.bc;
  P.N = (long long)g.n[0] * g.n[1] * g.n[2];
  P.h = g.h;
  P.inv_h2 = 1.0 / (g.h * g.h);
  P.inv_2h = 0.5 / g.h;
  P.inv_4h2 = 0.25 / (g.h * g.h);
  P.dt = 1.0; P.inv_dt = 1.0;
  P.theta = p.theta; P.gamma_c = p.gamma_c; P.gamma_eta = p.gamma_eta; P.kappa = p.kappa; P.eps0 = p.eps0;
  P.C11 = p.C11; P.C12 = p.C12; P.C44 = p.C44; P.Ls = p.Lscale; P.w_c = p.w_c;
  // App. B, P:1113-1121 (coefficients already divided by V_m dE)
  P.M0 = p.dE0 + (p.L0 - p.L1 + p.L2 - p.L3);
  P.m1a = -(2.0 * p.L0 - 6.0 * p.L1 + 10.0 * p.L2 - 14.0 * p.L3);
  P.m1b = 24.0 * p.U1 + 72.0 * p.U4;
  P.m2a = -(6.0 * p.L1 - 24.0 * p.L2 + 54.0 * p.L3);
  P.m2b = -216.0 * p.U4;
  P.m2c = -144.0 * p.U4;
  P.M3 = -(16.0 * p.L2 - 80.0 * p.L3);
  P.M4 = -40.0 * p.L3;
  P.m5a = -(24.0 * p.U1 + 72.0 * p.U4);   // M5(c) = -(24 U1 c^2 + 72 U4 (1-2c) c^2)
  P.m5b = 144.0 * p.U4;
  P.m6 = 144.0 * p.U4;                     // M6(c) = 144 U4 c^3
  P.S = p.S;
  for (int k = 1; k < kMaxS + 1; ++k) P.pcoef[k - 1] = (k <= p.S - 1) ? 1.0 / (2.0 * k * (2.0 * k + 1.0)) : 0.0;
  P.K = p.Lscale * (p.C11 + (g.dim - 1) * p.C12);
  P.cbar0 = 0.0;
  return P;
}

// Every group of kernel launches is followed by a launch-error check, so a failed launch (bad
// configuration, shared-memory opt-in missing on this device, ...) becomes NKS_E_CUDA at once instead
// of leaving stale data in its outputs.
void count_launch(nks_state* st, long long n) {
  st->launches += n;
  CK(cudaGetLastError());
}

// ---- phase profiling ---------------------------------------------------------------------------
cudaEvent_t take_event(nks_state* st) {
  if (st->ev_pool.empty()) {
    cudaEvent_t e;
    CK(cudaEventCreate(&e));
    return e;
  }
  cudaEvent_t e = st->ev_pool.back();
  st->ev_pool.pop_back();
  return e;
}

void ph_begin(nks_state* st, int ph) {
  if (!st->profile) return;
  cudaEvent_t e = take_event(st);
  CK(cudaEventRecord(e, st->stream));
  st->cur_phase = ph;
  st->cur_ev = e;
}

void ph_end(nks_state* st) {
  if (!st->profile || st->cur_phase < 0) return;
  cudaEvent_t e = take_event(st);
  CK(cudaEventRecord(e, st->stream));
  st->pend_phase.push_back(st->cur_phase);
  st->pend_ev.push_back(st->cur_ev);
  st->pend_ev.push_back(e);
  st->cur_phase = -1;
  if (st->pend_phase.size() > 20000) {   // drain to bound the pool
    CK(cudaStreamSynchronize(st->stream));
    for (size_t k = 0; k < st->pend_phase.size(); ++k) {
      float ms = 0.f;
      CK(cudaEventElapsedTime(&ms, st->pend_ev[2 * k], st->pend_ev[2 * k + 1]));
      st->phase_ms[st->pend_phase[k]] += ms;
      st->phase_cnt[st->pend_phase[k]] += 1;
      st->ev_pool.push_back(st->pend_ev[2 * k]);
      st->ev_pool.push_back(st->pend_ev[2 * k + 1]);
    }
    st->pend_phase.clear();
    st->pend_ev.clear();
  }
}

struct PhaseScope {
  nks_state* st;
  PhaseScope(nks_state* s, int ph) : st(s) { ph_begin(st, ph); }
  ~PhaseScope() noexcept(false) { ph_end(st); }
};

// ---- building blocks -------------------------------------------------------------------------------
void sync(nks_state* st) {
  CK(cudaStreamSynchronize(st->stream));
  st->syncs++;
}

// ---- z-slab communication ------------------------------------------------------------------------
bool slab(const nks_state* st) { return st->grid.zghost > 0; }
bool pencil(const nks_state* st) { return st->grid.yghost > 0; }

// Points of the whole (global) grid: own planes (and rows) of every rank.
long long global_points(const nks_state* st) {
  if (!slab(st)) return st->N;
  const long long ny = pencil(st) ? (long long)st->dp.nyg : st->grid.n[1];
  const long long nxy = (long long)st->grid.n[0] * ny;
  return st->dp.nzg > 0 ? nxy * st->dp.nzg : nxy * (st->grid.n[2] - 2 * st->grid.zghost);
}

// A global reduction point (counted on every state; an allreduce across ranks on a sharded one).
void comm_allreduce(nks_state* st, double* buf, long long n) {
  st->reductions += 1;
  if (!st->comm_set || st->nranks == 1) return;
  if (st->nccl) {
    if (nccl_allreduce_fixed(st->nccl, buf, n, st->gather, st->stream) != 0) throw CommError();
    return;
  }
  if (st->comm_allreduce(st->comm_user, buf, n, (void*)st->stream) != 0) throw CommError();
}

// Fill the ghost planes of the nf fields of vec (no-op on periodic states).
void halo(nks_state* st, double* vec, int nf) {
  if (!slab(st) || !st->comm_set) return;
  PhaseScope ps(st, PH_OTHER);   // halo exchanges are accounted under "other"
  if (st->nccl) {
    if (pencil(st)) {       // y blocks (packed through the pencil staging area), then whole planes
      if (nccl_halo_pencil(st->nccl, st->grid, vec, nf, st->ystage, st->stream) != 0) throw CommError();
      return;
    }
    const long long nxy = (long long)st->grid.n[0] * st->grid.n[1];
    if (nccl_halo(st->nccl, vec, nf, st->N, st->grid.n[2], nxy, st->grid.zghost, st->stream) != 0) throw CommError();
    return;
  }
  if (st->comm_halo(st->comm_user, vec, nf, st->N, (void*)st->stream) != 0) throw CommError();
}

// Zero the ghost planes of a Krylov-space vector: vectors that enter dot products keep zero ghosts.
void clean(nks_state* st, double* vec, int nf) {
  if (!slab(st)) return;
  launch_zero_ghosts(st->dp, nf, vec, st->stream);
  count_launch(st, 1);
}

void residual(nks_state* st, const double* Xb, double* F) {
  PhaseScope ps(st, PH_F);
  if (st->dp.bc) launch_residual_neumann(st->dp, st->Xn, Xb, st->Ta, F, st->stream);
  else launch_residual_tiled(st->dp, st->Xn, Xb, st->Ta, F, st->stream);
  count_launch(st, 1);
}

// (||F||, #inadmissible points of X) -- host sync
void norm_adm(nks_state* st, const double* F, const double* X, double& nrm, double& bad) {
  {
    PhaseScope ps(st, PH_RED);
    launch_norm_admissible(st->N, st->nf, F, X, st->red_part, st->red_out, st->stream);
    count_launch(st, 2);
  }
  comm_allreduce(st, st->red_out, 2);
  CK(cudaMemcpyAsync(st->h_red, st->red_out, 2 * sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  sync(st);
  nrm = std::sqrt(st->h_red[0]);
  bad = st->h_red[1];
}

void gauge(nks_state* st, double* X) {
  PhaseScope ps(st, PH_RED);
  if (st->dp.bc) {          // Neumann (single state): translations + discrete rotations (reading R38)
    launch_gauge_neumann(st->dp, X, st->red_part, st->red_out + 128, st->stream);
    comm_allreduce(st, st->red_out + 128, 0);
    count_launch(st, 3);
    return;
  }
  const int nsum = launch_gauge_sums(st->dp, X, st->red_part, st->red_out + 128, st->stream);
  comm_allreduce(st, st->red_out + 128, nsum);     // global sub-lattice sums (slab: own planes of every rank)
  launch_gauge_apply(st->dp, X, st->red_out + 128, st->stream);
  count_launch(st, 3);
}

void jv(nks_state* st, const double* v, double* out) {
  PhaseScope ps(st, PH_JV);
  if (st->dp.bc) launch_jv_neumann(st->dp, st->Xn, st->jac4, v, out, st->stream);
  else launch_jv_tiled(st->dp, st->Xn, st->jac4, v, out, st->stream);
  count_launch(st, 1);
}

void pc_apply(nks_state* st, const double* r, double* z) {
  if (st->prm.pc_type == NKS_PC_NONE) {
    CK(cudaMemcpyAsync(z, r, st->nvec * sizeof(double), cudaMemcpyDeviceToDevice, st->stream));
    return;
  }
  if (st->tl1) {
    // two-level (NKS_PC_RAS_SPECTRAL): global spectral correction, then RAS on the remaining residual
    //   z1 = S r,  t = r - J z1,  z = z1 + RAS(t)
    {
      PhaseScope ps(st, PH_RAS);
      if (launch_spectral_apply(st->spec, st->nf, r, st->tl1, st->pinv, st->specbuf, st->stream) != 0)
        throw std::runtime_error("cuFFT execution failed");
      count_launch(st, 1);
    }
    jv(st, st->tl1, st->tl2);
    {
      PhaseScope ps(st, PH_VEC);
      launch_xpay(st->nvec, r, -1.0, st->tl2, st->tl2, st->stream);
      count_launch(st, 1);
    }
    {
      PhaseScope ps(st, PH_RAS);
      if (st->ras2d) CK(r2::launch_apply(st->ras2d, st->tl2, z, st->stream));
      else launch_ras_apply(st->boxes, st->nf, st->N, st->fac, st->fac32, st->tl2, st->ybox, z, st->stream);
      count_launch(st, 1);
    }
    PhaseScope ps(st, PH_VEC);
    launch_axpby(st->nvec, 1.0, st->tl1, 1.0, z, st->stream);
    count_launch(st, 1);
    return;
  }
  PhaseScope ps(st, PH_RAS);
  if (st->spec) {
    if (launch_spectral_apply(st->spec, st->nf, r, z, st->pinv, st->specbuf, st->stream) != 0)
      throw std::runtime_error("cuFFT execution failed");
    count_launch(st, 1);
    return;
  }
  if (st->ras2d) CK(r2::launch_apply(st->ras2d, r, z, st->stream));
  else if (st->boxes.gen) launch_ras_apply_gen(st->boxes, st->nf, st->N, st->fac, r, st->ybox, z, st->stream);
  else launch_ras_apply(st->boxes, st->nf, st->N, st->fac, st->fac32, r, st->ybox, z, st->stream);
  count_launch(st, 1);
}

void pc_setup(nks_state* st, const double* Xb) {
  if (st->prm.pc_type == NKS_PC_NONE) return;
  if (st->spec) {
    PhaseScope ps(st, PH_FACT);
    launch_spectral_setup(st->spec, st->dp, st->nf, st->Xn, st->jac4, st->red_part, st->red_out + 192, st->pinv,
                          st->stream);
    count_launch(st, 3);
    if (!st->tl1) {
      st->pc_valid = true;
      st->pc_dt = st->dp.dt;
      return;
    }
  }
  if (st->dp.bc) {
    // Neumann (R38): the box blocks by probing J with 5^d colours x nf unit fields (precond.cu)
    const int nq2 = st->d == 3 ? 5 : 1;
    int first = 1;
    for (int f = 0; f < st->nf; ++f)
      for (int q2 = 0; q2 < nq2; ++q2)
        for (int q1 = 0; q1 < 5; ++q1)
          for (int q0 = 0; q0 < 5; ++q0) {
            {
              PhaseScope ps(st, PH_ASM);
              launch_probe_vector(st->dp, st->nf, q0, q1, q2, f, st->W2, st->stream);
              count_launch(st, 1);
            }
            jv(st, st->W2, st->Z);
            PhaseScope ps(st, PH_ASM);
            launch_probe_scatter(st->dp, st->boxes, st->nf, q0, q1, q2, f, first, st->Z, st->fac, st->stream);
            count_launch(st, 1);
            first = 0;
          }
  } else {
    PhaseScope ps(st, PH_ASM);
    if (st->boxes.gen) launch_assemble_gen(st->dp, st->boxes, st->nf, st->Xn, st->jac4, st->fac, st->stream);
    else launch_assemble(st->dp, st->boxes, st->nf, st->Xn, st->jac4, st->fac, st->stream);
    count_launch(st, 1);
  }
  {
    PhaseScope ps(st, PH_FACT);
    if (st->boxes.gen) launch_factor_gen(st->boxes, st->nf, st->fac, st->stream);
    else launch_factor(st->boxes, st->nf, st->fac, st->stream);
    count_launch(st, 1);
    if (st->ras2d) {
      r2::launch_pack(st->ras2d, st->fac, st->boxes.ld, st->stream);
      count_launch(st, 1);
    }
    if (st->fac32 && !st->ras2d) {
      launch_fac_to_fp32(st->boxes, st->nf, st->fac, st->fac32, st->stream);
      count_launch(st, 1);
    }
  }
  (void)Xb;
  st->pc_valid = true;
  st->pc_dt = st->dp.dt;
}

void set_dt(nks_state* st, double dt) {
  st->dp.dt = dt;
  st->dp.inv_dt = 1.0 / dt;
}

// Right-preconditioned restarted GMRES: J s = b with s0 = 0 (reading R18).  Returns 0
// converged, 1 gmres_maxit, 2 stagnation (opt-in), 3 projected past gmres_maxit (opt-in).
//
// Arnoldi by DCGS2 (krylov.cu): ONE global reduction per iteration (a = V^T u, b = V^T w, u.u, u.w in one
// fused pass, one allreduce on a slab state), one fused update pass.  Column j-1 of the Hessenberg matrix
// becomes final when iteration j's reduction arrives (the delayed reorthogonalisation), so the host's
// Givens / convergence test runs one column behind the device; with the one-iteration look-ahead the
// device never waits for the host.  The device computes r and gamma of every step itself (dcgs_scalars),
// the host replays the same doubles from a pinned copy (ring of 4 slots).
int gmres(nks_state* st, const double* b, double bnorm, double* s, double tol, int& its) {
  const int m = st->prm.gmres_restart;
  const long long n = st->nvec;
  double* V = st->V;
  std::vector<double> Hr((m + 1) * m, 0.0), R((m + 1) * m, 0.0), cs(m, 0.0), sn(m, 0.0), g(m + 1, 0.0), y(m, 0.0),
      hprev(m + 1, 0.0), hnew(m + 1, 0.0);
  CK(cudaMemsetAsync(s, 0, n * sizeof(double), st->stream));
  its = 0;
  double beta = bnorm;
  bool first = true;
  int stall = 0;
  constexpr int kProjWin = 5;                 // restart cycles in the projection's rate window
  std::vector<double> hist(1, bnorm);         // true residual at the start of every cycle
  std::vector<int> hits(1, 0);                // ... and the iterations done before it
  while (true) {
    if (beta <= tol) return 0;
    {
      PhaseScope ps(st, PH_VEC);
      launch_axpby(n, 1.0 / beta, first ? b : V, 0.0, V, st->stream);
      count_launch(st, 1);
    }
    first = false;
    std::fill(Hr.begin(), Hr.end(), 0.0);
    std::fill(R.begin(), R.end(), 0.0);
    std::fill(g.begin(), g.end(), 0.0);
    // one reduction (+ allreduce) per launched step, its values copied to ring slot jj % 4
    auto reduce_to_ring = [&](int jj) {
      comm_allreduce(st, st->red_out, 66);
      double* slot = st->h_ring + (jj % 4) * 128;
      CK(cudaMemcpyAsync(slot, st->red_out, 66 * sizeof(double), cudaMemcpyDeviceToHost, st->stream));
      CK(cudaEventRecord(st->gm_ev[jj % 4], st->stream));
    };
    auto launch_iter = [&](int jj) {            // u = V[jj] -> w = J M^-1 u into V[jj+1], then DCGS2 step jj
      double* u = V + (long long)jj * n;
      double* w = V + (long long)(jj + 1) * n;
      if (st->prm.pc_type != NKS_PC_NONE) halo(st, u, st->nf);   // RAS reads delta ghost planes of its input
      pc_apply(st, u, st->Z);
      if (st->prm.pc_type != NKS_PC_NONE) clean(st, u, st->nf);
      halo(st, st->Z, st->nf);
      jv(st, st->Z, w);
      {
        PhaseScope ps(st, PH_VEC);
        launch_dcgs_dot(n, jj, V, n, st->red_part, st->red_out, st->red_cnt, st->stream);
        count_launch(st, 2);
      }
      reduce_to_ring(jj);
      {
        PhaseScope ps(st, PH_VEC);
        launch_dcgs_update(n, jj, V, n, st->red_out, st->stream);
        count_launch(st, 1);
      }
    };
    auto launch_close = [&](int jj) {           // cycle end: reduction of the last candidate u_m only
      {
        PhaseScope ps(st, PH_VEC);
        launch_dcgs_dot_u(n, jj, V, n, st->red_part, st->red_out, st->red_cnt, st->stream);
        count_launch(st, 2);
      }
      reduce_to_ring(jj);
    };
    const int its0 = its;
    launch_iter(0);
    int k = 0;                                  // finalised Hessenberg columns of this cycle
    double resid = beta;
    for (int j = 0; j <= m; ++j) {
      // look-ahead: the next step is queued before the host waits for this one
      // (step jj yields column jj, final at processing jj + 1; the cycle stops at its0 + j >= gmres_maxit)
      if (j + 1 < m && its0 + j + 1 <= st->prm.gmres_maxit) launch_iter(j + 1);
      else if (j + 1 == m && its0 + m <= st->prm.gmres_maxit) launch_close(m);
      CK(cudaEventSynchronize(st->gm_ev[j % 4]));
      st->syncs++;
      const double* hv = st->h_ring + (j % 4) * 128;
      // r and gamma exactly as the device computed them (krylov.cu: dcgs_scalars)
      double aa = 0.0, ab = 0.0;
      for (int l = 0; l < j; ++l) {
        aa += hv[l] * hv[l];
        ab += hv[l] * hv[32 + l];
      }
      const double r = std::sqrt(std::max(hv[64] - aa, 0.0));
      const bool breakdown = !(r > 1e-300);
      if (j == 0) {
        g[0] = beta * r;                        // r0 = beta V0 = (beta r) v_0
      } else {
        // column j-1 final: h_prev + a, subdiagonal r
        for (int i = 0; i < j; ++i) Hr[i * m + j - 1] = hprev[i] + hv[i];
        Hr[j * m + j - 1] = r;
        for (int i = 0; i <= j; ++i) R[i * m + j - 1] = Hr[i * m + j - 1];
        const int c = j - 1;
        for (int q = 0; q < c; ++q) {
          const double a0 = R[q * m + c], b0 = R[(q + 1) * m + c];
          R[q * m + c] = cs[q] * a0 + sn[q] * b0;
          R[(q + 1) * m + c] = -sn[q] * a0 + cs[q] * b0;
        }
        const double a0 = R[c * m + c], b0 = R[(c + 1) * m + c];
        const double rr = std::hypot(a0, b0);
        cs[c] = rr > 0 ? a0 / rr : 1.0;
        sn[c] = rr > 0 ? b0 / rr : 0.0;
        R[c * m + c] = rr;
        R[(c + 1) * m + c] = 0.0;
        g[c + 1] = -sn[c] * g[c];
        g[c] = cs[c] * g[c];
        ++its;
        k = j;
        resid = std::fabs(g[c + 1]);
        if (resid <= tol || breakdown || its >= st->prm.gmres_maxit || j == m) break;
      }
      // tentative column j: h' = ([b; gamma] - H a)/r  (A M^-1 v_j = V h' + u_{j+1})
      const double inv_r = breakdown ? 0.0 : 1.0 / r;
      const double gamma = (hv[65] - ab) * inv_r;
      for (int i = 0; i <= j; ++i) {
        double ha = 0.0;
        for (int l = 0; l < j; ++l) ha += Hr[i * m + l] * hv[l];
        hnew[i] = ((i < j ? hv[32 + i] : gamma) - ha) * inv_r;
      }
      std::swap(hprev, hnew);
      if (breakdown) break;
    }
    // the look-ahead may have queued one more step: it only writes slots >= k + 1, never read below
    // y = R^{-1} g (upper triangular k x k)
    for (int q = k - 1; q >= 0; --q) {
      double acc = g[q];
      for (int l = q + 1; l < k; ++l) acc -= R[q * m + l] * y[l];
      y[q] = acc / R[q * m + q];
    }
    {
      PhaseScope ps(st, PH_VEC);
      launch_lincomb(n, k, V, n, y.data(), st->W2, st->stream);
      count_launch(st, 1);
    }
    if (st->prm.pc_type != NKS_PC_NONE) halo(st, st->W2, st->nf);
    pc_apply(st, st->W2, st->Z);
    clean(st, st->W2, st->nf);          // W2 receives J s below and must keep zero ghosts
    {
      PhaseScope ps(st, PH_VEC);
      launch_axpby(n, 1.0, st->Z, 1.0, s, st->stream);
      count_launch(st, 1);
    }
    if (st->debug) std::fprintf(stderr, "[nks] gmres cycle its=%d beta=%.3e resid_est=%.3e tol=%.3e\n", its, beta, resid, tol);
    if (resid <= tol) return 0;
    if (its >= st->prm.gmres_maxit) return 1;
    // restart: r = b - J s  -> V[0]
    halo(st, s, st->nf);
    jv(st, s, st->W2);
    {
      PhaseScope ps(st, PH_VEC);
      launch_xpay(n, b, -1.0, st->W2, V, st->stream);
      count_launch(st, 1);
    }
    {
      PhaseScope ps(st, PH_RED);
      launch_norm_admissible(n / st->nf, st->nf, V, nullptr, st->red_part, st->red_out, st->stream);
      count_launch(st, 2);
    }
    comm_allreduce(st, st->red_out, 1);
    CK(cudaMemcpyAsync(st->h_red, st->red_out, sizeof(double), cudaMemcpyDeviceToHost, st->stream));
    sync(st);
    {
      const double prev = beta;
      beta = std::sqrt(st->h_red[0]);
      // Stagnation (opt-in, nks_params.gmres_stall_cycles, reading R18): k restart cycles in a row that
      // each remove less than 0.1 % of the true residual are reported as divergence instead of running
      // to gmres_maxit.  Off by default (the paper's solver fails only at its iteration limit).
      stall = (beta > 0.999 * prev) ? stall + 1 : 0;
      if (st->prm.gmres_stall_cycles > 0 && stall >= st->prm.gmres_stall_cycles) return 2;
      // Projection (opt-in, the same parameter): after at least gmres_stall_cycles cycles, the convergence
      // rate of the last kProjWin restart cycles (all cycles while fewer) projects the iterations still
      // needed; a solve that would not reach tol within gmres_maxit even at twice that rate is reported now
      // instead of after running to the limit.  Restarted GMRES slows down as it stagnates, so the recent
      // rate is the faithful estimate (the mean since the start carries the first cycles' fast drop: at
      // config 2 it let a solve that fails at gmres_maxit run 4,350 iterations before being rejected); the
      // factor 2 keeps a margin for a solve that speeds up again (R18, profiles/r02_attempts*).
      hist.push_back(beta);
      hits.push_back(its);
      if (st->prm.gmres_stall_cycles > 0 && its >= st->prm.gmres_stall_cycles * m && beta > tol) {
        const int cyc = (int)hist.size() - 1;                          // hist[0] = bnorm
        const int w = std::min(cyc, kProjWin);
        const double rate = std::log(beta / hist[cyc - w]) / (double)std::max(1, its - hits[cyc - w]);   // < 0: converging
        const double need = rate < 0.0 ? std::log(tol / beta) / rate : 1e300;
        if (its + 0.5 * need > (double)st->prm.gmres_maxit) return 3;
      }
    }
    // V already holds r; scale below uses V as source (first == false)
  }
}

// sum of a.b over n doubles (own points: the ghost planes of slab vectors are kept zero), all ranks -- host sync
double dot(nks_state* st, const double* a, const double* b, long long n) {
  {
    PhaseScope ps(st, PH_RED);
    launch_dot(n, a, b, st->red_part, st->red_out, st->stream);
    count_launch(st, 2);
  }
  comm_allreduce(st, st->red_out, 1);
  CK(cudaMemcpyAsync(st->h_red, st->red_out, sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  sync(st);
  return st->h_red[0];
}

// u^0 of the current c (reading R13) by conjugate gradients on the elastic block, for the states the FFT
// does not cover (z-slabs, Neumann boundaries) or on request (nks_params.u0_cg): the u rows of F are
// A_uu u + A_uc (c - cbar0), A_uu is symmetric negative semi-definite with the gauge as its
// null space (R14 / R38), so CG on -A_uu u = A_uc (c - cbar0) with the right-hand side projected onto the
// gauge complement converges to the canonical-gauge equilibrium.  A_uu p is the u part of J (0, 0, p) (the
// J.v kernels; the pointwise partials are zeroed, they only enter the c and eta rows).  Stops at
// ||r|| <= 1e-13 ||b|| (or, when roundoff stalls it first, below 1e-10).  Returns 0 or 1 (not converged).
int init_u0_cg(nks_state* st, int& its_out) {
  const long long N = st->N, nvec = st->nvec, off = 2 * N, nu = st->d * N;
  double* x = st->S;
  double* r = st->Ft;
  double* p = st->W2;
  double* q = st->Z;
  CK(cudaMemsetAsync(st->Xn + off, 0, nu * sizeof(double), st->stream));
  CK(cudaMemsetAsync(st->jac4, 0, 4 * N * sizeof(double), st->stream));
  halo(st, st->Xn, st->nf);
  residual(st, st->Xn, st->F);                                // u rows: A_uc (c - cbar0)
  for (double* v : {x, r, p, q}) CK(cudaMemsetAsync(v, 0, nvec * sizeof(double), st->stream));
  {
    // A_uu u = -F_u(0)  <=>  (-A_uu) u = F_u(0): CG on the positive semi-definite -A_uu with b = F_u(0)
    PhaseScope ps(st, PH_VEC);
    launch_axpby(nu, 1.0, st->F + off, 0.0, r + off, st->stream);
    count_launch(st, 1);
  }
  gauge(st, r);
  clean(st, r, st->nf);
  CK(cudaMemcpyAsync(p, r, nvec * sizeof(double), cudaMemcpyDeviceToDevice, st->stream));
  double rr = dot(st, r + off, r + off, nu);
  const double bnorm = std::sqrt(rr);
  double best = bnorm;
  int since_best = 0, it = 0;
  const int maxit = 200000;
  bool ok = bnorm == 0.0;
  for (; !ok && it < maxit; ++it) {
    halo(st, p, st->nf);
    jv(st, p, q);                                             // q_u = A_uu p_u
    clean(st, p, st->nf);
    clean(st, q, st->nf);
    const double pq = -dot(st, p + off, q + off, nu);         // p . (-A) p > 0
    if (!(pq > 0.0)) break;
    const double alpha = rr / pq;
    {
      PhaseScope ps(st, PH_VEC);
      launch_axpby(nu, alpha, p + off, 1.0, x + off, st->stream);    // x += alpha p
      launch_axpby(nu, alpha, q + off, 1.0, r + off, st->stream);    // r -= alpha (-A p)
      count_launch(st, 2);
    }
    if (it % 64 == 63) gauge(st, r);                          // keep roundoff out of the null space
    const double rr2 = dot(st, r + off, r + off, nu);
    const double rn = std::sqrt(rr2);
    if (rn <= 1e-13 * bnorm) { ok = true; ++it; break; }
    if (rn < 0.5 * best) { best = rn; since_best = 0; } else if (++since_best > 2000) break;
    const double beta = rr2 / rr;
    rr = rr2;
    {
      PhaseScope ps(st, PH_VEC);
      launch_axpby(nu, 1.0, r + off, beta, p + off, st->stream);     // p = r + beta p
      count_launch(st, 1);
    }
  }
  if (!ok && best <= 1e-10 * bnorm) ok = true;
  its_out = it;
  CK(cudaMemcpyAsync(st->Xn + off, x + off, nu * sizeof(double), cudaMemcpyDeviceToDevice, st->stream));
  return ok ? 0 : 1;
}

void energy(nks_state* st, const double* X, double parts[4], double& mass) {
  {
    PhaseScope ps(st, PH_RED);
    launch_energy(st->dp, X, st->red_part, st->red_out, st->stream);
    count_launch(st, 2);
  }
  comm_allreduce(st, st->red_out, 5);
  CK(cudaMemcpyAsync(st->h_red, st->red_out, 5 * sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  sync(st);
  const double vol = std::pow(st->grid.h, st->d);
  for (int k = 0; k < 4; ++k) parts[k] = st->h_red[k] * vol;
  mass = st->h_red[4] * vol;
}

void level_prep(nks_state* st) {
  PhaseScope ps(st, PH_OTHER);
  launch_level_prep(st->dp, st->Xn, st->Ta, st->stream);
  count_launch(st, 1);
}

// One NKS step (transactional).
nks_status step_impl(nks_state* st, double dt, nks_step_info* info) {
  nks_step_info loc{};
  nks_step_info& I = info ? *info : loc;
  std::memset(&I, 0, sizeof(I));
  I.dt = dt;
  if (!(dt > 0)) { st->err = "dt must be > 0"; return NKS_E_INVALID; }
  set_dt(st, dt);
  const long long nbytes = st->nvec * sizeof(double);
  CK(cudaMemcpyAsync(st->Xb, st->Xn, nbytes, cudaMemcpyDeviceToDevice, st->stream));
  residual(st, st->Xb, st->F);
  double f, bad;
  norm_adm(st, st->F, st->Xb, f, bad);
  if (bad > 0 || !std::isfinite(f)) {
    I.reason = NKS_REASON_DOMAIN;
    st->err = "X^n inadmissible";
    return NKS_E_DOMAIN;
  }
  const double f0 = f;
  I.fnorm0 = f0;
  const nks_params& p = st->prm;
  int it = 0;
  for (;; ++it) {
    if (f <= std::max(p.newton_rtol * f0, p.newton_atol)) break;
    if (it == p.newton_maxit) {
      I.reason = NKS_REASON_NEWTON_MAXIT;
      I.fnorm = f;
      st->err = "Newton did not converge in newton_maxit iterations";
      return NKS_E_DIVERGED;
    }
    {
      PhaseScope ps(st, PH_OTHER);
      launch_pointwise_jac(st->dp, st->Xn, st->Xb, st->jac4, st->stream);
      count_launch(st, 1);
    }
    if (p.pc_type != NKS_PC_NONE) {
      bool refactor = p.pc_reuse == 0 || (p.pc_reuse == 1 && it == 0) ||
                      (p.pc_reuse == 2 && (!st->pc_valid || st->pc_dt != dt));
      if (refactor) {
        pc_setup(st, st->Xb);
        I.pc_setups++;
      }
    }
    // b = -F (into Ft), solve J S = b
    {
      PhaseScope ps(st, PH_VEC);
      launch_axpby(st->nvec, -1.0, st->F, 0.0, st->Ft, st->stream);
      count_launch(st, 1);
    }
    // Project b onto range(J): the left null space of J is spanned by the indicators of the u_I rows
    // on each parity sub-lattice (sub-lattice sums of D^(.) vanish identically, reading R14), so
    // the u-rows of F carry only an inconsistent roundoff component there.  Removing it (the same
    // sub-lattice-mean projection as the gauge) keeps GMRES from chasing an unreachable residual;
    // the oracle's pinned-row direct solve drops the same component.
    gauge(st, st->Ft);
    clean(st, st->Ft, st->nf);
    int gits = 0;
    const double tol = std::max(p.gmres_rtol * f, p.gmres_atol);
    const int grc = gmres(st, st->Ft, f, st->S, tol, gits);
    I.gmres_its += gits;
    if (grc != 0) {
      I.reason = grc == 2 ? NKS_REASON_GMRES_STAGNATION : (grc == 3 ? NKS_REASON_GMRES_PROJECTED : NKS_REASON_GMRES_MAXIT);
      I.fnorm = f;
      st->err = grc == 2 ? "GMRES stagnated (gmres_stall_cycles restart cycles with < 0.1 % residual reduction)"
                         : (grc == 3 ? "GMRES projected past gmres_maxit at its mean convergence rate"
                                     : "GMRES reached gmres_maxit");
      return NKS_E_DIVERGED;
    }
    // line search (reading R17)
    double lam = 1.0, ft = 0.0;
    bool accepted = false;
    for (int hv = 0; hv <= p.ls_max_halvings; ++hv) {
      {
        PhaseScope ps(st, PH_VEC);
        launch_xpay(st->nvec, st->Xb, lam, st->S, st->Xt, st->stream);
        count_launch(st, 1);
      }
      halo(st, st->Xt, st->nf);
      residual(st, st->Xt, st->Ft);
      norm_adm(st, st->Ft, st->Xt, ft, bad);
      if (bad == 0 && std::isfinite(ft) && ft <= (1.0 - p.ls_alpha * lam) * f) {
        accepted = true;
        break;
      }
      lam *= 0.5;
      I.ls_halvings++;
    }
    if (!accepted) {
      I.reason = NKS_REASON_LINE_SEARCH;
      I.fnorm = f;
      st->err = "line search failed";
      return NKS_E_DIVERGED;
    }
    std::swap(st->Xb, st->Xt);
    std::swap(st->F, st->Ft);
    f = ft;
    gauge(st, st->Xb);
  }
  I.newton_its = it;
  I.fnorm = f;
  I.converged = 1;
  // accept: X^{n-1} <- X^n, X^n <- X^b
  double* old = st->Xprev;
  st->Xprev = st->Xn;
  st->Xn = st->Xb;
  st->Xb = old;
  st->have_prev = true;
  st->dt_prev = dt;
  st->time += dt;
  level_prep(st);
  energy(st, st->Xn, I.energy_parts, I.mass);
  I.energy = I.energy_parts[0] + I.energy_parts[1] + I.energy_parts[2] + I.energy_parts[3];
  I.time = st->time;
  I.zeta = st->zeta;
  return NKS_OK;
}

double change_rate(nks_state* st) {
  const nks_params& p = st->prm;
  const long long n = p.xd_norm == 2 ? 2 * st->N : st->nvec;
  {
    PhaseScope ps(st, PH_VEC);
    launch_xpay(n, st->Xn, -1.0, st->Xprev, st->W2, st->stream);
    count_launch(st, 1);
  }
  clean(st, st->W2, (int)(n / st->N));
  {
    PhaseScope ps(st, PH_RED);
    launch_norm_admissible(n, 1, st->W2, nullptr, st->red_part, st->red_out, st->stream);
    count_launch(st, 2);
  }
  comm_allreduce(st, st->red_out, 1);
  CK(cudaMemcpyAsync(st->h_red, st->red_out, sizeof(double), cudaMemcpyDeviceToHost, st->stream));
  sync(st);
  double nrm = std::sqrt(st->h_red[0]);
  if (p.xd_norm == 0) nrm /= std::sqrt((double)global_points(st) * st->nf);
  return nrm / st->dt_prev;
}

template <typename F>
nks_status guarded(nks_state* st, F&& fn) {
  try {
    return fn();
  } catch (const CudaError& e) {
    if (st) st->err = std::string("CUDA error: ") + cudaGetErrorString(e.e);
    return NKS_E_CUDA;
  } catch (const CommError&) {
    if (st) st->err = "communication callback failed";
    return NKS_E_NCCL;
  } catch (const std::exception& e) {
    if (st) st->err = e.what();
    return NKS_E_CUDA;
  }
}

cudaMemcpyKind kind_in(int on_device) { return on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice; }
cudaMemcpyKind kind_out(int on_device) { return on_device ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost; }

}  // namespace

// =====================================================================================================
extern "C" {

const char* nks_version(void) { return "nks-b200 0.1 (sm_100a, fp64)"; }

size_t nks_workspace_bytes(const nks_grid* grid, const nks_params* params) {
  if (validate(grid, params)) return 0;
  try {
    return make_layout(*grid, *params).total;
  } catch (const std::exception&) {
    return 0;
  }
}

nks_status nks_create(const nks_grid* grid, const nks_params* params, int32_t rank, int32_t nranks,
                      const uint8_t* nccl_id, void* workspace, size_t workspace_bytes, void* cuda_stream,
                      nks_state** out) {
  if (!out) return NKS_E_INVALID;
  *out = nullptr;
  if (validate(grid, params)) return NKS_E_INVALID;
  if (!workspace) return NKS_E_INVALID;
  if (nranks < 1 || nranks > kMaxRanks || rank < 0 || rank >= nranks) return NKS_E_INVALID;
  if (grid->zghost == 0 && nranks != 1) return NKS_E_INVALID;     // a periodic whole-grid state is one rank
  if (grid->yghost > 0 && nranks != grid->pz * grid->py) return NKS_E_INVALID;   // pencil: the pz x py grid
  IlukPattern Kpat;
  Layout L;
  try {
    L = make_layout(*grid, *params, &Kpat);
  } catch (const std::exception&) {
    return NKS_E_INVALID;
  }
  if (workspace_bytes < L.total) return NKS_E_OOM;
  nks_state* st = new nks_state();
  st->grid = *grid;
  st->prm = *params;
  st->stream = (cudaStream_t)cuda_stream;
  st->d = grid->dim;
  st->nf = 2 + grid->dim;
  st->N = (long long)grid->n[0] * grid->n[1] * grid->n[2];
  st->nvec = st->nf * st->N;
  st->dp = make_devparams(*grid, *params);
  st->ws = (char*)workspace;
  st->ws_bytes = workspace_bytes;
  st->zeta = params->zeta;
  st->debug = std::getenv("NKS_DEBUG") != nullptr;
  st->rank = rank;
  st->nranks = nranks;
  if (grid->zghost > 0) {
    st->dp.zoff = grid->z_offset;
    st->dp.nzg = grid->nz_global;
  }
  if (grid->yghost > 0) {
    st->dp.yoff = grid->y_offset;
    st->dp.nyg = grid->ny_global;
  }
  const nks_status rc = guarded(st, [&]() -> nks_status {
    char* w = st->ws;
    double** Xs[7] = {&st->Xn, &st->Xprev, &st->Xb, &st->Xt, &st->S, &st->F, &st->Ft};
    for (int k = 0; k < 7; ++k) *Xs[k] = (double*)(w + L.off_X[k]);
    st->Ta = (double*)(w + L.off_Ta);
    st->jac4 = (double*)(w + L.off_jac4);
    st->V = (double*)(w + L.off_V);
    st->Z = (double*)(w + L.off_Z);
    st->W2 = (double*)(w + L.off_W2);
    st->red_part = (double*)(w + L.off_part);
    st->red_out = (double*)(w + L.off_out);
    st->red_cnt = (unsigned*)(st->red_out + 255);
    st->gather = (double*)(w + L.off_gather);
    st->ystage = (double*)(w + L.off_ystage);
    if (grid->zghost > 0 && nccl_id) {     // library-owned communicator (collective over the nranks ranks)
      std::string why;
      st->nccl = nccl_create(nccl_id, rank, nranks, why);
      if (!st->nccl) {
        st->err = why;
        throw CommError();
      }
      st->comm_set = true;
    }
    CK(cudaMemsetAsync(st->red_cnt, 0, sizeof(unsigned), st->stream));
    if (grid->zghost > 0) CK(cudaMemsetAsync(w, 0, L.off_part, st->stream));   // zero ghosts of every vector
    CK(cudaMallocHost(&st->h_red, 256 * sizeof(double)));
    CK(cudaMallocHost(&st->h_ring, 4 * 128 * sizeof(double)));
    for (int k = 0; k < 4; ++k) CK(cudaEventCreateWithFlags(&st->gm_ev[k], cudaEventDisableTiming));
    if (params->pc_type == NKS_PC_SPECTRAL || params->pc_type == NKS_PC_RAS_SPECTRAL) {
      std::string why;
      st->spec = spectral_plan(*grid, st->nf, st->stream, why);
      if (!st->spec) throw std::runtime_error(why);
      st->specbuf = w + L.off_spec;
      st->pinv = w + L.off_pinv;
      if (params->pc_type == NKS_PC_RAS_SPECTRAL) {
        st->tl1 = (double*)(w + L.off_tl);
        st->tl2 = st->tl1 + st->nvec;
      }
    }
    if (params->pc_type != NKS_PC_NONE && params->pc_type != NKS_PC_SPECTRAL) {
      BoxSet& B = st->boxes;
      build_slot_tables(grid->dim, B);
      const bool gen = params->ilu_level != 0;
      if (gen) {          // level-k ILU: the slot tables of the fill pattern go to device memory
        B.gen = true;
        B.nslots = Kpat.nslots;
        B.diag = Kpat.diag;
        B.g_nlower = (int)Kpat.lower.size();
        B.g_nupper = (int)Kpat.upper.size();
        std::vector<int> tab;
        for (const auto& o3 : Kpat.off) tab.insert(tab.end(), o3.begin(), o3.end());
        int* t0 = (int*)(w + L.off_gtab);
        B.g_off = t0;
        B.g_lower = B.g_off + 3 * Kpat.nslots;
        B.g_upper = B.g_lower + Kpat.lower.size();
        B.g_pair_ptr = B.g_upper + Kpat.upper.size();
        B.g_pair_b = B.g_pair_ptr + Kpat.pair_ptr.size();
        B.g_pair_t = B.g_pair_b + Kpat.pair_b.size();
        for (const auto* v : {&Kpat.lower, &Kpat.upper, &Kpat.pair_ptr, &Kpat.pair_b, &Kpat.pair_t})
          tab.insert(tab.end(), v->begin(), v->end());
        CK(cudaMemcpyAsync(t0, tab.data(), tab.size() * sizeof(int), cudaMemcpyHostToDevice, st->stream));
      }
      HostBoxes H = build_boxes_host(*grid, B, gen ? &Kpat : nullptr);
      B.nbox = L.nbox;
      B.P = H.P;
      B.ld = L.ld;
      B.max_levels = H.max_levels;
      B.max_level_width = H.max_width;
      if ((long long)H.lev_ptr.size() > L.nlevptr) throw std::runtime_error("level table overflow");
      st->fac = (double*)(w + L.off_fac);
      st->fac32 = params->factor_fp32 ? (float*)(w + L.off_fac32) : nullptr;
      st->ybox = (double*)(w + L.off_ybox);
      B.gidx = (int*)(w + L.off_gidx);
      B.nbr = (int*)(w + L.off_nbr);
      B.box_lev_off = (int*)(w + L.off_levoff);
      B.lev_ptr = (int*)(w + L.off_levptr);
      B.box_pos_off = (int*)(w + L.off_posoff);
      B.h_box_lev_off = H.box_lev_off;
      B.h_box_pos_off = H.box_pos_off;
      CK(cudaMemcpyAsync(B.gidx, H.gidx.data(), H.gidx.size() * sizeof(int), cudaMemcpyHostToDevice, st->stream));
      CK(cudaMemcpyAsync(B.nbr, H.nbr.data(), H.nbr.size() * sizeof(int), cudaMemcpyHostToDevice, st->stream));
      CK(cudaMemcpyAsync(B.box_lev_off, H.box_lev_off.data(), H.box_lev_off.size() * sizeof(int), cudaMemcpyHostToDevice,
                         st->stream));
      CK(cudaMemcpyAsync(B.lev_ptr, H.lev_ptr.data(), H.lev_ptr.size() * sizeof(int), cudaMemcpyHostToDevice, st->stream));
      CK(cudaMemcpyAsync(B.box_pos_off, H.box_pos_off.data(), H.box_pos_off.size() * sizeof(int), cudaMemcpyHostToDevice,
                         st->stream));
      B.variant = params->pc_type == NKS_PC_AS_BILU0 ? 1 : (params->pc_type == NKS_PC_RRAS_BILU0 ? 2 : 0);
      B.cta_per_box = params->ras_cta_per_box;
      std::vector<int> cov_off, cov_pos;
      if (B.variant != 0) {        // CSR of the box positions covering every grid point, increasing position
        const long long Np = st->N;
        cov_off.assign(Np + 1, 0);
        for (long long q = 0; q < H.P; ++q) {
          const int gi = H.gidx[q] >= 0 ? H.gidx[q] : ~H.gidx[q];
          cov_off[gi + 1]++;
        }
        for (long long i = 0; i < Np; ++i) cov_off[i + 1] += cov_off[i];
        cov_pos.assign(H.P, 0);
        std::vector<int> fill(cov_off.begin(), cov_off.end() - 1);
        for (long long q = 0; q < H.P; ++q) {
          const int gi = H.gidx[q] >= 0 ? H.gidx[q] : ~H.gidx[q];
          cov_pos[fill[gi]++] = (int)q;
        }
        B.cover_off = (int*)(w + L.off_cover_off);
        B.cover_pos = (int*)(w + L.off_cover_pos);
        CK(cudaMemcpyAsync(B.cover_off, cov_off.data(), cov_off.size() * sizeof(int), cudaMemcpyHostToDevice, st->stream));
        CK(cudaMemcpyAsync(B.cover_pos, cov_pos.data(), cov_pos.size() * sizeof(int), cudaMemcpyHostToDevice, st->stream));
      }
      CK(cudaStreamSynchronize(st->stream));
      if (grid->dim == 2 && B.variant == 0 && !gen) {
        // one lane per row, one warp per component, a cluster of stripes per box (ras2d_rows.cu); boxes
        // the plan cannot take (e.g. > 8 stripes) use the level-synchronous apply of precond.cu
        std::string why;
        st->ras2d = r2::plan(*grid, B, w + L.off_geo, L.geo_bytes, st->stream, why, params->factor_fp32 != 0);
        if (st->debug)
          std::fprintf(stderr, "[nks] ras2d pipeline: %s (cluster %d)\n", st->ras2d ? "on" : why.c_str(),
                       r2::cluster_of(st->ras2d));
        CK(cudaStreamSynchronize(st->stream));
      }
    }
    return NKS_OK;
  });
  if (rc != NKS_OK) {
    if (st->h_red) cudaFreeHost(st->h_red);
    if (st->h_ring) cudaFreeHost(st->h_ring);
    for (int k = 0; k < 4; ++k)
      if (st->gm_ev[k]) cudaEventDestroy(st->gm_ev[k]);
    delete st;
    return rc;
  }
  *out = st;
  return NKS_OK;
}

nks_status nks_set_fields(nks_state* st, const double* c, const double* eta, const double* u, int32_t on_device) {
  if (!st || !c || !eta) return NKS_E_INVALID;
  return guarded(st, [&]() -> nks_status {
    const long long N = st->N;
    CK(cudaMemcpyAsync(st->Xn, c, N * sizeof(double), kind_in(on_device), st->stream));
    CK(cudaMemcpyAsync(st->Xn + N, eta, N * sizeof(double), kind_in(on_device), st->stream));
    if (u) CK(cudaMemcpyAsync(st->Xn + 2 * N, u, st->d * N * sizeof(double), kind_in(on_device), st->stream));
    halo(st, st->Xn, st->nf);
    // cbar0 = mean(c): the energy kernel's 5th sum is sum c (own planes; allreduced on slabs)
    {
      PhaseScope ps(st, PH_RED);
      launch_energy(st->dp, st->Xn, st->red_part, st->red_out, st->stream);  // u garbage only affects E3 here
      count_launch(st, 2);
    }
    comm_allreduce(st, st->red_out, 5);
    CK(cudaMemcpyAsync(st->h_red, st->red_out, 5 * sizeof(double), cudaMemcpyDeviceToHost, st->stream));
    sync(st);
    st->dp.cbar0 = st->h_red[4] / (double)global_points(st);
    if (!u) {
      if (slab(st) || st->dp.bc || st->prm.u0_cg) {
        // z-slabs (no whole-grid FFT), Neumann boundaries (not diagonalised by the DFT), or on request
        int its = 0;
        if (init_u0_cg(st, its) != 0) {
          st->err = "u0: conjugate gradients on the elastic block did not converge";
          return NKS_E_DIVERGED;
        }
        st->u0_cg_its = its;
        halo(st, st->Xn, st->nf);                 // the slab's u ghost planes from the neighbours' u^0
      } else {
        std::string e;
        if (init_displacement_fft(st->dp, st->Xn, st->Xn + 2 * N, st->V, st->stream, e) != 0) {
          st->err = e;
          return NKS_E_CUDA;
        }
        count_launch(st, 3 + st->d);
      }
    }
    gauge(st, st->Xn);
    level_prep(st);
    double nrm, bad;
    CK(cudaMemsetAsync(st->F, 0, st->nvec * sizeof(double), st->stream));
    norm_adm(st, st->F, st->Xn, nrm, bad);
    st->time = 0.0;
    st->have_prev = false;
    st->have_fields = true;
    st->pc_valid = false;
    st->zeta = st->prm.zeta;
    if (bad > 0) {
      st->err = "initial state inadmissible";
      return NKS_E_DOMAIN;
    }
    return NKS_OK;
  });
}

nks_status nks_set_comm(nks_state* st, nks_allreduce_fn allreduce, nks_halo_fn halo_fn, void* user) {
  if (!st || !slab(st) || !halo_fn) return NKS_E_INVALID;
  if (st->nccl) return NKS_E_STATE;                  // the state already owns an NCCL communicator
  if (st->nranks > 1 && !allreduce) return NKS_E_INVALID;
  st->comm_allreduce = allreduce;
  st->comm_halo = halo_fn;
  st->comm_user = user;
  st->comm_set = true;
  st->pc_valid = false;
  return NKS_OK;
}

int32_t nks_halo_plan(const nks_grid* local, int32_t rank, int32_t nranks, int32_t nfields, nks_halo_msg* out,
                      int32_t cap) {
  if (!local || local->zghost <= 0 || nranks < 1 || rank < 0 || rank >= nranks || nfields < 1) return -1;
  std::vector<nks_halo_msg> plan;
  if (local->yghost > 0) {
    if (local->pz < 1 || local->py < 1 || nranks != local->pz * local->py) return -1;
    pencil_halo_plan(*local, rank, nfields, plan);
    for (int k = 0; k < (int)plan.size() && k < cap && out; ++k) out[k] = plan[k];
    return (int32_t)plan.size();
  }
  const long long nxy = (long long)local->n[0] * local->n[1];
  halo_plan(rank, nranks, nfields, nxy * local->n[2], local->n[2], nxy, local->zghost, plan);
  for (int k = 0; k < (int)plan.size() && k < cap && out; ++k) out[k] = plan[k];
  return (int32_t)plan.size();
}

nks_status nks_get_unique_id(uint8_t id[128]) {
  if (!id) return NKS_E_INVALID;
  return nccl_unique_id(id) == 0 ? NKS_OK : NKS_E_NCCL;
}

nks_status nks_decompose_pencil(const nks_grid* global, const nks_params* params, int32_t rank, int32_t pz, int32_t py,
                                nks_grid* local) {
  if (!global || !params || !local || pz < 1 || py < 1 || pz * py > kMaxRanks) return NKS_E_INVALID;
  if (validate(global, params)) return NKS_E_INVALID;
  nks_grid loc{};
  if (pencil_decompose(*global, params->pc_type, rank, pz, py, loc) != 0) return NKS_E_INVALID;
  if (validate(&loc, params)) return NKS_E_INVALID;
  *local = loc;
  return NKS_OK;
}

nks_status nks_decompose(const nks_grid* global, const nks_params* params, int32_t rank, int32_t nranks,
                         nks_grid* local) {
  if (!global || !params || !local) return NKS_E_INVALID;
  if (validate(global, params)) return NKS_E_INVALID;
  if (nranks > kMaxRanks) return NKS_E_INVALID;
  int zoff = 0;
  nks_grid loc{};
  if (slab_decompose(*global, params->pc_type, rank, nranks, loc, zoff) != 0) return NKS_E_INVALID;
  loc.z_offset = zoff;
  loc.nz_global = global->n[2];
  if (validate(&loc, params)) return NKS_E_INVALID;
  *local = loc;
  return NKS_OK;
}

nks_status nks_set_cbar0(nks_state* st, double cbar0) {
  if (!st) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    st->dp.cbar0 = cbar0;
    level_prep(st);
    sync(st);
    return NKS_OK;
  });
}

nks_status nks_set_state(nks_state* st, const double* c, const double* eta, const double* u, int32_t on_device) {
  if (!st || !c || !eta || !u) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  if (slab(st) && !st->comm_set) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    const long long N = st->N;
    CK(cudaMemcpyAsync(st->Xn, c, N * sizeof(double), kind_in(on_device), st->stream));
    CK(cudaMemcpyAsync(st->Xn + N, eta, N * sizeof(double), kind_in(on_device), st->stream));
    CK(cudaMemcpyAsync(st->Xn + 2 * N, u, st->d * N * sizeof(double), kind_in(on_device), st->stream));
    halo(st, st->Xn, st->nf);
    gauge(st, st->Xn);
    level_prep(st);
    double nrm, bad;
    CK(cudaMemsetAsync(st->F, 0, st->nvec * sizeof(double), st->stream));
    norm_adm(st, st->F, st->Xn, nrm, bad);
    st->pc_valid = false;
    if (bad > 0) {
      st->err = "state inadmissible";
      return NKS_E_DOMAIN;
    }
    return NKS_OK;
  });
}

nks_status nks_get_fields(const nks_state* cst, double* c, double* eta, double* u, int32_t on_device) {
  nks_state* st = const_cast<nks_state*>(cst);
  if (!st || !c || !eta || !u) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    const long long N = st->N;
    CK(cudaMemcpyAsync(c, st->Xn, N * sizeof(double), kind_out(on_device), st->stream));
    CK(cudaMemcpyAsync(eta, st->Xn + N, N * sizeof(double), kind_out(on_device), st->stream));
    CK(cudaMemcpyAsync(u, st->Xn + 2 * N, st->d * N * sizeof(double), kind_out(on_device), st->stream));
    sync(st);
    return NKS_OK;
  });
}

nks_status nks_step(nks_state* st, double dt, nks_step_info* info) {
  if (!st) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  if (slab(st) && !st->comm_set) return NKS_E_STATE;
  return guarded(st, [&]() { return step_impl(st, dt, info); });
}

nks_status nks_run_adaptive(nks_state* st, int32_t max_steps, double t_end, nks_step_info* per_step, int32_t* done) {
  if (!st || max_steps < 0) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  if (slab(st) && !st->comm_set) return NKS_E_STATE;
  if (done) *done = 0;
  return guarded(st, [&]() -> nks_status {
    const nks_params& p = st->prm;
    for (int n = 0; n < max_steps; ++n) {
      if (t_end > 0 && st->time >= t_end) break;
      double dt, xd = 0.0;
      if (!st->have_prev) {
        dt = p.dt_init;
      } else {
        xd = change_rate(st);
        dt = std::max(p.dt_min, p.dt_max / std::sqrt(1.0 + st->zeta * xd * xd));   // Eq. (sencondt)
      }
      int retries = 0;
      nks_step_info info{};
      while (true) {
        const nks_status rc = step_impl(st, dt, &info);
        if (rc == NKS_OK) break;
        if (rc != NKS_E_DIVERGED) return rc;
        dt /= std::sqrt(2.0);
        st->zeta *= 2.0;
        ++retries;
        if (dt < p.dt_min * p.dt_floor_factor) {
          info.reason = NKS_REASON_DT_FLOOR;
          if (per_step) per_step[n] = info;
          st->err = "adaptive controller: dt fell below dt_min * dt_floor_factor";
          return NKS_E_DIVERGED;
        }
      }
      info.retries = retries;
      info.xd = xd;
      info.zeta = st->zeta;
      if (per_step) per_step[n] = info;
      if (done) *done = n + 1;
    }
    return NKS_OK;
  });
}

nks_status nks_energy(nks_state* st, double parts[4], double* mass) {
  if (!st || !parts || !mass) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  if (slab(st) && !st->comm_set) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    energy(st, st->Xn, parts, *mass);
    return NKS_OK;
  });
}

nks_status nks_eval_residual(nks_state* st, double dt, const double* x_b, double* F, int32_t on_device) {
  if (!st || !x_b || !F || !(dt > 0)) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    set_dt(st, dt);
    const size_t nb = st->nvec * sizeof(double);
    CK(cudaMemcpyAsync(st->Xt, x_b, nb, kind_in(on_device), st->stream));
    if (pencil(st)) halo(st, st->Xt, st->nf);          // pencils fill their ghosts here (slabs: the caller)
    residual(st, st->Xt, st->Ft);
    CK(cudaMemcpyAsync(F, st->Ft, nb, kind_out(on_device), st->stream));
    sync(st);
    return NKS_OK;
  });
}

nks_status nks_eval_jv(nks_state* st, double dt, const double* x_b, const double* v, double* Jv, int32_t on_device) {
  if (!st || !x_b || !v || !Jv || !(dt > 0)) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    set_dt(st, dt);
    const size_t nb = st->nvec * sizeof(double);
    CK(cudaMemcpyAsync(st->Xt, x_b, nb, kind_in(on_device), st->stream));
    CK(cudaMemcpyAsync(st->W2, v, nb, kind_in(on_device), st->stream));
    if (pencil(st)) {
      halo(st, st->Xt, st->nf);
      halo(st, st->W2, st->nf);
    }
    {
      PhaseScope ps(st, PH_OTHER);
      launch_pointwise_jac(st->dp, st->Xn, st->Xt, st->jac4, st->stream);
      count_launch(st, 1);
    }
    jv(st, st->W2, st->Ft);
    CK(cudaMemcpyAsync(Jv, st->Ft, nb, kind_out(on_device), st->stream));
    sync(st);
    return NKS_OK;
  });
}

nks_status nks_pc_setup(nks_state* st, double dt, const double* x_b, int32_t on_device) {
  if (!st || !x_b || !(dt > 0)) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    set_dt(st, dt);
    CK(cudaMemcpyAsync(st->Xb, x_b, st->nvec * sizeof(double), kind_in(on_device), st->stream));
    {
      PhaseScope ps(st, PH_OTHER);
      launch_pointwise_jac(st->dp, st->Xn, st->Xb, st->jac4, st->stream);
      count_launch(st, 1);
    }
    pc_setup(st, st->Xb);
    sync(st);
    return NKS_OK;
  });
}

nks_status nks_pc_apply(nks_state* st, const double* r, double* z, int32_t on_device) {
  if (!st || !r || !z) return NKS_E_INVALID;
  if (st->prm.pc_type != NKS_PC_NONE && !st->pc_valid) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    const size_t nb = st->nvec * sizeof(double);
    CK(cudaMemcpyAsync(st->W2, r, nb, kind_in(on_device), st->stream));
    pc_apply(st, st->W2, st->Z);
    CK(cudaMemcpyAsync(z, st->Z, nb, kind_out(on_device), st->stream));
    sync(st);
    return NKS_OK;
  });
}

nks_status nks_gmres_solve(nks_state* st, double dt, const double* x_b, const double* rhs, double* s, int32_t on_device,
                           int32_t* its) {
  if (!st || !x_b || !rhs || !s || !(dt > 0)) return NKS_E_INVALID;
  if (!st->have_fields) return NKS_E_STATE;
  return guarded(st, [&]() -> nks_status {
    set_dt(st, dt);
    const size_t nb = st->nvec * sizeof(double);
    CK(cudaMemcpyAsync(st->Xb, x_b, nb, kind_in(on_device), st->stream));
    CK(cudaMemcpyAsync(st->Ft, rhs, nb, kind_in(on_device), st->stream));
    {
      PhaseScope ps(st, PH_OTHER);
      launch_pointwise_jac(st->dp, st->Xn, st->Xb, st->jac4, st->stream);
      count_launch(st, 1);
    }
    if (st->prm.pc_type != NKS_PC_NONE) pc_setup(st, st->Xb);
    double bn, bad;
    norm_adm(st, st->Ft, nullptr, bn, bad);
    int it = 0;
    const double tol = std::max(st->prm.gmres_rtol * bn, st->prm.gmres_atol);
    const int rc = gmres(st, st->Ft, bn, st->S, tol, it);
    if (its) *its = it;
    CK(cudaMemcpyAsync(s, st->S, nb, kind_out(on_device), st->stream));
    sync(st);
    if (rc != 0) {
      st->err = rc == 2 ? "GMRES stagnated" : (rc == 3 ? "GMRES projected past gmres_maxit" : "GMRES reached gmres_maxit");
      return NKS_E_DIVERGED;
    }
    return NKS_OK;
  });
}

nks_status nks_counters(const nks_state* st, int64_t* kernel_launches, int64_t* host_syncs, int64_t* reductions) {
  if (!st) return NKS_E_INVALID;
  if (kernel_launches) *kernel_launches = st->launches;
  if (host_syncs) *host_syncs = st->syncs;
  if (reductions) *reductions = st->reductions;
  return NKS_OK;
}

nks_status nks_set_profiling(nks_state* st, int32_t enable) {
  if (!st) return NKS_E_INVALID;
  st->profile = enable != 0;
  return NKS_OK;
}

nks_status nks_phase_times(nks_state* st, double ms[8], int64_t counts[8], int32_t reset) {
  if (!st) return NKS_E_INVALID;
  return guarded(st, [&]() -> nks_status {
    CK(cudaStreamSynchronize(st->stream));
    for (size_t k = 0; k < st->pend_phase.size(); ++k) {
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, st->pend_ev[2 * k], st->pend_ev[2 * k + 1]));
      st->phase_ms[st->pend_phase[k]] += t;
      st->phase_cnt[st->pend_phase[k]] += 1;
      st->ev_pool.push_back(st->pend_ev[2 * k]);
      st->ev_pool.push_back(st->pend_ev[2 * k + 1]);
    }
    st->pend_phase.clear();
    st->pend_ev.clear();
    for (int k = 0; k < 8; ++k) {
      if (ms) ms[k] = st->phase_ms[k];
      if (counts) counts[k] = st->phase_cnt[k];
      if (reset) { st->phase_ms[k] = 0; st->phase_cnt[k] = 0; }
    }
    return NKS_OK;
  });
}

nks_status nks_destroy(nks_state* st) {
  if (!st) return NKS_E_INVALID;
  cudaStreamSynchronize(st->stream);
  for (auto e : st->ev_pool) cudaEventDestroy(e);
  for (auto e : st->pend_ev) cudaEventDestroy(e);
  if (st->h_red) cudaFreeHost(st->h_red);
  if (st->h_ring) cudaFreeHost(st->h_ring);
  for (int k = 0; k < 4; ++k)
    if (st->gm_ev[k]) cudaEventDestroy(st->gm_ev[k]);
  if (st->ras2d) r2::free_plan(st->ras2d);
  if (st->spec) spectral_free(st->spec);
  if (st->nccl) nccl_destroy(st->nccl);
  delete st;
  return NKS_OK;
}

const char* nks_last_error(const nks_state* st) { return st ? st->err.c_str() : "NULL state"; }

}  // extern "C"
