/*
 * nks.h -- C ABI of the B200 (sm_100a) Newton-Krylov-Schwarz time step of arXiv 2209.08001.
 *
 * The library solves, once per time step, the nonlinear system F(X^{n+1}; X^n, dt) = 0 of the
 * discrete-variational-derivative scheme NSOA-1 (Eq. NSOA-1) for the
 * reduced Ni-alloy phase-field model: composition c, one long-range order parameter eta and the
 * quasi-static displacement u_1..u_d.  Method (Sec. 4):
 * inexact Newton with line search, restarted right-preconditioned GMRES, restricted additive
 * Schwarz (left-RAS, Cai-Sarkis) with point-block ILU(0) subdomain solves, adaptive dt (Eq.
 * sencondt).  All arithmetic is fp64 on the device; the host only steers.
 *
 * Conventions
 *   - Field layout at the ABI: field-major arrays (c, then eta, then u_1..u_d), each field in C
 *     order over (z, y, x) with x fastest, no halo, n[0]*n[1]*n[2] points per field.  u_I is the
 *     displacement component along axis I (I = 1 is x).
 *   - "on_device" = 1: the pointer is a CUDA device pointer on the state's device; 0: host memory.
 *   - Every call returns nks_status (NKS_OK = 0); no C++ exception crosses the ABI; the per-state
 *     message of the last failure is returned by nks_last_error().
 *   - Ownership: the caller owns every array, info struct and the workspace, which must outlive
 *     the state; the library keeps no caller pointer past return except the workspace.  The
 *     library owns the events/plans it creates and destroys them in nks_destroy().
 *   - Threading: one state per stream; no global mutable state.  Calls on one state must not
 *     overlap.
 *   - Determinism: every reduction is a fixed-order two-stage tree; results are bitwise
 *     reproducible for a given grid, params and launch configuration.
 */
#ifndef NKS_H
#define NKS_H

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define NKS_API __attribute__((visibility("default")))
#else
#define NKS_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

typedef enum {
  NKS_OK = 0,
  NKS_E_INVALID = 1,   /* bad argument: grid/params out of range, NULL pointer, size mismatch   */
  NKS_E_DOMAIN = 2,    /* state inadmissible: c, p = c*eta or q = c*(4-3*eta) not in (0,1), NaN */
  NKS_E_DIVERGED = 3,  /* Newton max-its, line-search failure or GMRES max-its (reading R24)     */
  NKS_E_CUDA = 4,      /* CUDA / cuFFT runtime error (message in nks_last_error)                */
  NKS_E_NCCL = 5,      /* NCCL (library-owned communicator) or a communication callback failed */
  NKS_E_OOM = 6,       /* workspace too small                                                   */
  NKS_E_STATE = 7      /* call order violated (e.g. nks_step before nks_set_fields)            */
} nks_status;

/* Divergence reasons reported in nks_step_info.reason. */
enum { NKS_REASON_NONE = 0, NKS_REASON_NEWTON_MAXIT = 1, NKS_REASON_LINE_SEARCH = 2,
       NKS_REASON_GMRES_MAXIT = 3, NKS_REASON_DOMAIN = 4, NKS_REASON_DT_FLOOR = 5,
       NKS_REASON_GMRES_STAGNATION = 6 /* gmres_stall_cycles cycles each removing < 0.1 % of the residual */,
       NKS_REASON_GMRES_PROJECTED = 7 /* the solve's mean rate projects it past gmres_maxit (opt-in, same param) */ };

/* Preconditioner types (the variants are SURVEY 8(f)-1's Schwarz family, Cai-Sarkis):
 *   RAS    z = sum_i R_i^{0T} (L_i U_i)^{-1} R_i^delta r     (left restricted additive Schwarz, default)
 *   AS     z = sum_i R_i^{deltaT} (L_i U_i)^{-1} R_i^delta r (classical additive Schwarz)
 *   RRAS   z = sum_i R_i^{deltaT} (L_i U_i)^{-1} R_i^0 r     (right-restricted: input restricted to owned points)
 * AS and RRAS sum the overlapping boxes' contributions in a fixed box order (deterministic); they are
 * single-state only (a z-slab state would need a reverse halo exchange) and use the level-synchronous
 * subdomain solve. */
enum { NKS_PC_NONE = 0, NKS_PC_RAS_BILU0 = 2, NKS_PC_AS_BILU0 = 3, NKS_PC_RRAS_BILU0 = 4, NKS_PC_SPECTRAL = 5,
       NKS_PC_RAS_SPECTRAL = 6 };
/* NKS_PC_RAS_SPECTRAL: two-level -- the spectral preconditioner below as a global (coarse) correction, then
 * left-RAS/BILU(0) on the remaining residual: z1 = S r, z = z1 + RAS(r - J z1).  Periodic single states. */
/* NKS_PC_SPECTRAL (not the paper's): the inverse of J with its variable coefficients
 * (the pointwise partials of G1 + G2S, the level-n mobility) replaced by their grid means, applied per
 * wave number with cuFFT -- exact for a uniform state, so GMRES needs few iterations while the fields are
 * near-uniform.  Periodic single-GPU states only.  Like every preconditioner it changes GMRES's iteration
 * count, never the converged step. */

typedef struct {
  int32_t dim;       /* 2 or 3                                                          */
  int32_t n[3];      /* grid points per axis, n[0] = x (fastest); n[2] = 1 when dim == 2.       */
                     /* Periodic.  Each n[j] >= 5 (stencil radius 2 must not alias).    */
  double h;          /* uniform mesh size (0.25)                                         */
  int32_t nsub[3];   /* RAS subdomain boxes per axis (1 <= nsub[j] <= n[j]); nsub[2]=1 in 2D     */
  int32_t overlap;   /* delta: cells added on each side of every box (0..8)      */
  int32_t zghost;    /* 0: periodic grid.  2..8: this state is one z-slab of a z-sharded 3D grid  */
                     /* (SURVEY 8(e)): n[2] counts zghost ghost planes on each side, filled by the  */
                     /* halo callback of nks_set_comm (or by the caller for the eval hooks); F,    */
                     /* J.v, energy and the gauge sums cover the own planes only, with no z wrap.  */
                     /* With pc_type RAS the nsub[2] boxes split the OWN planes (the caller aligns */
                     /* slabs with the global box grid) and zghost >= overlap + 1.                 */
                     /* nks_decompose() fills a rank's slab grid from the global one.              */
  int32_t z_offset;  /* zghost > 0: global z of this slab's first own plane                      */
  int32_t nz_global; /* zghost > 0: planes of the global periodic grid                            */
  int32_t bc;        /* 0: periodic.  1: homogeneous Neumann, Eq. (boundaryequ)    */
                     /* (reading R38: cell-centred mirror ghosts; traction-free u through odd stress */
                     /* ghosts; gauge = translations + discrete rotations).  Single-GPU states with */
                     /* pc_type NONE or SPECTRAL; nks_set_fields then needs u (no FFT u^0).        */
  int32_t yghost;    /* 0: no y split.  2..8: this state is one z x y PENCIL of a 3D grid sharded on a  */
                     /* pz x py process grid (SURVEY 8(e), configs 4/5 "slab- then pencil-sharded"): */
                     /* n[1] counts yghost ghost rows on each side as n[2] counts zghost (>= 2) ghost */
                     /* planes.  Pencil states run everything a z-slab runs (pc_type NONE or RAS with */
                     /* BILU(0) boxes; nks_eval_residual / nks_eval_jv fill their ghosts themselves). */
                     /* nks_decompose_pencil() fills a rank's pencil grid.                           */
  int32_t y_offset;  /* yghost > 0: global y of this pencil's first own row                        */
  int32_t ny_global; /* yghost > 0: rows of the global periodic grid                                 */
  int32_t pz, py;    /* yghost > 0: the process grid (rank = rz * py + ry); ignored otherwise         */
  int32_t pad_;
} nks_grid;

/* ---- communication callbacks of a z-sharded state --------------------------------
 * Both are called from inside the library's calls, on the calling thread, with the state's stream;
 * the callback must leave its result ordered on that stream (e.g. an NCCL collective enqueued on
 * it, or a host-staged exchange followed by a copy on it).  Return 0 on success; any other value
 * makes the library call fail with NKS_E_NCCL. */
/* Sum n doubles at device pointer buf over all ranks, in place; every rank must get identical bits. */
typedef int32_t (*nks_allreduce_fn)(void* user, double* buf, int64_t n, void* cuda_stream);
/* Fill the zghost ghost planes on both z sides of nfields fields (field f at vec + f*field_stride,
 * each a local (n[2], n[1], n[0]) C-order array) from the periodic z neighbours' own planes. */
typedef int32_t (*nks_halo_fn)(void* user, double* vec, int32_t nfields, int64_t field_stride, void* cuda_stream);

typedef struct {
  /* ---- model, dimensionless (App. A/B).  CALPHAD-style coefficients in units of
   *      V_m*dE; the library derives M0..M6 of App. B from them.              */
  double theta;      /* theta of E_G                                                 */
  double gamma_c;    /* gradient coefficient of c                                       */
  double gamma_eta;  /* gradient coefficient of eta (enters as 3*gamma_eta)              */
  double kappa;      /* mobility scale, M = kappa c(1-c)                       */
  double eps0;       /* eigenstrain coefficient                                 */
  double C11, C12, C44;   /* cubic Hooke tensor                                  */
  double Lscale;     /* multiplier of the Hooke tensor, script-L of P:634                      */
  double w_c;        /* weight of theta*Psi(c) in E_G: 1 = main text P:66 (reading R2)         */
  double L0, L1, L2, L3, U1, U4;   /* App. A/B coefficients / (V_m dE)                          */
  double dE0;        /* (E0_Al - E0_Ni)/(V_m dE): M0 = dE0 + L0 - L1 + L2 - L3         */
  int32_t S;         /* Taylor order of Psi_S (10); 1..16                    */
  /* ---- Newton / GMRES (readings R16-R18, R24) */
  double newton_rtol, newton_atol;   /* stop when ||F|| <= max(rtol*||F0||, atol) */
  double gmres_rtol, gmres_atol;     /* ||J S + F|| <= max(rtol*||F||, atol) */
  int32_t newton_maxit;              /* > this many Newton iterations -> DIVERGED             */
  int32_t gmres_restart;             /* GMRES(m) restart length, 1..64                        */
  int32_t gmres_maxit;               /* total GMRES iterations per Newton solve -> DIVERGED    */
  int32_t pc_type;                   /* NKS_PC_NONE, NKS_PC_RAS_BILU0, _AS_BILU0, _RRAS_BILU0 */
  int32_t pc_reuse;                  /* 0: refactor every Newton iterate; 1: once per step;    */
                                     /* 2: keep factors across steps while dt is unchanged     */
  double ls_alpha;                   /* sufficient decrease ||F(X+lS)|| <= (1-alpha l)||F||    */
  int32_t ls_max_halvings;           /* lambda = 1, 1/2, ... 2^-max before line-search failure */
  /* ---- adaptive controller (Eq. sencondt; readings R23/R24) */
  double zeta, dt_min, dt_max, dt_init;
  double dt_floor_factor;            /* abort when the retried dt < dt_min * factor            */
  int32_t xd_norm;                   /* ||X^n - X^{n-1}||: 0 RMS, 1 Euclidean, 2 (c,eta) Eucl. */
  int32_t factor_fp32;               /* 1: the level-synchronous subdomain solves read fp32 copies */
                                     /* of the BILU(0) factors (factorisation stays fp64; the    */
                                     /* preconditioner only changes GMRES's iteration count, not */
                                     /* the converged step -- SURVEY 8(f)-1).  0: fp64 factors.  */
  int32_t gmres_stall_cycles;        /* 0 (default, the paper's behaviour): a Newton solve fails    */
                                     /* only at gmres_maxit.  k > 0: k consecutive restart cycles   */
                                     /* that each remove < 0.1 % of the true residual are reported */
                                     /* as NKS_REASON_GMRES_STAGNATION (DIVERGED), and after k      */
                                     /* cycles a solve whose mean convergence rate projects it past */
                                     /* gmres_maxit as NKS_REASON_GMRES_PROJECTED, so the controller */
                                     /* retries without running to gmres_maxit.  A     */
                                     /* property of the linear solver, not of Eq. NSOA-1: it can   */
                                     /* change the accepted dt sequence (reading R18).   */
  int32_t ilu_level;                 /* Schwarz subdomain solver (Table 1): 0 = point-block */
                                     /* ILU(0) (default; reading R21), k = 1..8: ILU(k) on Saad's    */
                                     /* level-of-fill pattern, -1 = exact block LU (no pivoting,     */
                                     /* natural order).  k != 0 uses the level-synchronous solves;   */
                                     /* its factor storage grows with the fill (NKS_E_OOM / INVALID  */
                                     /* from nks_workspace_bytes when it cannot be held).            */
  int32_t u0_cg;                     /* u^0 when nks_set_fields gets u = NULL (reading R13): 0 = the */
                                     /* FFT solve on periodic whole-grid states, conjugate gradients */
                                     /* on the elastic block otherwise (z-slabs: no whole-grid FFT;  */
                                     /* Neumann); 1 = conjugate gradients always.                    */
  int32_t ras_cta_per_box;           /* level-synchronous RAS apply (3D; 2D boxes the pipelined apply */
                                     /* does not take): 0 = auto (a cluster of 2 CTAs per box when   */
                                     /* the boxes fill at most half the SMs), 1 = one CTA per box,   */
                                     /* 2 or 4 = a cluster of that many CTAs per box.  Same results  */
                                     /* bit for bit; only the work split over SMs changes.          */
} nks_params;

typedef struct {
  int32_t converged;        /* 1 if the step was accepted                                      */
  int32_t reason;           /* NKS_REASON_* of the last failure                               */
  int32_t newton_its;       /* Newton iterations of the accepted attempt                       */
  int32_t gmres_its;        /* GMRES iterations summed over those Newton iterations            */
  int32_t retries;          /* dt halvings by sqrt(2) before acceptance (nks_run_adaptive)     */
  int32_t ls_halvings;      /* line-search halvings summed over the Newton iterations          */
  int32_t pc_setups;        /* preconditioner (re)factorisations in this step                  */
  int32_t pad_;
  double dt;                /* accepted dt                                                     */
  double time;              /* t_{n+1}                                                         */
  double energy;            /* discrete free energy E~^{n+1}, cell volume h^d      */
  double energy_parts[4];   /* E~1..E~4                                                        */
  double mass;              /* h^d sum c                                               */
  double fnorm0, fnorm;     /* ||F(X_0)||, ||F(X_final)||                                      */
  double zeta;              /* controller zeta after the step (doubles on every retry)  */
  double xd;                /* X'_d used to predict this step's dt (0 for the first step)      */
} nks_step_info;

typedef struct nks_state nks_state;

/* Bytes of device workspace nks_create needs for this grid/params (0 on invalid input). */
NKS_API size_t nks_workspace_bytes(const nks_grid* grid, const nks_params* params);

/* NCCL unique id for a sharded run: rank 0 calls this and sends the 128 bytes to every rank
 * (e.g. a torch.distributed broadcast); each rank then passes them to nks_create.  NKS_E_NCCL on failure. */
NKS_API nks_status nks_get_unique_id(uint8_t id[128]);

/* The z-slab of `rank` out of `nranks` for a GLOBAL periodic 3D grid (zghost = 0) -- host only, no GPU.
 * Each rank owns a contiguous run of whole layers of the global RAS box grid (nsub[2] layers dealt out, the
 * first nsub[2] mod nranks ranks one more; without RAS the planes themselves), so the preconditioner and the
 * iteration counts do not depend on the number of ranks.  *local receives the slab grid:
 * own planes + zghost = max(2, overlap + 1) ghost planes per side (2 without RAS), nsub[2] = its box layers,
 * z_offset / nz_global set.  NKS_E_INVALID if the grid is not 3D, has fewer box layers than ranks, or a slab
 * would own fewer than 2 planes. */
NKS_API nks_status nks_decompose(const nks_grid* global, const nks_params* params, int32_t rank, int32_t nranks,
                                 nks_grid* local);

/* The pencil of `rank` on a pz x py process grid (rank = rz * py + ry) for a GLOBAL periodic 3D grid --
 * host only.  With pc_type RAS, rz owns a contiguous run of the nsub[2] global box layers along z and ry of
 * the nsub[1] layers along y (dealt out like nks_decompose), so every rank holds whole boxes and the
 * iteration counts do not depend on the process grid; ghosts = max(2, overlap + 1) planes / rows per side.
 * With pc_type NONE the planes and rows themselves are dealt out, 2 ghosts per side.  *local gets the own
 * extents + ghosts, z_offset / y_offset / nz_global / ny_global / pz / py and its box layers.
 * NKS_E_INVALID if the grid is not 3D, has fewer box layers than parts along an axis, or a part would own
 * fewer than 2 planes / rows. */
NKS_API nks_status nks_decompose_pencil(const nks_grid* global, const nks_params* params, int32_t rank, int32_t pz,
                                        int32_t py, nks_grid* local);

/* One message of a halo exchange: kind 0 = send, 1 = receive of a contiguous run (`count` doubles at
 * `offset` from the vector's start, field f at f * n[0]*n[1]*n[2]): the ghost PLANES of a slab or a pencil.
 * kind 2 = send, 3 = receive of a pencil's y block: `count` doubles (yghost rows) at `offset` in the first
 * own plane, repeated over every own plane with the plane stride n[0]*n[1] (packed plane after plane).  A
 * pencil exchanges y blocks first, then whole planes (ghost rows included), so the (y, z) edge cells the
 * stencil's (0, +-1, +-1) offsets read arrive through the second phase. */
typedef struct {
  int32_t kind;
  int32_t peer;
  int64_t offset;
  int64_t count;
} nks_halo_msg;

/* The ordered halo message list the library issues (grouped ncclSend/ncclRecv, matched per peer in issue order)
 * for a slab grid from nks_decompose or a pencil grid from nks_decompose_pencil (nranks = pz * py) -- host
 * only, no GPU.  Writes up to cap messages, returns how many the exchange has (4 per field for a slab; 4 y
 * messages then 4 plane messages per field for a pencil, y phase first), or -1 on invalid input. */
NKS_API int32_t nks_halo_plan(const nks_grid* local, int32_t rank, int32_t nranks, int32_t nfields, nks_halo_msg* out,
                              int32_t cap);

/* Create a state on the current CUDA device.
 *   grid: the whole periodic grid (zghost = 0; then rank = 0, nranks = 1), or this rank's z-slab from
 *         nks_decompose (zghost > 0).
 *   rank, nranks: this process's place in the sharded run (1 <= nranks <= 64).
 *   nccl_id: slab states only -- the 128-byte id of nks_get_unique_id (the same on every rank): the library
 *         creates and owns an NCCL communicator (ncclCommInitRank: collective, every rank must call
 *         nks_create), exchanges halos with grouped ncclSend/ncclRecv and reduces with ncclAllGather + a
 *         rank-ordered sum on its stream.  NULL: the caller attaches host callbacks with nks_set_comm
 *         (e.g. host-staged exchanges of emulated ranks).  Ignored for whole-grid states.
 *   workspace: device buffer of >= nks_workspace_bytes() bytes, 256-byte aligned, caller-owned
 *              (PyTorch allocates it); must outlive the state.
 *   cuda_stream: cudaStream_t on which every kernel and NCCL call of this state is issued (NULL = legacy).
 * Errors: NKS_E_INVALID (grid/params/rank), NKS_E_OOM (workspace too small), NKS_E_NCCL, NKS_E_CUDA. */
NKS_API nks_status nks_create(const nks_grid* grid, const nks_params* params, int32_t rank, int32_t nranks,
                              const uint8_t* nccl_id, void* workspace, size_t workspace_bytes, void* cuda_stream,
                              nks_state** out);

/* Set X^n.  c, eta: N doubles each; u: d*N doubles (u_1 block first) or NULL, in which case
 * u^0 solves the discrete mechanical equilibrium [D^ sigma^el]^0 = 0 (reading R13)
 * by an fp64 FFT (periodic whole grid) or by conjugate gradients on the elastic block (z-slabs, with
 * halos and allreduces; Neumann; params.u0_cg) -- NKS_E_DIVERGED if CG does not converge.  Sets cbar0 = mean(c) and projects u onto the canonical gauge
 * (zero mean per component and parity sub-lattice, reading R14).  Resets time, step history,
 * zeta and cached factors.  NKS_E_DOMAIN if the state is inadmissible. */
NKS_API nks_status nks_set_fields(nks_state* st, const double* c, const double* eta, const double* u,
                          int32_t on_device);

/* Replace X^n by (c, eta, u) -- u required -- WITHOUT restarting the run: time, the X^{n-1} history of
 * the controller (Eq. sencondt), zeta and cbar0 are kept; u is projected onto the
 * canonical gauge (reading R14) and T^n is recomputed.  This is how a caller streams the state
 * through host memory between steps (bench.py's end-to-end leg).  NKS_E_DOMAIN if inadmissible,
 * NKS_E_STATE before nks_set_fields. */
NKS_API nks_status nks_set_state(nks_state* st, const double* c, const double* eta, const double* u, int32_t on_device);

/* Set cbar0, the mean composition of the eigenstrain, explicitly -- used by z-slab states,
 * whose local mean is not the grid's.  Recomputes T^n. */
NKS_API nks_status nks_set_cbar0(nks_state* st, double cbar0);

/* Attach host communication callbacks to a z-slab state created without an NCCL id (the callback backend;
 * a state that owns an NCCL communicator returns NKS_E_STATE).  allreduce may be NULL only when nranks == 1;
 * halo must not be NULL.  A slab state needs its communication (NCCL or callbacks) before nks_set_fields /
 * nks_set_state / nks_step / nks_run_adaptive / nks_energy (NKS_E_STATE otherwise).  Every rank must make the
 * same sequence of calls: all control decisions (Newton and GMRES convergence, line search, dt) are taken
 * from reduced values that are bitwise identical on every rank.  On a slab state nks_set_fields takes local
 * arrays including ghost planes (ghost values are ignored) and needs u; cbar0 is the global mean of c. */
NKS_API nks_status nks_set_comm(nks_state* st, nks_allreduce_fn allreduce, nks_halo_fn halo, void* user);

/* Copy X^n out (same layout as nks_set_fields; u must hold d*N doubles). */
NKS_API nks_status nks_get_fields(const nks_state* st, double* c, double* eta, double* u, int32_t on_device);

/* One NKS time step X^n -> X^{n+1} with the given dt.
 * Transactional: on failure X^n is unchanged, status NKS_E_DIVERGED / NKS_E_DOMAIN and
 * info->reason tell why.  info may be NULL. */
NKS_API nks_status nks_step(nks_state* st, double dt, nks_step_info* info);

/* Adaptive time stepping (Eq. sencondt): up to max_steps accepted steps, stopping
 * early once time >= t_end (t_end <= 0: no time limit).  Step 0 uses dt_init; a diverged
 * attempt retries with dt/sqrt(2) and zeta*2; aborts with NKS_E_DIVERGED when dt would drop
 * below dt_min*dt_floor_factor.  per_step: array of max_steps records (or NULL); *done receives
 * the number of accepted steps. */
NKS_API nks_status nks_run_adaptive(nks_state* st, int32_t max_steps, double t_end,
                            nks_step_info* per_step, int32_t* done);

/* Discrete energy parts E~1..E~4 and mass of X^n. */
NKS_API nks_status nks_energy(nks_state* st, double parts[4], double* mass);

/* ---- test / benchmark hooks on the current X^n (level a) --------------------------------- */

/* F(x_b) of Eq. NSOA-1 for level a = X^n: x_b and F hold (2+d)*N doubles. */
NKS_API nks_status nks_eval_residual(nks_state* st, double dt, const double* x_b, double* F, int32_t on_device);

/* J(x_b) v (matrix-free analytic Jacobian). */
NKS_API nks_status nks_eval_jv(nks_state* st, double dt, const double* x_b, const double* v, double* Jv,
                       int32_t on_device);

/* Assemble and factor the RAS/BILU(0) preconditioner at x_b, then z = M^{-1} r. */
NKS_API nks_status nks_pc_setup(nks_state* st, double dt, const double* x_b, int32_t on_device);
NKS_API nks_status nks_pc_apply(nks_state* st, const double* r, double* z, int32_t on_device);

/* Solve J(x_b) s = rhs by the library's right-preconditioned GMRES (after nks_pc_setup when
 * pc_type != NONE) to ||J s - rhs|| <= max(gmres_rtol ||rhs||, gmres_atol).  *its receives the
 * iteration count.  NKS_E_DIVERGED at gmres_maxit. */
NKS_API nks_status nks_gmres_solve(nks_state* st, double dt, const double* x_b, const double* rhs, double* s,
                           int32_t on_device, int32_t* its);

/* Counters of this state since creation: kernels issued by the library, host synchronisations, and
 * global reductions (each an allreduce on a sharded state): one per GMRES Arnoldi step (DCGS2, north_star
 * item 5), one per GMRES restart / Newton norm / energy / gauge / X'_d evaluation.  Any pointer may be NULL. */
NKS_API nks_status nks_counters(const nks_state* st, int64_t* kernel_launches, int64_t* host_syncs, int64_t* reductions);

/* Phase profiling with CUDA events recorded on the state's stream around every launch of a
 * phase: [0] residual F, [1] J.v, [2] RAS apply, [3] assembly, [4] BILU(0) factorisation,
 * [5] GMRES vector ops, [6] reductions (norms, energy, gauge), [7] other.
 * nks_set_profiling(st, 1) enables recording (it costs two event records per launch);
 * nks_phase_times synchronises the stream and returns accumulated ms and launch counts;
 * reset = 1 clears the accumulators afterwards. */
NKS_API nks_status nks_set_profiling(nks_state* st, int32_t enable);
NKS_API nks_status nks_phase_times(nks_state* st, double ms[8], int64_t counts[8], int32_t reset);

NKS_API nks_status nks_destroy(nks_state* st);

/* Message of the last failure on this state ("" if none); valid until the next call. */
NKS_API const char* nks_last_error(const nks_state* st);

/* Library version string. */
NKS_API const char* nks_version(void);

#ifdef __cplusplus
}
#endif

#endif /* NKS_H */
