// Library-owned communication of a z-sharded state: the NCCL
// communicator created in nks_create from the caller's unique id, halo exchanges as grouped
// ncclSend/ncclRecv on the state's stream, and fixed-order reductions (ncclAllGather of every rank's
// partial sums + a rank-ordered sum on the device, so every rank holds identical bits and takes the same
// control decisions -- reading R37).  Plus the host-only decomposition the ranks agree on.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "nks_internal.cuh"

namespace nks {

// ------------------------------------------------------------------------------------------ decomposition
// Rank r owns a contiguous run of the nsub[2] global box layers along z (the first nsub[2] mod nranks ranks
// one layer more), so every rank holds whole RAS boxes of the global box grid and the preconditioner -- hence
// the iteration counts -- does not depend on the number of ranks.  Without RAS the planes
// themselves are dealt out the same way.
static void deal(int n, int parts, int r, int& lo, int& len) {
  const int base = n / parts, rem = n % parts;
  lo = r * base + std::min(r, rem);
  len = base + (r < rem ? 1 : 0);
}

int slab_decompose(const nks_grid& global, int pc_type, int rank, int nranks, nks_grid& local, int& z_offset) {
  if (global.dim != 3 || global.zghost != 0 || nranks < 1 || rank < 0 || rank >= nranks) return 1;
  const int nz = global.n[2];
  int lo = 0, own = 0, nbz = 1;
  const bool ras = pc_type != NKS_PC_NONE;
  if (ras) {
    const int nsz = global.nsub[2];
    if (nsz < nranks) return 1;
    int b0, nb;
    deal(nsz, nranks, rank, b0, nb);
    // global box starts: the first nz mod nsz boxes one plane longer
    const int base = nz / nsz, rem = nz % nsz;
    auto start = [&](int b) { return b * base + std::min(b, rem); };
    lo = start(b0);
    own = start(b0 + nb) - lo;
    nbz = nb;
  } else {
    deal(nz, nranks, rank, lo, own);
  }
  const int zg = ras ? std::max(2, global.overlap + 1) : 2;
  if (own < 2 || zg > 8) return 1;
  local = global;
  local.n[2] = own + 2 * zg;
  local.zghost = zg;
  local.nsub[2] = nbz;
  z_offset = lo;
  return 0;
}

// Pencil of rank r = rz * py + ry on a pz x py process grid (z x y; x stays whole).  With RAS every rank owns
// whole layers of the global box grid along z AND y (nsub[2] layers dealt over pz, nsub[1] over py, as the
// slab deals its z layers), so the preconditioner -- and the iteration counts -- do not depend on the process
// grid; ghosts = max(2, overlap + 1) planes / rows per side.  Without RAS the planes and rows themselves are
// dealt out, 2 ghosts per side (the stencil radius of F and J.v).
int pencil_decompose(const nks_grid& global, int pc_type, int rank, int pz, int py, nks_grid& local) {
  if (global.dim != 3 || global.zghost != 0 || global.yghost != 0 || pz < 1 || py < 1 || rank < 0 || rank >= pz * py)
    return 1;
  const int rz = rank / py, ry = rank % py;
  const bool ras = pc_type != NKS_PC_NONE;
  int z0, nzo, y0, nyo, nbz = 1, nby = 1;
  auto layers = [&](int n, int nsub, int parts, int r, int& lo, int& own, int& nb) -> bool {
    if (nsub < parts) return false;
    int b0;
    deal(nsub, parts, r, b0, nb);
    const int base = n / nsub, rem = n % nsub;
    auto start = [&](int b) { return b * base + std::min(b, rem); };
    lo = start(b0);
    own = start(b0 + nb) - lo;
    return true;
  };
  if (ras) {
    if (!layers(global.n[2], global.nsub[2], pz, rz, z0, nzo, nbz)) return 1;
    if (!layers(global.n[1], global.nsub[1], py, ry, y0, nyo, nby)) return 1;
  } else {
    deal(global.n[2], pz, rz, z0, nzo);
    deal(global.n[1], py, ry, y0, nyo);
  }
  const int gh = ras ? std::max(2, global.overlap + 1) : 2;
  if (nzo < 2 || nyo < 2 || gh > 8) return 1;
  local = global;
  local.n[2] = nzo + 2 * gh;
  local.n[1] = nyo + 2 * gh;
  local.zghost = gh;
  local.yghost = gh;
  local.z_offset = z0;
  local.nz_global = global.n[2];
  local.y_offset = y0;
  local.ny_global = global.n[1];
  local.pz = pz;
  local.py = py;
  local.nsub[2] = nbz;
  local.nsub[1] = nby;
  if (!ras) local.nsub[0] = local.nsub[1] = local.nsub[2] = 1;
  return 0;
}

// Pencil halo plan: phase 1, per field, the y blocks of the own planes (kind 2 send / 3 receive: yg rows per
// own plane, packed plane after plane) with the y neighbours (rz, ry -+ 1); phase 2 the z planes -- whole
// local planes, ghost rows included, so the (y, z) edge cells arrive -- with the z neighbours (rz -+ 1, ry).
// Per peer the messages are matched in issue order, as in the slab plan (up == down for two parts).
void pencil_halo_plan(const nks_grid& g, int rank, int nf, std::vector<nks_halo_msg>& out) {
  const int pz = g.pz, py = g.py, rz = rank / py, ry = rank % py;
  const int nx = g.n[0], nyl = g.n[1], nzl = g.n[2], yg = g.yghost, zg = g.zghost;
  const long long nxy = (long long)nx * nyl, fstride = nxy * nzl;
  const int yup = rz * py + (ry + 1) % py, ydn = rz * py + (ry + py - 1) % py;
  const int zup = ((rz + 1) % pz) * py + ry, zdn = ((rz + pz - 1) % pz) * py + ry;
  const long long ycnt = (long long)yg * nx, zcnt = (long long)zg * nxy;
  out.clear();
  for (int f = 0; f < nf; ++f) {
    const long long b = (long long)f * fstride + (long long)zg * nxy;           // first own plane
    out.push_back({2, ydn, b + (long long)yg * nx, ycnt});                       // own rows lo -> ry-1's top ghosts
    out.push_back({2, yup, b + (long long)(nyl - 2 * yg) * nx, ycnt});           // own rows hi -> ry+1's bottom ghosts
    out.push_back({3, yup, b + (long long)(nyl - yg) * nx, ycnt});               // top ghost rows <- ry+1
    out.push_back({3, ydn, b, ycnt});                                            // bottom ghost rows <- ry-1
  }
  for (int f = 0; f < nf; ++f) {
    const long long base = (long long)f * fstride;
    out.push_back({0, zdn, base + (long long)zg * nxy, zcnt});
    out.push_back({0, zup, base + (long long)(nzl - 2 * zg) * nxy, zcnt});
    out.push_back({1, zup, base + (long long)(nzl - zg) * nxy, zcnt});
    out.push_back({1, zdn, base, zcnt});
  }
}

// ------------------------------------------------------------------------------------------ NCCL
struct NcclComm {
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
};

__global__ void k_rank_sum(const double* __restrict__ gathered, int nranks, long long n, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x) {
    double s = 0.0;
    for (int r = 0; r < nranks; ++r) s += gathered[(long long)r * n + i];     // rank order 0, 1, ...
    out[i] = s;
  }
}

int nccl_unique_id(uint8_t id[128]) {
  ncclUniqueId u;
  if (ncclGetUniqueId(&u) != ncclSuccess) return 1;
  static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
  std::memcpy(id, &u, 128);
  return 0;
}

void* nccl_create(const uint8_t id[128], int rank, int nranks, std::string& err) {
  NcclComm* C = new NcclComm();
  ncclUniqueId u;
  std::memcpy(&u, id, 128);
  const ncclResult_t r = ncclCommInitRank(&C->comm, nranks, u, rank);
  if (r != ncclSuccess) {
    err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
    delete C;
    return nullptr;
  }
  C->rank = rank;
  C->nranks = nranks;
  return C;
}

void nccl_destroy(void* c) {
  NcclComm* C = (NcclComm*)c;
  if (!C) return;
  ncclCommDestroy(C->comm);
  delete C;
}

// The halo exchange as an ordered message list (host only; exported as nks_halo_plan so that the CPU tests run
// the very same plan over gloo): per field, send the first own planes down, the last own planes up, receive the
// top ghosts from up, the bottom ghosts from down.  NCCL pairs the messages between two ranks in issue order,
// so with two ranks (up == down) the first send (own_lo) meets the peer's first receive (its top ghosts) and the
// second (own_hi) its second (its bottom ghosts) -- the planes the periodic neighbours need.
void halo_plan(int rank, int nranks, int nf, long long fstride, int nzl, long long nxy, int zg,
               std::vector<nks_halo_msg>& out) {
  const int up = (rank + 1) % nranks, dn = (rank + nranks - 1) % nranks;
  const long long cnt = (long long)zg * nxy;
  out.clear();
  for (int f = 0; f < nf; ++f) {
    const long long base = (long long)f * fstride;
    out.push_back({0, dn, base + (long long)zg * nxy, cnt});               // own_lo -> rank-1's top ghosts
    out.push_back({0, up, base + (long long)(nzl - 2 * zg) * nxy, cnt});   // own_hi -> rank+1's bottom ghosts
    out.push_back({1, up, base + (long long)(nzl - zg) * nxy, cnt});       // top ghosts <- rank+1's own_lo
    out.push_back({1, dn, base, cnt});                                     // bottom ghosts <- rank-1's own_hi
  }
}

// Fill the zg ghost planes on both z sides of nf fields (field f at vec + f * fstride, local (nzl, nxy)).
int nccl_halo(void* c, double* vec, int nf, long long fstride, int nzl, long long nxy, int zg, cudaStream_t s) {
  NcclComm* C = (NcclComm*)c;
  std::vector<nks_halo_msg> plan;
  halo_plan(C->rank, C->nranks, nf, fstride, nzl, nxy, zg, plan);
  if (ncclGroupStart() != ncclSuccess) return 1;
  for (const auto& m : plan) {
    const ncclResult_t r = m.kind == 0 ? ncclSend(vec + m.offset, (size_t)m.count, ncclDouble, m.peer, C->comm, s)
                                       : ncclRecv(vec + m.offset, (size_t)m.count, ncclDouble, m.peer, C->comm, s);
    if (r != ncclSuccess) {
      ncclGroupEnd();
      return 1;
    }
  }
  return ncclGroupEnd() == ncclSuccess ? 0 : 1;
}

// Pencil halo (plan above): y blocks are packed plane after plane into `stage` (cudaMemcpy2DAsync, one per
// message), exchanged in one NCCL group, unpacked; then the planes go as in the slab exchange.
int nccl_halo_pencil(void* c, const nks_grid& g, double* vec, int nf, double* stage, cudaStream_t s) {
  NcclComm* C = (NcclComm*)c;
  std::vector<nks_halo_msg> plan;
  pencil_halo_plan(g, C->rank, nf, plan);
  const long long nxy = (long long)g.n[0] * g.n[1];
  const int nzo = g.n[2] - 2 * g.zghost;
  const size_t pitch = (size_t)nxy * sizeof(double);
  std::vector<double*> st(plan.size(), nullptr);
  double* p = stage;
  for (size_t k = 0; k < plan.size(); ++k) {
    if (plan[k].kind < 2) continue;
    st[k] = p;
    p += plan[k].count * nzo;
    if (plan[k].kind == 2 &&
        cudaMemcpy2DAsync(st[k], plan[k].count * sizeof(double), vec + plan[k].offset, pitch, plan[k].count * sizeof(double),
                          nzo, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return 1;
  }
  if (ncclGroupStart() != ncclSuccess) return 1;
  for (size_t k = 0; k < plan.size(); ++k) {
    const auto& m = plan[k];
    if (m.kind < 2) continue;
    const size_t n = (size_t)m.count * nzo;
    const ncclResult_t r = m.kind == 2 ? ncclSend(st[k], n, ncclDouble, m.peer, C->comm, s)
                                       : ncclRecv(st[k], n, ncclDouble, m.peer, C->comm, s);
    if (r != ncclSuccess) { ncclGroupEnd(); return 1; }
  }
  if (ncclGroupEnd() != ncclSuccess) return 1;
  for (size_t k = 0; k < plan.size(); ++k)
    if (plan[k].kind == 3 &&
        cudaMemcpy2DAsync(vec + plan[k].offset, pitch, st[k], plan[k].count * sizeof(double), plan[k].count * sizeof(double),
                          nzo, cudaMemcpyDeviceToDevice, s) != cudaSuccess)
      return 1;
  if (ncclGroupStart() != ncclSuccess) return 1;
  for (const auto& m : plan) {
    if (m.kind > 1) continue;
    const ncclResult_t r = m.kind == 0 ? ncclSend(vec + m.offset, (size_t)m.count, ncclDouble, m.peer, C->comm, s)
                                       : ncclRecv(vec + m.offset, (size_t)m.count, ncclDouble, m.peer, C->comm, s);
    if (r != ncclSuccess) { ncclGroupEnd(); return 1; }
  }
  return ncclGroupEnd() == ncclSuccess ? 0 : 1;
}

// buf[0..n) <- sum over ranks in rank order (gather: nranks * n doubles of workspace).
int nccl_allreduce_fixed(void* c, double* buf, long long n, double* gather, cudaStream_t s) {
  NcclComm* C = (NcclComm*)c;
  if (C->nranks == 1) return 0;
  if (ncclAllGather(buf, gather, (size_t)n, ncclDouble, C->comm, s) != ncclSuccess) return 1;
  k_rank_sum<<<1, 256, 0, s>>>(gather, C->nranks, n, buf);
  return cudaGetLastError() == cudaSuccess ? 0 : 1;
}

}  // namespace nks
