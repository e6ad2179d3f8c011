// Initial mechanical equilibrium u^0 (a0 of SURVEY 8(a); reading R13): solve the discrete
// equilibrium [D^ sigma^el(u, c^0)] = 0 once per run.  With periodic boundaries the
// central-difference operator is diagonalised by the DFT: D^_J -> i s_J, s_J = sin(k_J h)/h, so
// per wavenumber the d x d system
//   sum_M A_IM u^_M = i s_I Lscale K eps0 rho^,   A_II = -L(C11 s_I^2 + C44 sum_{J!=I} s_J^2),
//                                                 A_IM = -L(C12 + C44) s_I s_M   (I != M)
// is solved in closed form; modes with every s_J = 0 are the gauge null space (set to zero).
// fp64 cuFFT (library primitive, init only -- not on the per-step hot path).
#include <cufft.h>

#include "nks_internal.cuh"

namespace nks {

__global__ void k_rho(long long N, const double* __restrict__ c, double cbar, cufftDoubleComplex* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    out[i] = make_cuDoubleComplex(c[i] - cbar, 0.0);
}

__global__ void k_symbol_solve(DevParams P, const cufftDoubleComplex* __restrict__ rho, cufftDoubleComplex* __restrict__ u0,
                               cufftDoubleComplex* __restrict__ u1, cufftDoubleComplex* __restrict__ u2) {
  const double two_pi = 6.283185307179586476925286766559;
  const int d = P.dim;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < P.N; i += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(i % P.nx), y = (int)((i / P.nx) % P.ny), z = (int)(i / ((long long)P.nx * P.ny));
    double s[3] = {sin(two_pi * x / P.nx) / P.h, sin(two_pi * y / P.ny) / P.h, d == 3 ? sin(two_pi * z / P.nz) / P.h : 0.0};
    // exact zeros for k = 0 and k = pi (sin of an exact multiple of pi may round to ~1e-16)
    if (x == 0 || 2 * x == P.nx) s[0] = 0.0;
    if (y == 0 || 2 * y == P.ny) s[1] = 0.0;
    if (d < 3 || z == 0 || 2 * z == P.nz) s[2] = 0.0;
    const cufftDoubleComplex r = rho[i];
    const double f = P.K * P.eps0;     // Lscale * K' * eps0
    // rhs_I = i s_I f rho
    double br[3], bi[3];
    for (int I = 0; I < 3; ++I) { br[I] = -s[I] * f * r.y; bi[I] = s[I] * f * r.x; }
    double A[3][3];
    for (int I = 0; I < 3; ++I)
      for (int M = 0; M < 3; ++M) {
        if (I >= d || M >= d) { A[I][M] = (I == M) ? 1.0 : 0.0; continue; }
        if (I == M) {
          double o = 0.0;
          for (int J = 0; J < d; ++J) if (J != I) o += s[J] * s[J];
          A[I][M] = -P.Ls * (P.C11 * s[I] * s[I] + P.C44 * o);
        } else {
          A[I][M] = -P.Ls * (P.C12 + P.C44) * s[I] * s[M];
        }
      }
    double ur[3] = {0, 0, 0}, ui[3] = {0, 0, 0};
    const bool null = s[0] == 0.0 && s[1] == 0.0 && s[2] == 0.0;
    if (!null) {
      // Cramer's rule on the (real symmetric) 3x3 (identity-padded in 2D)
      const double det = A[0][0] * (A[1][1] * A[2][2] - A[1][2] * A[2][1]) - A[0][1] * (A[1][0] * A[2][2] - A[1][2] * A[2][0]) +
                         A[0][2] * (A[1][0] * A[2][1] - A[1][1] * A[2][0]);
      double inv[3][3];
      inv[0][0] = (A[1][1] * A[2][2] - A[1][2] * A[2][1]) / det;
      inv[0][1] = (A[0][2] * A[2][1] - A[0][1] * A[2][2]) / det;
      inv[0][2] = (A[0][1] * A[1][2] - A[0][2] * A[1][1]) / det;
      inv[1][0] = (A[1][2] * A[2][0] - A[1][0] * A[2][2]) / det;
      inv[1][1] = (A[0][0] * A[2][2] - A[0][2] * A[2][0]) / det;
      inv[1][2] = (A[0][2] * A[1][0] - A[0][0] * A[1][2]) / det;
      inv[2][0] = (A[1][0] * A[2][1] - A[1][1] * A[2][0]) / det;
      inv[2][1] = (A[0][1] * A[2][0] - A[0][0] * A[2][1]) / det;
      inv[2][2] = (A[0][0] * A[1][1] - A[0][1] * A[1][0]) / det;
      for (int I = 0; I < 3; ++I)
        for (int M = 0; M < 3; ++M) { ur[I] += inv[I][M] * br[M]; ui[I] += inv[I][M] * bi[M]; }
    }
    u0[i] = make_cuDoubleComplex(ur[0], ui[0]);
    u1[i] = make_cuDoubleComplex(ur[1], ui[1]);
    if (d == 3) u2[i] = make_cuDoubleComplex(ur[2], ui[2]);
  }
}

__global__ void k_real_part(long long N, const cufftDoubleComplex* __restrict__ in, double scale, double* __restrict__ out) {
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i].x * scale;
}

// Computes u^0 into u (d*N doubles) from c; scratch >= (d+1)*N complex.  Returns 0 on success.
int init_displacement_fft(const DevParams& P, const double* c, double* u, void* scratch, cudaStream_t s, std::string& err) {
  const long long N = P.N;
  cufftDoubleComplex* rho = (cufftDoubleComplex*)scratch;
  cufftDoubleComplex* uh[3] = {rho + N, rho + 2 * N, rho + 3 * N};
  cufftHandle plan;
  cufftResult r = P.dim == 2 ? cufftPlan2d(&plan, P.ny, P.nx, CUFFT_Z2Z) : cufftPlan3d(&plan, P.nz, P.ny, P.nx, CUFFT_Z2Z);
  if (r != CUFFT_SUCCESS) { err = "cufftPlan failed: " + std::to_string((int)r); return 1; }
  cufftSetStream(plan, s);
  const int blocks = (int)std::min<long long>((N + 255) / 256, 148 * 16);
  k_rho<<<blocks, 256, 0, s>>>(N, c, P.cbar0, rho);
  r = cufftExecZ2Z(plan, rho, rho, CUFFT_FORWARD);
  if (r != CUFFT_SUCCESS) { cufftDestroy(plan); err = "cufftExecZ2Z forward failed"; return 1; }
  k_symbol_solve<<<blocks, 256, 0, s>>>(P, rho, uh[0], uh[1], uh[2]);
  for (int I = 0; I < P.dim; ++I) {
    r = cufftExecZ2Z(plan, uh[I], uh[I], CUFFT_INVERSE);
    if (r != CUFFT_SUCCESS) { cufftDestroy(plan); err = "cufftExecZ2Z inverse failed"; return 1; }
    k_real_part<<<blocks, 256, 0, s>>>(N, uh[I], 1.0 / (double)N, u + I * N);
  }
  cudaStreamSynchronize(s);
  cufftDestroy(plan);
  return 0;
}

}  // namespace nks
