// Spectral (mean-coefficient Fourier) preconditioner of the Newton systems -- a B200-native
// alternative to the paper's one-level Schwarz preconditioners, kept beside them
// (nks_params.pc_type = NKS_PC_SPECTRAL).
//
// J (its rows in SURVEY 8(c).1 step 8) has three variable coefficients: the pointwise partials
// a_kl of G1 + G2S and the level-n face mobility M~.  With each replaced by its grid mean, J is
// translation invariant on the periodic grid, so the DFT diagonalises it into one (2+d) x (2+d)
// complex matrix per wave number k:
//   D^_J -> i s_J,  s_J = sin(k_J h)/h;     Lap_h -> -lam,  lam = sum_J (2 - 2 cos k_J h)/h^2;
//   c row:   v_c/dt + Mbar lam [ (a11 + (eps0 K d eps0)/2 + gamma_c lam/2) v_c + a12 v_eta
//                                - (eps0 K/2) sum_J i s_J v_uJ ]
//   eta row: a21 v_c + (1/dt + a22 + 3 gamma_eta lam/2) v_eta
//   u_I row: -i s_I K eps0 v_c + sum_M A_IM v_uM,  A_II = -L(C11 s_I^2 + C44 sum_{J!=I} s_J^2),
//            A_IM = -L(C12 + C44) s_I s_M
// (K = L(C11 + (d-1)C12)).  The preconditioner applies the inverse of that matrix per wave number:
// real-to-complex FFT of the nf fields (cuFFT, one batched plan), one fused per-k multiply by the stored
// inverse (1/N folded in), complex-to-real FFT.  On the gauge modes (every s_J = 0, reading R14) the u
// block is singular; the preconditioned u is zero there, so every Krylov vector stays in the gauge.
// The inverse is rebuilt whenever the preconditioner is set up (pc_reuse decides how often); it only
// steers GMRES -- the converged Newton step is the same root (tests/test_gpu_parity.py).
#include <cufft.h>

#include "nks_internal.cuh"

namespace nks {

// sums of a11, a12, a21, a22 and of m = c^a (1 - c^a) over the (own) points -> part[block][5]
__global__ void k_spec_sums(DevParams P, const double* __restrict__ Xa, const double* __restrict__ jac4,
                            double* __restrict__ part) {
  __shared__ double sred[5][kRedThreads / 32];
  double acc[5] = {0, 0, 0, 0, 0};
  const long long N = P.N;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < N; i += (long long)gridDim.x * blockDim.x) {
    acc[0] += jac4[i];
    acc[1] += jac4[N + i];
    acc[2] += jac4[2 * N + i];
    acc[3] += jac4[3 * N + i];
    const double c = Xa[i];
    acc[4] += c * (1.0 - c);
  }
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int k = 0; k < 5; ++k) {
    double v = acc[k];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_down_sync(0xffffffffu, v, o);
    if (lane == 0) sred[k][wid] = v;
  }
  __syncthreads();
  if (threadIdx.x < 5) {
    double v = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) v += sred[threadIdx.x][w];
    part[blockIdx.x * 5 + threadIdx.x] = v;
  }
}

__global__ void k_spec_means(const double* __restrict__ part, int nb, double inv_n, double* __restrict__ out) {
  if (threadIdx.x < 5) {
    double v = 0.0;
    for (int b = 0; b < nb; ++b) v += part[b * 5 + threadIdx.x];     // fixed order
    out[threadIdx.x] = v * inv_n;
  }
}

struct cplx {
  double re, im;
};
__device__ __forceinline__ cplx cmul(cplx a, cplx b) { return {a.re * b.re - a.im * b.im, a.re * b.im + a.im * b.re}; }
__device__ __forceinline__ cplx csub(cplx a, cplx b) { return {a.re - b.re, a.im - b.im}; }
__device__ __forceinline__ cplx cdivv(cplx a, cplx b) {
  const double den = b.re * b.re + b.im * b.im;
  return {(a.re * b.re + a.im * b.im) / den, (a.im * b.re - a.re * b.im) / den};
}

// Per wave number of the half spectrum (x: 0..nx/2): build the mean-coefficient symbol and store its
// inverse / N at pinv[(row * NF + col) * Nh + k].
template <int NF>
__global__ void k_spec_build(DevParams P, const double* __restrict__ means, int nxh, long long Nh,
                             cufftDoubleComplex* __restrict__ pinv) {
  const double two_pi = 6.283185307179586476925286766559;
  const int d = NF - 2;
  const double a11 = means[0], a12 = means[1], a21 = means[2], a22 = means[3];
  const double Mbar = P.kappa * means[4];
  const double invN = 1.0 / (double)P.N;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < Nh; t += (long long)gridDim.x * blockDim.x) {
    const int x = (int)(t % nxh), y = (int)((t / nxh) % P.ny), z = (int)(t / ((long long)nxh * P.ny));
    const int kk[3] = {x, y, z};
    const int nn[3] = {P.nx, P.ny, P.nz};
    double s[3] = {0, 0, 0}, lam = 0.0;
    bool null = true;
    for (int J = 0; J < d; ++J) {
      const double th = two_pi * kk[J] / nn[J];
      s[J] = (kk[J] == 0 || 2 * kk[J] == nn[J]) ? 0.0 : sin(th) / P.h;     // exact zeros at 0 and pi
      lam += (2.0 - 2.0 * cos(th)) * P.inv_h2;
      if (s[J] != 0.0) null = false;
    }
    cplx A[NF][NF];
    for (int r = 0; r < NF; ++r)
      for (int c = 0; c < NF; ++c) A[r][c] = {0.0, 0.0};
    const double K = P.K;
    A[0][0] = {P.inv_dt + Mbar * lam * (a11 + 0.5 * P.eps0 * K * d * P.eps0 + 0.5 * P.gamma_c * lam), 0.0};
    A[0][1] = {Mbar * lam * a12, 0.0};
    for (int J = 0; J < d; ++J) A[0][2 + J] = {0.0, -Mbar * lam * 0.5 * P.eps0 * K * s[J]};
    A[1][0] = {a21, 0.0};
    A[1][1] = {P.inv_dt + a22 + 1.5 * P.gamma_eta * lam, 0.0};
    for (int I = 0; I < d; ++I) {
      A[2 + I][0] = {0.0, -s[I] * K * P.eps0};
      for (int M = 0; M < d; ++M) {
        double v;
        if (I == M) {
          double o = 0.0;
          for (int J = 0; J < d; ++J)
            if (J != I) o += s[J] * s[J];
          v = -P.Ls * (P.C11 * s[I] * s[I] + P.C44 * o);
        } else {
          v = -P.Ls * (P.C12 + P.C44) * s[I] * s[M];
        }
        A[2 + I][2 + M] = {v, 0.0};
      }
    }
    // gauge modes: periodic -- u block -> I, zeroed below; Neumann (reading R38) -- the Fourier modes are not
    // its eigenvectors and its gauge is not the parity classes: a regular stand-in of the elastic diagonal's
    // scale, nothing zeroed (the preconditioner is approximate there, which only costs GMRES iterations)
    if (null)
      for (int I = 0; I < d; ++I) A[2 + I][2 + I] = {P.bc ? -P.Ls * P.C11 * P.inv_h2 : 1.0, 0.0};
    // Gauss-Jordan with partial pivoting on the complex NF x NF matrix
    cplx B[NF][NF];
    for (int r = 0; r < NF; ++r)
      for (int c = 0; c < NF; ++c) B[r][c] = {r == c ? 1.0 : 0.0, 0.0};
    for (int k = 0; k < NF; ++k) {
      int piv = k;
      double best = A[k][k].re * A[k][k].re + A[k][k].im * A[k][k].im;
      for (int r = k + 1; r < NF; ++r) {
        const double m = A[r][k].re * A[r][k].re + A[r][k].im * A[r][k].im;
        if (m > best) { best = m; piv = r; }
      }
      if (piv != k)
        for (int c = 0; c < NF; ++c) {
          cplx tmp = A[k][c]; A[k][c] = A[piv][c]; A[piv][c] = tmp;
          tmp = B[k][c]; B[k][c] = B[piv][c]; B[piv][c] = tmp;
        }
      const cplx p = A[k][k];
      for (int c = 0; c < NF; ++c) { A[k][c] = cdivv(A[k][c], p); B[k][c] = cdivv(B[k][c], p); }
      for (int r = 0; r < NF; ++r) {
        if (r == k) continue;
        const cplx f = A[r][k];
        for (int c = 0; c < NF; ++c) { A[r][c] = csub(A[r][c], cmul(f, A[k][c])); B[r][c] = csub(B[r][c], cmul(f, B[k][c])); }
      }
    }
    for (int r = 0; r < NF; ++r)
      for (int c = 0; c < NF; ++c) {
        const bool zero = null && !P.bc && (r >= 2 || c >= 2);
        pinv[(long long)(r * NF + c) * Nh + t] = zero ? make_cuDoubleComplex(0.0, 0.0)
                                                      : make_cuDoubleComplex(B[r][c].re * invN, B[r][c].im * invN);
      }
  }
}

// zh_r(k) = sum_c pinv_rc(k) rh_c(k), in place on the [NF][Nh] spectrum
template <int NF>
__global__ void k_spec_mul(long long Nh, const cufftDoubleComplex* __restrict__ pinv, cufftDoubleComplex* __restrict__ h) {
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < Nh; t += (long long)gridDim.x * blockDim.x) {
    cplx v[NF];
#pragma unroll
    for (int c = 0; c < NF; ++c) {
      const cufftDoubleComplex q = h[c * Nh + t];
      v[c] = {q.x, q.y};
    }
#pragma unroll
    for (int r = 0; r < NF; ++r) {
      double re = 0.0, im = 0.0;
#pragma unroll
      for (int c = 0; c < NF; ++c) {
        const cufftDoubleComplex m = __ldg(pinv + (long long)(r * NF + c) * Nh + t);
        re = fma(m.x, v[c].re, fma(-m.y, v[c].im, re));
        im = fma(m.x, v[c].im, fma(m.y, v[c].re, im));
      }
      h[r * Nh + t] = make_cuDoubleComplex(re, im);
    }
  }
}

struct SpecPlan {
  cufftHandle fwd = 0, inv = 0;
  long long Nh = 0;
  int nxh = 0;
};

long long spectral_half(const nks_grid& g) { return (long long)(g.n[0] / 2 + 1) * g.n[1] * g.n[2]; }

void* spectral_plan(const nks_grid& g, int nf, cudaStream_t s, std::string& err) {
  SpecPlan* P = new SpecPlan();
  P->nxh = g.n[0] / 2 + 1;
  P->Nh = spectral_half(g);
  int n[3], rank = g.dim;
  if (g.dim == 2) { n[0] = g.n[1]; n[1] = g.n[0]; }
  else { n[0] = g.n[2]; n[1] = g.n[1]; n[2] = g.n[0]; }
  const int N = g.n[0] * g.n[1] * g.n[2];
  const int Nh = (int)P->Nh;
  cufftResult r = cufftPlanMany(&P->fwd, rank, n, nullptr, 1, N, nullptr, 1, Nh, CUFFT_D2Z, nf);
  if (r == CUFFT_SUCCESS) r = cufftPlanMany(&P->inv, rank, n, nullptr, 1, Nh, nullptr, 1, N, CUFFT_Z2D, nf);
  if (r != CUFFT_SUCCESS) {
    err = "cufftPlanMany failed: " + std::to_string((int)r);
    if (P->fwd) cufftDestroy(P->fwd);
    delete P;
    return nullptr;
  }
  cufftSetStream(P->fwd, s);
  cufftSetStream(P->inv, s);
  return P;
}

void spectral_free(void* p) {
  SpecPlan* P = (SpecPlan*)p;
  if (!P) return;
  cufftDestroy(P->fwd);
  cufftDestroy(P->inv);
  delete P;
}

// Rebuild the per-k inverse from the current level-n state and pointwise partials (jac4).
void launch_spectral_setup(void* plan, const DevParams& dp, int nf, const double* Xa, const double* jac4, double* part,
                           double* means, void* pinv, cudaStream_t s) {
  SpecPlan* P = (SpecPlan*)plan;
  const int nb = (int)std::min<long long>((dp.N + kRedThreads - 1) / kRedThreads, kRedBlocks);
  k_spec_sums<<<nb, kRedThreads, 0, s>>>(dp, Xa, jac4, part);
  k_spec_means<<<1, 32, 0, s>>>(part, nb, 1.0 / (double)dp.N, means);
  const int blocks = (int)std::min<long long>((P->Nh + 127) / 128, 148 * 8);
  if (nf == 4) k_spec_build<4><<<blocks, 128, 0, s>>>(dp, means, P->nxh, P->Nh, (cufftDoubleComplex*)pinv);
  else k_spec_build<5><<<blocks, 128, 0, s>>>(dp, means, P->nxh, P->Nh, (cufftDoubleComplex*)pinv);
}

// z = M^-1 r: the cuFFT transforms read r / write z; spec = [nf][Nh] complex scratch.
int launch_spectral_apply(void* plan, int nf, const double* r, double* z, const void* pinv, void* spec, cudaStream_t s) {
  SpecPlan* P = (SpecPlan*)plan;
  cufftDoubleComplex* h = (cufftDoubleComplex*)spec;
  if (cufftExecD2Z(P->fwd, const_cast<double*>(r), h) != CUFFT_SUCCESS) return 1;
  const int blocks = (int)std::min<long long>((P->Nh + 255) / 256, 148 * 8);
  if (nf == 4) k_spec_mul<4><<<blocks, 256, 0, s>>>(P->Nh, (const cufftDoubleComplex*)pinv, h);
  else k_spec_mul<5><<<blocks, 256, 0, s>>>(P->Nh, (const cufftDoubleComplex*)pinv, h);
  if (cufftExecZ2D(P->inv, h, z) != CUFFT_SUCCESS) return 1;
  return 0;
}

}  // namespace nks
