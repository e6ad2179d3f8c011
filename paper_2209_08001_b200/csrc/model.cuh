// Pointwise physics of scheme NSOA-1 on the device (fp64).
//
// G^1 (App. B), G^{2,S} (Eq. D2-1) with the Psi_S quotient of
// P:452-456 evaluated in closed form: only odd Taylor orders survive the antisymmetric
// difference, so Psi_S[y1,y2] = ln(ybar/(1-ybar)) + P(D/(1-ybar)^2) - P(D/ybar^2) with
// D = delta^2 and P(x) = sum_{k=1}^{S-1} x^k / (2k(2k+1)) (Horner), one log and two reciprocals.
#pragma once

#include "nks_internal.cuh"

namespace nks {

// Horner evaluation of P(x) = sum_{k=1}^{S-1} c_k x^k and P'(x).
__device__ __forceinline__ void horner_P(const DevParams& P, double x, double& p, double& dp) {
  const int K = P.S - 1;
  double acc = 0.0, dacc = 0.0;
  for (int k = K; k >= 1; --k) {
    dacc = fma(dacc, x, acc);           // derivative of the running polynomial
    acc = fma(acc, x, P.pcoef[k - 1]);
  }
  // acc = sum_{k>=1} c_k x^(k-1); p = x*acc; dp = acc + x*dacc
  p = acc * x;
  dp = fma(dacc, x, acc);
}

__device__ __forceinline__ double horner_only(const DevParams& P, double x) {
  const int K = P.S - 1;
  double acc = 0.0;
  for (int k = K; k >= 1; --k) acc = fma(acc, x, P.pcoef[k - 1]);
  return acc * x;
}

// P(x) with the trip count fixed at compile time (S = 10, the paper's order): the loop
// unrolls, so the six Horner chains of a point (three Psi_S, two arguments each) interleave.
template <int K>
__device__ __forceinline__ double horner_fixed(const DevParams& P, double x) {
  double acc = 0.0;
#pragma unroll
  for (int k = K; k >= 1; --k) acc = fma(acc, x, P.pcoef[k - 1]);
  return acc * x;
}

// Psi_S[y_b, y_a] (symmetric in its arguments).  One division for both reciprocals:
// 1/ybar = (1-ybar) r, 1/(1-ybar) = ybar r with r = 1/(ybar (1-ybar)).
__device__ __forceinline__ double psiS(const DevParams& P, double ya, double yb) {
  const double ybar = 0.5 * (ya + yb);
  const double e = 0.5 * (yb - ya);
  const double D = e * e;
  const double zbar = 1.0 - ybar;
  const double rr = 1.0 / (ybar * zbar);
  const double iy = zbar * rr;
  const double iz = ybar * rr;
  const double a = D * iy * iy, b = D * iz * iz;
  if (P.S == 10) return log(ybar * iz) + horner_fixed<9>(P, b) - horner_fixed<9>(P, a);
  return log(ybar * iz) + horner_only(P, b) - horner_only(P, a);
}

template <int K>
__device__ __forceinline__ void horner_P_fixed(const DevParams& P, double x, double& p, double& dp) {
  double acc = 0.0, dacc = 0.0;
#pragma unroll
  for (int k = K; k >= 1; --k) {
    dacc = fma(dacc, x, acc);
    acc = fma(acc, x, P.pcoef[k - 1]);
  }
  p = acc * x;
  dp = fma(dacc, x, acc);
}

// Psi_S and its derivative with respect to the level-b argument y_b.
__device__ __forceinline__ void psiS_d(const DevParams& P, double ya, double yb, double& val, double& dval) {
  const double ybar = 0.5 * (ya + yb);
  const double e = 0.5 * (yb - ya);
  const double D = e * e;
  const double zbar = 1.0 - ybar;
  const double rr = 1.0 / (ybar * zbar);
  const double iy = zbar * rr;
  const double iz = ybar * rr;
  const double iy2 = iy * iy, iz2 = iz * iz;
  const double a = D * iy2, b = D * iz2;
  double pa, dpa, pb, dpb;
  if (P.S == 10) {
    horner_P_fixed<9>(P, a, pa, dpa);
    horner_P_fixed<9>(P, b, pb, dpb);
  } else {
    horner_P(P, a, pa, dpa);
    horner_P(P, b, pb, dpb);
  }
  val = log(ybar * iz) + pb - pa;
  // d/dy_b = 1/2 d/dybar + e d/dD
  dval = 0.5 * iy * iz + dpb * b * iz + dpa * a * iy + e * (dpb * iz2 - dpa * iy2);
}

__device__ __forceinline__ double M1f(const DevParams& P, double phi) { return fma(P.m1b, phi * phi, P.m1a); }
__device__ __forceinline__ double M2f(const DevParams& P, double phi) {
  return P.m2a + phi * phi * fma(P.m2c, phi, P.m2b);
}
__device__ __forceinline__ double M5f(const DevParams& P, double c) { return c * c * fma(P.m5b, c, P.m5a); }
__device__ __forceinline__ double M6f(const DevParams& P, double c) { return P.m6 * c * c * c; }

// Pointwise G^1 + G^{2,S} (c and eta components).
__device__ __forceinline__ void pointwise_G(const DevParams& P, double ca, double cb, double ea, double eb,
                                            double& gc, double& ge) {
  const double pa = 1.0 - ea, pb = 1.0 - eb;
  const double ch = 0.5 * (ca + cb), phih = 0.5 * (pa + pb), eh = 0.5 * (ea + eb);
  const double q3 = fma(cb, cb + ca, ca * ca);                         // cb^2 + cb ca + ca^2
  const double q4 = (cb + ca) * fma(cb, cb, ca * ca);                  // (cb+ca)(cb^2+ca^2)
  const double q5 = fma(cb, q4, ca * ca * ca * ca);                    // cb*q4 + ca^4
  const double g1c = 0.5 * (M1f(P, pa) + M1f(P, pb)) * ch + (M2f(P, pa) + M2f(P, pb)) * (1.0 / 6.0) * q3 +
                     0.25 * P.M3 * q4 + 0.2 * P.M4 * q5 + P.M0;
  const double r3 = fma(pb, pb + pa, pa * pa);
  const double g1e = 0.5 * (M5f(P, ca) + M5f(P, cb)) * phih + (M6f(P, ca) + M6f(P, cb)) * (1.0 / 6.0) * r3;
  const double Pc = psiS(P, ca, cb);
  const double Pp = psiS(P, ca * ea, cb * eb);
  const double Pq = psiS(P, ca * (4.0 - 3.0 * ea), cb * (4.0 - 3.0 * eb));
  const double t4 = 0.25 * P.theta;
  gc = g1c + t4 * (4.0 * P.w_c * Pc + 3.0 * eh * Pp + (4.0 - 3.0 * eh) * Pq);
  ge = g1e + t4 * 3.0 * ch * (Pp - Pq);
}

// Pointwise partial derivatives a_kl = d(G^1 + G^{2,S})_k / d(c^b, eta^b)_l.
__device__ __forceinline__ void pointwise_dG(const DevParams& P, double ca, double cb, double ea, double eb,
                                             double& a11, double& a12, double& a21, double& a22) {
  const double pa = 1.0 - ea, pb = 1.0 - eb;
  const double ch = 0.5 * (ca + cb), phih = 0.5 * (pa + pb), eh = 0.5 * (ea + eb);
  const double q3 = fma(cb, cb + ca, ca * ca);
  // G^1 part
  const double dq3 = 2.0 * cb + ca;
  const double dq4 = cb * (3.0 * cb + 2.0 * ca) + ca * ca;
  const double dq5 = cb * cb * (4.0 * cb + 3.0 * ca) + ca * ca * (2.0 * cb + ca);
  double g11 = 0.25 * (M1f(P, pa) + M1f(P, pb)) + (M2f(P, pa) + M2f(P, pb)) * (1.0 / 6.0) * dq3 +
               0.25 * P.M3 * dq4 + 0.2 * P.M4 * dq5;
  const double dM1 = 2.0 * P.m1b * pb;
  const double dM2 = pb * fma(3.0 * P.m2c, pb, 2.0 * P.m2b);
  double g12 = -(0.5 * dM1 * ch + (1.0 / 6.0) * dM2 * q3);
  const double r3 = fma(pb, pb + pa, pa * pa);
  const double dM5 = cb * fma(3.0 * P.m5b, cb, 2.0 * P.m5a);
  const double dM6 = 3.0 * P.m6 * cb * cb;
  double g21 = 0.5 * dM5 * phih + (1.0 / 6.0) * dM6 * r3;
  double g22 = -(0.25 * (M5f(P, ca) + M5f(P, cb)) + (M6f(P, ca) + M6f(P, cb)) * (1.0 / 6.0) * (2.0 * pb + pa));
  // G^{2,S} part
  const double qa_ = ca * (4.0 - 3.0 * ea), qb_ = cb * (4.0 - 3.0 * eb);
  double Pc, dPc, Pp, dPp, Pq, dPq;
  psiS_d(P, ca, cb, Pc, dPc);
  psiS_d(P, ca * ea, cb * eb, Pp, dPp);
  psiS_d(P, qa_, qb_, Pq, dPq);
  const double t4 = 0.25 * P.theta;
  const double fb = 4.0 - 3.0 * eb, fh = 4.0 - 3.0 * eh;
  g11 += t4 * (4.0 * P.w_c * dPc + 3.0 * eh * dPp * eb + fh * dPq * fb);
  g12 += t4 * (1.5 * Pp + 3.0 * eh * dPp * cb - 1.5 * Pq - 3.0 * fh * dPq * cb);
  g21 += t4 * 3.0 * (0.5 * (Pp - Pq) + ch * (dPp * eb - dPq * fb));
  g22 += t4 * 3.0 * ch * cb * (dPp + 3.0 * dPq);
  a11 = g11; a12 = g12; a21 = g21; a22 = g22;
}

__device__ __forceinline__ double psi_fn(double z) { return z * log(z) + (1.0 - z) * log1p(-z); }

// E1 + E2 at a point: Phi via the antiderivative of App. B's dE_G/dc at fixed phi.
__device__ __forceinline__ void local_energy(const DevParams& P, double c, double eta, double& e1, double& e2) {
  const double phi = 1.0 - eta;
  const double c2 = c * c;
  e1 = c * (P.M0 + c * (0.5 * M1f(P, phi) + c * ((1.0 / 3.0) * M2f(P, phi) + c * (0.25 * P.M3 + 0.2 * P.M4 * c))));
  (void)c2;
  e2 = P.theta * (P.w_c * psi_fn(c) + 0.75 * psi_fn(c * eta) + 0.25 * psi_fn(c * (4.0 - 3.0 * eta)));
}

}  // namespace nks
