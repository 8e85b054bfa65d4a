// device_math.cuh -- FP64 device helpers of the sm_100a hot path.
//
// Everything here is the CUDA side's own arithmetic; it
// shares nothing with oracle/.  Citations are PAPER.md lines.
#pragma once
#include <cstdint>

#include "sfactor_coeffs.inc"

namespace ser {

constexpr double kPi = 3.14159265358979323846;
constexpr double kInvSqrtPi = 0.56418958354775628695;   // 1/sqrt(pi)
constexpr double kTwoOverSqrtPi = 1.12837916709551257390;  // 2/sqrt(pi)

// 1/sqrt(x) for finite x > 0: MUFU.RSQ64H seed (~2^-20 relative) + one
// third-order Newton correction y(1 + e/2 + 3e^2/8), e = 1 - x y^2: 5 FP64
// instructions, no special-case branch (callers guarantee x > 0 finite or
// discard the result).  Max relative error measured 1.1e-16 (tools/probes).
__device__ __forceinline__ double rsqrt_nr(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  const double p = fma(e, 0.375, 0.5);
  return fma(y * e, p, y);
}

// I0, I2 of eqs. (18)-(19), PAPER.md:114-121 (|lambda| per the paper).
__device__ __forceinline__ void I0_I2(double lam, double& I0, double& I2) {
  const double a = fabs(lam);
  const double e = exp(-lam * lam) * kInvSqrtPi;
  const double ec = erfc(a);
  I0 = e - a * ec;
  I2 = (2.0 / 3.0) * ((0.5 - lam * lam) * e + a * a * a * ec);
}

// Extrapolation weights: u = sum_k w_k u^{delta_k} solves eq. (17)
// with rows A_k = [1, rho_k I0(lambda_k), rho_k^3 I2(lambda_k)],
// lambda_k = b/delta_k.  w = first row of A^{-1} = cofactors of column 1 / det
// (R6).  |b| > cutoff*delta_3 (no near pairs: all u^{delta_k} equal)
// or a singular A return (1, 0, 0) (R7).
__device__ __forceinline__ void extrap_weights(double b, double h, const double rho[3], double cutoff,
                                               double w[3]) {
  w[0] = 1.0; w[1] = 0.0; w[2] = 0.0;
  if (fabs(b) > cutoff * rho[2] * h) return;
  double a2[3], a3[3];
#pragma unroll
  for (int k = 0; k < 3; ++k) {
    double I0, I2;
    I0_I2(b / (rho[k] * h), I0, I2);
    a2[k] = rho[k] * I0;
    a3[k] = rho[k] * rho[k] * rho[k] * I2;
  }
  const double c0 = a2[1] * a3[2] - a3[1] * a2[2];
  const double c1 = a3[0] * a2[2] - a2[0] * a3[2];
  const double c2 = a2[0] * a3[1] - a3[0] * a2[1];
  const double det = c0 + c1 + c2;
  if (!(fabs(det) > 0.0) || !isfinite(det)) return;
  const double inv = 1.0 / det;
  const double w0 = c0 * inv, w1 = c1 * inv, w2 = c2 * inv;
  if (!isfinite(w0) || !isfinite(w1) || !isfinite(w2)) return;
  w[0] = w0; w[1] = w1; w[2] = w2;
}

// Per-k smoothing factors (eqs. (14)-(16)) at t = r/delta:
//   s1 = erf t, s2 = s1 - G t, s3 = s2 - G (2/3) t^3, G = (2/sqrt(pi)) e^{-t^2}.
// Returned as s1, s2, s3 and c23 = s2 - s3 = G (2/3) t^3 (exact, no cancellation).
__device__ __forceinline__ void s_factors(double t, double& s1, double& s2, double& s3, double& c23) {
  const double E = erf(t);
  const double G = kTwoOverSqrtPi * exp(-t * t);
  const double gt = G * t;
  s1 = E;
  s2 = E - gt;
  c23 = gt * (2.0 / 3.0) * t * t;
  s3 = s2 - c23;
}

// e^{-u} for u >= 0: Cody-Waite reduction u = n ln2 + r, |r| <= ln2/2, degree-11
// polynomial (tools/gen_sfactor_coeffs.py), scale 2^n by building the exponent
// bits.  No special-case branches.  For u > ~708 the exponent field would
// underflow: n is clamped at -1022 (an integer max, off the FP64 pipe), which
// returns a value below 2e-308 -- 0 to every sum it enters -- instead of e^{-u}.
// (t = r/delta_k reaches 6 rho_3/rho_1 on a near pair: u > 708 once rho_3/rho_1 > 4.4.)
__device__ __forceinline__ double exp_neg(double u) {
  const double x = -u;
  const double kd = fma(x, 1.4426950408889634074, 6755399441055744.0);  // round(x/ln2) + 1.5*2^52
  const int n = max(__double2loint(kd), -1022);
  const double nd = kd - 6755399441055744.0;
  double r = fma(nd, -6.93147180559945286227e-01, x);
  r = fma(nd, -2.31904681384629955842e-17, r);
  double p = kExpPoly[kExpDeg];
#pragma unroll
  for (int j = kExpDeg - 1; j >= 0; --j) p = fma(p, r, kExpPoly[j]);
  return p * __hiloint2double((n + 1023) << 20, 0);
}

// 1/x for finite x > 0: MUFU.RCP64H seed + one third-order Newton step
// y(1 + e + e^2), e = 1 - x y (3 FP64 instructions, no special cases).
__device__ __forceinline__ double rcp_nr(double x) {
  double y;
  asm("rcp.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y, 1.0);
  return fma(y, fma(e, e, e), y);
}

// The two ingredients of the smoothing factors at t = r/delta for t >= 0.5:
//   e = e^{-t^2} and P = erfcx(t) as ONE degree-12 polynomial in v = 1/(2.5 + t)
//   (tools/gen_sfactor_coeffs.py; |error of 1 - e P| <= 2.2e-16 for every t >= 0.5: fitted on
//   [0.5, 6], and past 6 the polynomial still follows erfcx while e < 2.3e-16 -- checked to t = 40),
//   so erf t = 1 - e P with no table, no piece selection and no clamp; u = t^2 is returned too.
// Branch-free; for t < 0.5 it returns finite values the caller discards.
__device__ __forceinline__ void sfactor_eP(double t, double& e, double& P, double& u) {
  u = t * t;
  e = exp_neg(u);  // any u >= 0 (exp_neg clamps its exponent)
  const double x = fma(rcp_nr(kErfcxKappa + t), kErfcxVA, kErfcxVB);
  double p = kErfcxV[kErfcxDeg];
#pragma unroll
  for (int j = kErfcxDeg - 1; j >= 0; --j) p = fma(p, x, kErfcxV[j]);
  P = p;
}

// Smoothing factors (eqs. (14)-(16)) at t >= 0.5 from sfactor_eP:
//   E = erf t = 1 - e P,  s2 = E - (2/sqrt pi) t e,  c23 = s2 - s3 = (2/sqrt pi)(2/3) t^3 e.
__device__ __forceinline__ void sfactor_s(double t, double& E, double& s2, double& c23, double* e_out = nullptr) {
  double e, p, u;
  sfactor_eP(t, e, p, u);
  if (e_out) *e_out = e;  // e^{-t^2}, for callers that need it too (the s# factors)
  E = fma(-e, p, 1.0);
  const double gt = (kTwoOverSqrtPi * e) * t;
  s2 = E - gt;
  c23 = gt * (2.0 / 3.0) * u;
}

// t < 0.5: s1/t, s2/t^3, s3/t^5 and (s2 - s3)/t^3 from their series in u = t^2
// (cancellation-free, exact r -> 0 limits), scaled to A += w s_i/(t delta)^p.
__device__ __forceinline__ void sfactor_series_add(double t, double invd, double w, double& A1, double& A3,
                                                   double& A5, double& AP) {
  const double u = t * t;
  double f1 = kPhi1[kSeriesTerms - 1], f3 = kPhi3[kSeriesTerms - 1], f5 = kPhi5[kSeriesTerms - 1];
#pragma unroll
  for (int j = kSeriesTerms - 2; j >= 0; --j) {
    f1 = fma(f1, u, kPhi1[j]);
    f3 = fma(f3, u, kPhi3[j]);
    f5 = fma(f5, u, kPhi5[j]);
  }
  const double wi = w * invd, wi3 = wi * invd * invd, wi5 = wi3 * invd * invd;
  A1 = fma(wi, f1, A1);
  A3 = fma(wi3, f3, A3);
  A5 = fma(wi5, f5, A5);
  AP = fma(wi3, (2.0 / 3.0) * kTwoOverSqrtPi * exp_neg(u), AP);  // (4/(3 sqrt pi)) e^{-t^2}
}

// NEXT-1 on-surface factors at one delta, t = r/delta:
//   t >= 0.5: s1# = E + (2/(3 sqrt pi))(5t - 2t^3) e, s2# = E - (2/(3 sqrt pi))(3t - 14t^3 + 4t^5) e,
//             s3# = E - (2/(9 sqrt pi))(9t + 6t^3 - 4t^5) e   (E, e from the same exp + erfcx chain)
//   t <  0.5: s#/t, s#/t^3, s#/t^5 from their series (coefficients generated and self-checked).
// Returns A1 = s1#/r, A3 = s2#/r^3, A5 = s3#/r^5.
__device__ __forceinline__ void sharp_weights(double r, double ri, double invd,
                                              double& A1, double& A3, double& A5) {
  const double t = r * invd;
  if (t < 0.5) {
    const double u = t * t;
    double f1 = kPhi1S[kSeriesTerms - 1], f3 = kPhi3S[kSeriesTerms - 1], f5 = kPhi5S[kSeriesTerms - 1];
#pragma unroll
    for (int j = kSeriesTerms - 2; j >= 0; --j) {
      f1 = fma(f1, u, kPhi1S[j]);
      f3 = fma(f3, u, kPhi3S[j]);
      f5 = fma(f5, u, kPhi5S[j]);
    }
    const double i3 = invd * invd * invd;
    A1 = f1 * invd;
    A3 = f3 * i3;
    A5 = f5 * i3 * invd * invd;
    return;
  }
  double E, s2, c23, et;
  sfactor_s(t, E, s2, c23, &et);
  const double e = et * kInvSqrtPi;  // e^{-t^2}/sqrt(pi), shared with E's evaluation
  const double t2 = t * t, t3 = t2 * t, t5 = t3 * t2;
  const double s1s = fma((2.0 / 3.0) * e, fma(-2.0, t3, 5.0 * t), E);
  const double s2s = fma(-(2.0 / 3.0) * e, fma(4.0, t5, fma(-14.0, t3, 3.0 * t)), E);
  const double s3s = fma(-(2.0 / 9.0) * e, fma(-4.0, t5, fma(6.0, t3, 9.0 * t)), E);
  const double ri3 = ri * ri * ri;
  A1 = s1s * ri;
  A3 = s2s * ri3;
  A5 = s3s * ri3 * ri * ri;
}

}  // namespace ser
