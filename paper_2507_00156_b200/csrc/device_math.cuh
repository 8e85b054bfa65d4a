// device_math.cuh -- FP64 device helpers of the sm_100a hot path.
//
// Everything here is the CUDA side's own arithmetic; it
// shares nothing with oracle/.  Citations are PAPER.md lines.
#pragma once
#include <cstdint>

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

// On-surface factors s#_i of PAPER.md:130-138 (NEXT-1), same convention.
__device__ __forceinline__ void s_sharp_factors(double t, double& s1, double& s2, double& s3, double& c23) {
  const double E = erf(t);
  const double e = exp(-t * t) * kInvSqrtPi;
  const double t2 = t * t, t3 = t2 * t, t5 = t3 * t2;
  s1 = E + (2.0 / 3.0) * (5.0 * t - 2.0 * t3) * e;
  s2 = E - (2.0 / 3.0) * (3.0 * t - 14.0 * t3 + 4.0 * t5) * e;
  s3 = E - (2.0 / 9.0) * (9.0 * t + 6.0 * t3 - 4.0 * t5) * e;
  c23 = s2 - s3;
}

}  // namespace ser
