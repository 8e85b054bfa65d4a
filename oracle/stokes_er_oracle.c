/*
 * stokes_er_oracle.c -- the CPU ORACLE for the extrapolated-regularization
 * Stokes layer potentials of PAPER.md (arXiv 2507.00156).
 *
 * TEST INFRASTRUCTURE ONLY.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline / `--impl reference` leg may load or call this
 * library.  It shares no code, header, table or constant generator with the
 * CUDA path under paper_2507_00156_b200/ and never calls it.
 *
 * Plain, slow, obviously-correct FP64 C: libm erf/erfc/exp/sqrt, Neumaier
 * compensated sums, explicit rank-3 tensor loops for the stresslet split,
 * pivoted Gaussian elimination for the 3x3 extrapolation system.  OpenMP
 * splits the target loop only.
 *
 * What is computed, per target y with signed distance b, closest point
 * x0 = y - b n0, and per delta_k = rho_k h:
 *
 *   u^dk_i = 1/(8pi) sum_s S^dk_ia(y,x_s) [f_a(x_s) - (f(x0).n0) n_a(x_s)] w_s        eq. (10)
 *   v^dk_i = 1/(8pi) sum_s T^dk_iac(y,x_s) [q_a(x_s) - q_a(x0)] n_c(x_s) w_s + chi q_i(x0)  eq. (11)
 *
 *   S^d_ia = delta_ia s1(r/d)/r + yh_i yh_a s2(r/d)/r^3                         eq. (12)
 *   T^d    = T1 s2(r/d) + T2 s3(r/d),  T1 = -6 t1/r^3,                          eq. (13)
 *            T2 = -6 (t2 - (r^2 - b^2) t1)/r^5                                  eq. (7)
 *   t1_iac = b n_i n_a n_c - (xh_i n_a n_c + n_i xh_a n_c + n_i n_a xh_c)      eq. (8)
 *   t2_iac = b (xh_i xh_a n_c + xh_i n_a xh_c + n_i xh_a xh_c) - xh_i xh_a xh_c eq. (9)
 *            (n = n0, xh = x_s - x0)
 *   s1 = erf t, s2 = erf t - (2/sqrt pi) t e^{-t^2},
 *   s3 = erf t - (2/sqrt pi)(t + 2/3 t^3) e^{-t^2}                              eqs. (14)-(16) PAPER.md:90-102
 *   chi = 1 inside (b<0), 0 outside (b>0), 1/2 on the surface (b=0)
 *
 * then, per target, the 3x3 system of eq. (17)
 *   u + c1 rho_k I0(lambda_k) + c2 rho_k^3 I2(lambda_k) = u^dk,  lambda_k = b/delta_k
 * with I0, I2 of eqs. (18)-(19), solved for u; the same
 * system serves the stresslet.
 *
 * Two summation modes:
 *   definition (localized = 0): every pair uses the regularized kernels for
 *     every delta_k -- the definition the method reaches up to rounding.
 *   localized  (localized = 1): the paper's algorithm:
 *     pairs with r > c*delta_max (c = 6) contribute the
 *     unregularized S (eq. 3) and T (eq. 4)
 *     once to a far sum shared by all three delta_k (eq. 26 `near_far`).
 *
 * Readings where the paper is silent:
 *   R3  r = 0 (a node coinciding with the target): the r -> 0 limits
 *       s1/r -> 2/(sqrt(pi) d), s2/r^3 -> 4/(3 sqrt(pi) d^3),
 *       s3/r^5 -> 8/(15 sqrt(pi) d^5), used when r < 1e-8 * delta_1.
 *   R7  singular extrapolation matrix (I0 = I2 = 0 after underflow): return u^d1.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#ifdef _OPENMP
#include <omp.h>
#endif

#define ORACLE_PI 3.14159265358979323846
#define ORACLE_SQRT_PI 1.77245385090551602730
#define ORACLE_CUTOFF 6.0 /* PAPER.md:175 "s1 = s2 = s3 = 1 for t = r/delta > 6" */

/* ---- compensated (Neumaier) accumulator ---------------------------------- */
typedef struct { double s, c; } nsum;
static void nadd(nsum* a, double x) {
  double t = a->s + x;
  if (fabs(a->s) >= fabs(x)) a->c += (a->s - t) + x;
  else a->c += (x - t) + a->s;
  a->s = t;
}
static double nval(const nsum* a) { return a->s + a->c; }

/* ---- smoothing factors, eqs. (14)-(16), PAPER.md:90-102 ------------------- */
void oracle_s_factors(double t, double s[3]) {
  double E = erf(t);
  double G = 2.0 / ORACLE_SQRT_PI * exp(-t * t);
  s[0] = E;
  s[1] = E - G * t;
  s[2] = E - G * (t + 2.0 / 3.0 * t * t * t);
}

/* ---- on-surface factors s#, PAPER.md:130-138 (Sec. 2.1) ------------------- */
void oracle_s_sharp_factors(double t, double s[3]) {
  double E = erf(t);
  double e = exp(-t * t);
  double t3 = t * t * t, t5 = t3 * t * t;
  s[0] = E + 2.0 / (3.0 * ORACLE_SQRT_PI) * (5.0 * t - 2.0 * t3) * e;
  s[1] = E - 2.0 / (3.0 * ORACLE_SQRT_PI) * (3.0 * t - 14.0 * t3 + 4.0 * t5) * e;
  s[2] = E - 2.0 / (9.0 * ORACLE_SQRT_PI) * (9.0 * t + 6.0 * t3 - 4.0 * t5) * e;
}

/* ---- I0, I2: eqs. (18)-(19), PAPER.md:114-121 ----------------------------- */
double oracle_I0(double lam) {
  double a = fabs(lam);
  return exp(-lam * lam) / ORACLE_SQRT_PI - a * erfc(a);
}
double oracle_I2(double lam) {
  double a = fabs(lam);
  return 2.0 / 3.0 * ((0.5 - lam * lam) * exp(-lam * lam) / ORACLE_SQRT_PI + a * a * a * erfc(a));
}

/* ---- kernel weights A1 = s1/r, A3 = s2/r^3, A5 = s3/r^5 for one delta ------ */
static void reg_weights(double r, double delta, double delta1, int sharp, double A[3]) {
  if (r < 1e-8 * delta1) { /* reading R3: exact r -> 0 limits */
    if (!sharp) {
      A[0] = 2.0 / (ORACLE_SQRT_PI * delta);
      A[1] = 4.0 / (3.0 * ORACLE_SQRT_PI * delta * delta * delta);
      A[2] = 8.0 / (15.0 * ORACLE_SQRT_PI * pow(delta, 5));
    } else {
      /* limits of s#_i(t)/t^p from the series erf t = k(t - t^3/3 + t^5/10 - ...),
       * e^{-t^2} = 1 - t^2 + t^4/2 - ..., k = 2/sqrt(pi):
       *  s1#: t^1 coefficient  k + (2/(3 sqrt pi)) 5
       *  s2#: t^1: k - (2/(3 sqrt pi)) 3 = 0;  t^3: -k/3 + (2/(3 sqrt pi)) 17
       *  s3#: t^1, t^3 vanish;  t^5: k/10 + (2/(9 sqrt pi)) 11/2              */
      const double k = 2.0 / ORACLE_SQRT_PI;
      A[0] = (k + 10.0 / (3.0 * ORACLE_SQRT_PI)) / delta;
      A[1] = (-k / 3.0 + 34.0 / (3.0 * ORACLE_SQRT_PI)) / (delta * delta * delta);
      A[2] = (k / 10.0 + 11.0 / (9.0 * ORACLE_SQRT_PI)) / pow(delta, 5);
    }
    return;
  }
  double t = r / delta, s[3];
  if (sharp) oracle_s_sharp_factors(t, s);
  else oracle_s_factors(t, s);
  A[0] = s[0] / r;
  A[1] = s[1] / (r * r * r);
  A[2] = s[2] / (r * r * r * r * r);
}

/* ---- one target, sources s0 <= s < s1 (arrays of stride N): accumulate the
 * pair terms into the per-delta sums Us, Vs (near, or every pair in definition
 * mode) and the shared far sums Uf, Vf (localized mode, r^2 > rc2). -------- */
static void accum_pairs(const double* src_xyz, const double* src_normal, const double* src_weight,
                        const double* f, const double* q, int64_t N, int64_t s0, int64_t s1,
                        const double y[3], double b, const double n0[3], const double x0[3], double alpha,
                        const double q0[3], const double delta[3], int ndelta, int mode, int localized,
                        int sharp, double rc2, nsum Us[3][3], nsum Vs[3][3], nsum Uf[3], nsum Vf[3]) {
  for (int64_t s = s0; s < s1; ++s) {
    double x[3], m[3], yh[3], xh[3], g[3], dq[3];
    for (int i = 0; i < 3; ++i) {
      x[i] = src_xyz[i * N + s];
      m[i] = src_normal[i * N + s];
      yh[i] = y[i] - x[i];                                         /* y - x */
      xh[i] = x[i] - x0[i];                                        /* x - x0 */
    }
    const double w = src_weight[s];
    const double r2 = yh[0] * yh[0] + yh[1] * yh[1] + yh[2] * yh[2];
    const double r = sqrt(r2);
    if (mode & 1)
      for (int a = 0; a < 3; ++a) g[a] = f[a * N + s] - alpha * m[a];
    if (mode & 2)
      for (int a = 0; a < 3; ++a) dq[a] = q[a * N + s] - q0[a];

    if (localized && r2 > rc2) {
      /* far pair: unregularized Stokeslet (eq. 3) and stresslet (eq. 4), shared by all delta */
      const double r3 = r2 * r, r5 = r3 * r2;
      if (mode & 1)
        for (int i = 0; i < 3; ++i)
          for (int a = 0; a < 3; ++a) {
            double S = (i == a ? 1.0 / r : 0.0) + yh[i] * yh[a] / r3;
            nadd(&Uf[i], S * g[a] * w);
          }
      if (mode & 2)
        for (int i = 0; i < 3; ++i)
          for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) {
              double T = -6.0 * yh[i] * yh[a] * yh[c] / r5;
              nadd(&Vf[i], T * dq[a] * m[c] * w);
            }
      continue;
    }

    /* t1, t2 of eqs. (8)-(9): explicit rank-3 tensors */
    double t1[3][3][3], t2[3][3][3];
    if (mode & 2)
      for (int i = 0; i < 3; ++i)
        for (int a = 0; a < 3; ++a)
          for (int c = 0; c < 3; ++c) {
            t1[i][a][c] = b * n0[i] * n0[a] * n0[c] -
                          (xh[i] * n0[a] * n0[c] + n0[i] * xh[a] * n0[c] + n0[i] * n0[a] * xh[c]);
            t2[i][a][c] = b * (xh[i] * xh[a] * n0[c] + xh[i] * n0[a] * xh[c] + n0[i] * xh[a] * xh[c]) -
                          xh[i] * xh[a] * xh[c];
          }
    for (int k = 0; k < ndelta; ++k) {
      double A[3];
      reg_weights(r, delta[k], delta[0], sharp, A);
      if (mode & 1)
        for (int i = 0; i < 3; ++i)
          for (int a = 0; a < 3; ++a) {
            double S = (i == a ? A[0] : 0.0) + yh[i] * yh[a] * A[1];  /* eq. (12) */
            nadd(&Us[k][i], S * g[a] * w);
          }
      if ((mode & 2) && !sharp)
        for (int i = 0; i < 3; ++i)
          for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) {
              /* T^d = T1 s2 + T2 s3 (eq. 13) with T1, T2 of eq. (7) */
              double T = -6.0 * (t1[i][a][c] * A[1] + (t2[i][a][c] - (r2 - b * b) * t1[i][a][c]) * A[2]);
              nadd(&Vs[k][i], T * dq[a] * m[c] * w);
            }
      if ((mode & 2) && sharp)
        for (int i = 0; i < 3; ++i)
          for (int a = 0; a < 3; ++a)
            for (int c = 0; c < 3; ++c) {
              /* reading R16: on the surface the stresslet is regularized unsplit,
               * T# = T s3#(r/d) = -6 yh_i yh_a yh_c s3#/r^5 (eq. 4 times s3#) */
              double T = -6.0 * yh[i] * yh[a] * yh[c] * A[2];
              nadd(&Vs[k][i], T * dq[a] * m[c] * w);
            }
    }
  }
}

/* per-delta totals: (near + far)/(8 pi), + chi q(x0) for the DL (eqs. (10)-(11)) */
static void finish_target(double b, const double q0[3], int ndelta, nsum Us[3][3], nsum Vs[3][3],
                          nsum Uf[3], nsum Vf[3], double U[3][3], double V[3][3]) {
  const double chi = b < 0.0 ? 1.0 : (b > 0.0 ? 0.0 : 0.5);
  for (int k = 0; k < ndelta; ++k)
    for (int i = 0; i < 3; ++i) {
      nsum u = Us[k][i], v = Vs[k][i];
      nadd(&u, nval(&Uf[i]));
      nadd(&v, nval(&Vf[i]));
      U[k][i] = nval(&u) / (8.0 * ORACLE_PI);
      V[k][i] = nval(&v) / (8.0 * ORACLE_PI) + chi * q0[i];
    }
}

/* ---- one target: the three regularized sums ------------------------------- */
static void eval_target(const double* src_xyz, const double* src_normal, const double* src_weight,
                        const double* f, const double* q, const double y[3], double b,
                        const double n0[3], const double f0[3], const double q0[3], int64_t N,
                        const double delta[3], int ndelta, int mode, int localized, int sharp,
                        double cutoff, double U[3][3], double V[3][3]) {
  nsum Us[3][3], Vs[3][3], Uf[3], Vf[3];
  memset(Us, 0, sizeof(Us)); memset(Vs, 0, sizeof(Vs));
  memset(Uf, 0, sizeof(Uf)); memset(Vf, 0, sizeof(Vf));
  double x0[3], alpha = 0.0;
  for (int i = 0; i < 3; ++i) x0[i] = y[i] - b * n0[i];           /* y = x0 + b n0 */
  for (int i = 0; i < 3; ++i) alpha += f0[i] * n0[i];             /* f(x0).n(x0) */
  double dmax = delta[0];
  for (int k = 1; k < ndelta; ++k) dmax = fmax(dmax, delta[k]);
  const double rc2 = (cutoff * dmax) * (cutoff * dmax);
  accum_pairs(src_xyz, src_normal, src_weight, f, q, N, 0, N, y, b, n0, x0, alpha, q0, delta, ndelta, mode,
              localized, sharp, rc2, Us, Vs, Uf, Vf);
  finish_target(b, q0, ndelta, Us, Vs, Uf, Vf, U, V);
}

static int check_args(const double* src_xyz, const double* src_normal, const double* src_weight,
                      const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                      const double* tgt_x0_density, int64_t M, int64_t N, double h, int mode) {
  if (M < 0 || N < 1 || !(h > 0.0) || !isfinite(h)) return 1;
  if (mode < 1 || mode > 3) return 1;
  if (!src_xyz || !src_normal || !src_weight || !tgt_xyz || !tgt_b || !tgt_x0_density) return 1;
  if ((mode & 1) && !f) return 1;
  if ((mode & 2) && !q) return 1;
  return 0;
}

/* Per-delta values u^dk, v^dk.  out_udelta / out_vdelta: [3][3][M] = [k][i][m]
 * (NULL allowed when the mode does not produce it).  Returns 0 or 1 (EINVAL). */
int oracle_eval_deltas(const double* src_xyz, const double* src_normal, const double* src_weight,
                       const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                       const double* tgt_x0_density, int64_t M, int64_t N, double h,
                       const double rho[3], int mode, int localized, int nthreads,
                       double* out_udelta, double* out_vdelta) {
  if (check_args(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, mode))
    return 1;
  if (!(rho[0] > 0.0 && rho[1] > rho[0] && rho[2] > rho[1])) return 1;
  double delta[3] = {rho[0] * h, rho[1] * h, rho[2] * h};
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < M; ++t) {
    double y[3], n0[3], f0[3], q0[3], U[3][3], V[3][3];
    for (int i = 0; i < 3; ++i) {
      y[i] = tgt_xyz[i * M + t];
      n0[i] = tgt_x0_density[i * M + t];
      f0[i] = tgt_x0_density[(3 + i) * M + t];
      q0[i] = tgt_x0_density[(6 + i) * M + t];
    }
    eval_target(src_xyz, src_normal, src_weight, f, q, y, tgt_b[t], n0, f0, q0, N, delta, 3, mode,
                localized, 0, ORACLE_CUTOFF, U, V);
    for (int k = 0; k < 3; ++k)
      for (int i = 0; i < 3; ++i) {
        if (out_udelta && (mode & 1)) out_udelta[(k * 3 + i) * M + t] = U[k][i];
        if (out_vdelta && (mode & 2)) out_vdelta[(k * 3 + i) * M + t] = V[k][i];
      }
  }
  return 0;
}

/* Solve the 3x3 system of eq. (17) for every target and C right-hand sides.
 * in_delta: [3][C][M] (k, component, target); out: [C][M].
 * Gaussian elimination with partial pivoting (reading R6). */
int oracle_extrapolate(const double* tgt_b, int64_t M, double h, const double rho[3],
                       const double* in_delta, int C, double* out) {
  if (M < 0 || !(h > 0.0) || C < 1 || C > 64 || !tgt_b || !in_delta || !out) return 1;
  if (!(rho[0] > 0.0 && rho[1] > rho[0] && rho[2] > rho[1])) return 1;
#pragma omp parallel for schedule(static)
  for (int64_t t = 0; t < M; ++t) {
    double A[3][3], B[3][64];
    const double b = tgt_b[t];
    for (int k = 0; k < 3; ++k) {
      const double lam = b / (rho[k] * h);                       /* lambda = b/delta */
      A[k][0] = 1.0;
      A[k][1] = rho[k] * oracle_I0(lam);
      A[k][2] = rho[k] * rho[k] * rho[k] * oracle_I2(lam);
      for (int c = 0; c < C; ++c) B[k][c] = in_delta[((int64_t)k * C + c) * M + t];
    }
    int singular = 0;
    for (int col = 0; col < 3 && !singular; ++col) {
      int p = col;
      for (int r = col + 1; r < 3; ++r)
        if (fabs(A[r][col]) > fabs(A[p][col])) p = r;
      if (A[p][col] == 0.0) { singular = 1; break; }
      if (p != col) {
        for (int j = 0; j < 3; ++j) { double tmp = A[p][j]; A[p][j] = A[col][j]; A[col][j] = tmp; }
        for (int c = 0; c < C; ++c) { double tmp = B[p][c]; B[p][c] = B[col][c]; B[col][c] = tmp; }
      }
      for (int r = col + 1; r < 3; ++r) {
        const double l = A[r][col] / A[col][col];
        for (int j = col; j < 3; ++j) A[r][j] -= l * A[col][j];
        for (int c = 0; c < C; ++c) B[r][c] -= l * B[col][c];
      }
    }
    for (int c = 0; c < C; ++c) {
      double x2 = 0, x1 = 0, x0 = 0;
      if (!singular) {
        x2 = B[2][c] / A[2][2];
        x1 = (B[1][c] - A[1][2] * x2) / A[1][1];
        x0 = (B[0][c] - A[0][1] * x1 - A[0][2] * x2) / A[0][0];
      }
      if (singular || !isfinite(x0)) x0 = in_delta[(int64_t)c * M + t]; /* reading R7: u^d1 */
      out[(int64_t)c * M + t] = x0;
    }
  }
  return 0;
}

/* Full evaluation: per-delta sums, then extrapolation.  out_u, out_v: [3][M]. */
int oracle_eval(const double* src_xyz, const double* src_normal, const double* src_weight,
                const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho[3],
                int mode, int localized, int nthreads, double* out_u, double* out_v) {
  if (M == 0) return check_args(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density,
                                M, N, h, mode);
  double* ud = (mode & 1) ? (double*)malloc(sizeof(double) * 9 * (size_t)M) : NULL;
  double* vd = (mode & 2) ? (double*)malloc(sizeof(double) * 9 * (size_t)M) : NULL;
  int rc = oracle_eval_deltas(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M,
                              N, h, rho, mode, localized, nthreads, ud, vd);
  if (!rc && (mode & 1)) rc = oracle_extrapolate(tgt_b, M, h, rho, ud, 3, out_u);
  if (!rc && (mode & 2)) rc = oracle_extrapolate(tgt_b, M, h, rho, vd, 3, out_v);
  free(ud);
  free(vd);
  return rc;
}

/* NEXT-1 (Sec. 2.1; used at delta = 3h for self
 * surfaces): a single delta with the s# factors, no
 * extrapolation.  Cutoff c# passed in (reading R15: c = 7 for s#).
 * out_u, out_v: [3][M]. */
int oracle_eval_sharp(const double* src_xyz, const double* src_normal, const double* src_weight,
                      const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                      const double* tgt_x0_density, int64_t M, int64_t N, double delta, int mode,
                      int localized, double cutoff, int nthreads, double* out_u, double* out_v) {
  if (check_args(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, delta, mode))
    return 1;
  double dl[3] = {delta, delta, delta};
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4)
  for (int64_t t = 0; t < M; ++t) {
    double y[3], n0[3], f0[3], q0[3], U[3][3], V[3][3];
    for (int i = 0; i < 3; ++i) {
      y[i] = tgt_xyz[i * M + t];
      n0[i] = tgt_x0_density[i * M + t];
      f0[i] = tgt_x0_density[(3 + i) * M + t];
      q0[i] = tgt_x0_density[(6 + i) * M + t];
    }
    eval_target(src_xyz, src_normal, src_weight, f, q, y, tgt_b[t], n0, f0, q0, N, dl, 1, mode,
                localized, 1, cutoff, U, V);
    for (int i = 0; i < 3; ++i) {
      if (out_u && (mode & 1)) out_u[i * M + t] = U[0][i];
      if (out_v && (mode & 2)) out_v[i * M + t] = V[0][i];
    }
  }
  return 0;
}

int oracle_max_threads(void) {
#ifdef _OPENMP
  return omp_get_max_threads();
#else
  return 1;
#endif
}

/* ===================================================================== NEXT-3
 * The kernel-independent treecode of PAPER.md Sec. 3.4 (lines 194-233) for the
 * far part of the localized sums, step by step in the paper's order:
 *   1. the quadrature points are partitioned into an octree until at most N0
 *      points remain in a cluster (a leaf)
 *   2. modified weights (eq. (32) `mod_weights`) at the tensor Chebyshev points
 *      s_k of each cluster box, for f w and n w (SL) and q n w and n w (DL)
 *                                                               PAPER.md:215-230
 *   3. per target, from the root: if the MAC r_c/R <= theta (eq. (28)) holds the
 *      cluster's interaction is eq. (31) with the unregularized S, T at the s_k;
 *      otherwise the children are checked; a leaf that fails is summed directly
 *      with the localized regularization (3 deltas near, shared far) PAPER.md:232
 * Readings (R22-R25):
 *   R22 tree: root box = tight box of the points; a cluster with > N0 points and
 *       a box of non-zero extent is split at its box midpoint in every axis of
 *       non-zero extent (x_d >= mid_d goes up), points keep their order within
 *       an octant, empty octants are dropped, children in octant order
 *       (bit d = upper half in axis d); every box then shrinks to its points'
 *       tight box.  r_c = half the box diagonal, centre = box midpoint.
 *   R23 acceptance = MAC AND the box lies beyond the regularization cutoff
 *       (gap^2 > (c delta_max)^2), so no pair with r <= c delta_max is ever
 *       approximated; both tests in plain (non-fused) FP64 in a fixed order:
 *       R^2 = (dx*dx + dy*dy) + dz*dz, accept iff r_c <= theta*sqrt(R^2).
 *   R24 Chebyshev points of the second kind s_k = c + (w/2) cos(k pi/p), k = 0..p,
 *       barycentric weights (-1)^k, halved at k = 0 and p; a coordinate within
 *       1e-14 w of a node takes that node's cardinal value; an axis of zero
 *       extent interpolates with L_0 = 1.
 *   R25 far part of a target = sum over accepted clusters of eq. (31) with the
 *       subtraction structure: SL weights g^fw - alpha g^nw, DL weights
 *       g^qn_ac - q0_a g^nw_c.
 *   R26 an accepted cluster with at most (p+1)^3 points is summed directly
 *       (its far pairs exactly) instead of through its (p+1)^3 Chebyshev points,
 *       which would cost more and be less accurate; the paper is silent. */
typedef struct {
  double lo[3], hi[3], c[3], rc;
  int64_t begin, end;  /* tree-order range */
  int first_child, nchild;
} tnode;

static void tight_box(const double* xyz, int64_t N, const int64_t* idx, int64_t b, int64_t e, double lo[3],
                      double hi[3]) {
  for (int d = 0; d < 3; ++d) { lo[d] = INFINITY; hi[d] = -INFINITY; }
  for (int64_t j = b; j < e; ++j)
    for (int d = 0; d < 3; ++d) {
      const double v = xyz[d * N + idx[j]];
      if (v < lo[d]) lo[d] = v;
      if (v > hi[d]) hi[d] = v;
    }
}

static void set_geometry(tnode* t) {
  double s = 0.0;
  for (int d = 0; d < 3; ++d) {
    const double w = t->hi[d] - t->lo[d];
    t->c[d] = 0.5 * (t->lo[d] + t->hi[d]);
    s = s + w * w;
  }
  t->rc = 0.5 * sqrt(s);
}

/* recursive build (R22); returns the node count or -1 if max_nodes is exceeded */
static int build_node(const double* xyz, int64_t N, int64_t* idx, int64_t* tmp, tnode* nodes, int self,
                      int* count, int max_nodes, int64_t N0) {
  tnode* t = &nodes[self];
  t->first_child = -1;
  t->nchild = 0;
  const int64_t n = t->end - t->begin;
  int split_axes = 0;
  for (int d = 0; d < 3; ++d)
    if (t->hi[d] > t->lo[d]) split_axes |= 1 << d;
  if (n <= N0 || !split_axes) return 0;
  double mid[3];
  for (int d = 0; d < 3; ++d) mid[d] = 0.5 * (t->lo[d] + t->hi[d]);
  int64_t cnt[8] = {0}, start[8];
  for (int64_t j = t->begin; j < t->end; ++j) {
    int o = 0;
    for (int d = 0; d < 3; ++d)
      if ((split_axes >> d & 1) && xyz[d * N + idx[j]] >= mid[d]) o |= 1 << d;
    cnt[o]++;
  }
  start[0] = t->begin;
  for (int o = 1; o < 8; ++o) start[o] = start[o - 1] + cnt[o - 1];
  int64_t pos[8];
  memcpy(pos, start, sizeof(pos));
  for (int64_t j = t->begin; j < t->end; ++j) {
    int o = 0;
    for (int d = 0; d < 3; ++d)
      if ((split_axes >> d & 1) && xyz[d * N + idx[j]] >= mid[d]) o |= 1 << d;
    tmp[pos[o]++] = idx[j];
  }
  memcpy(idx + t->begin, tmp + t->begin, sizeof(int64_t) * (size_t)n);
  int nc = 0;
  for (int o = 0; o < 8; ++o) nc += cnt[o] > 0;
  if (*count + nc > max_nodes) return -1;
  const int first = *count;
  *count += nc;
  t->first_child = first;
  t->nchild = nc;
  int k = first;
  for (int o = 0; o < 8; ++o) {
    if (!cnt[o]) continue;
    tnode* ch = &nodes[k];
    ch->begin = start[o];
    ch->end = start[o] + cnt[o];
    tight_box(xyz, N, idx, ch->begin, ch->end, ch->lo, ch->hi);
    set_geometry(ch);
    ++k;
  }
  for (int j = first; j < first + nc; ++j)
    if (build_node(xyz, N, idx, tmp, nodes, j, count, max_nodes, N0) < 0) return -1;
  return 0;
}

/* 1-D barycentric Lagrange basis at x on the second-kind Chebyshev points of [lo, hi] (R24) */
static void lagrange_1d(double x, double lo, double hi, int p, double L[]) {
  const double w = hi - lo;
  for (int k = 0; k <= p; ++k) L[k] = 0.0;
  if (!(w > 0.0)) { L[0] = 1.0; return; }
  const double c = 0.5 * (lo + hi), half = 0.5 * w;
  double s[64], bw[64];
  for (int k = 0; k <= p; ++k) {
    s[k] = c + half * cos(k * ORACLE_PI / p);
    bw[k] = ((k & 1) ? -1.0 : 1.0) * ((k == 0 || k == p) ? 0.5 : 1.0);
    if (fabs(x - s[k]) <= 1e-14 * w) { for (int j = 0; j <= p; ++j) L[j] = 0.0; L[k] = 1.0; return; }
  }
  double den = 0.0;
  for (int k = 0; k <= p; ++k) den += bw[k] / (x - s[k]);
  for (int k = 0; k <= p; ++k) L[k] = (bw[k] / (x - s[k])) / den;
}

#define TC_CH 15 /* channels: fw (3), nw (3), q_a n_c w (9) */

typedef struct {
  int p, nnodes;
  tnode* nodes;
  int64_t* perm;      /* tree order -> input index */
  double* mw;         /* [node][(p+1)^3][TC_CH] modified weights */
} tree_t;

/* Evaluate targets with the treecode.  Inputs as oracle_eval, plus leaf size N0,
 * degree p and MAC theta.  out_u, out_v: [3][M].  out_stats (may be NULL):
 * [0] nodes, [1] accepted (target, cluster) pairs, [2] directly summed
 * (target, source) pairs.  Returns 0, 1 (EINVAL) or 2 (tree too large). */
/* sharp = 1: NEXT-1's on-surface single-delta s# evaluation (delta = h, rho
 * ignored, cutoff 7 (R15), no extrapolation) with the same treecode far part. */
static int eval_tree_impl(const double* src_xyz, const double* src_normal, const double* src_weight,
                          const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                          const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho_in[3],
                          int mode, int64_t N0, int p, double theta, int nthreads, int sharp, double* out_u,
                          double* out_v, double* out_stats) {
  const double one[3] = {1.0, 1.0, 1.0};
  const double* rho = sharp ? one : rho_in;
  if (check_args(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, mode)) return 1;
  if ((!sharp && !(rho[0] > 0.0 && rho[1] > rho[0] && rho[2] > rho[1])) || N0 < 1 || p < 1 || p > 40 ||
      !(theta >= 0.0))
    return 1;
  /* 1. tree (R22) */
  const int max_nodes = (int)(8 * (N / N0) + 4096);
  tree_t T;
  T.p = p;
  T.nodes = (tnode*)calloc((size_t)max_nodes, sizeof(tnode));
  T.perm = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  int64_t* tmp = (int64_t*)malloc(sizeof(int64_t) * (size_t)N);
  for (int64_t j = 0; j < N; ++j) T.perm[j] = j;
  T.nodes[0].begin = 0;
  T.nodes[0].end = N;
  tight_box(src_xyz, N, T.perm, 0, N, T.nodes[0].lo, T.nodes[0].hi);
  set_geometry(&T.nodes[0]);
  int count = 1;
  if (build_node(src_xyz, N, T.perm, tmp, T.nodes, 0, &count, max_nodes, N0) < 0) {
    free(T.nodes); free(T.perm); free(tmp);
    return 2;
  }
  free(tmp);
  T.nnodes = count;
  /* sources in tree order */
  double *X = (double*)malloc(sizeof(double) * 3 * (size_t)N), *Nr = (double*)malloc(sizeof(double) * 3 * (size_t)N);
  double *W = (double*)malloc(sizeof(double) * (size_t)N);
  double *F = (double*)calloc(3 * (size_t)N, sizeof(double)), *Q = (double*)calloc(3 * (size_t)N, sizeof(double));
  for (int64_t j = 0; j < N; ++j) {
    const int64_t s = T.perm[j];
    W[j] = src_weight[s];
    for (int d = 0; d < 3; ++d) {
      X[d * N + j] = src_xyz[d * N + s];
      Nr[d * N + j] = src_normal[d * N + s];
      if (mode & 1) F[d * N + j] = f[d * N + s];
      if (mode & 2) Q[d * N + j] = q[d * N + s];
    }
  }
  /* 2. modified weights, eq. (32): g^_k = sum_j L_k1(x_j1) L_k2(x_j2) L_k3(x_j3) g(x_j) */
  const int P1 = p + 1, NP = P1 * P1 * P1;
  T.mw = (double*)calloc((size_t)T.nnodes * NP * TC_CH, sizeof(double));
#pragma omp parallel for schedule(dynamic, 1)
  for (int c = 0; c < T.nnodes; ++c) {
    const tnode* t = &T.nodes[c];
    double* G = T.mw + (size_t)c * NP * TC_CH;
    for (int64_t j = t->begin; j < t->end; ++j) {
      double L[3][64], g[TC_CH];
      for (int d = 0; d < 3; ++d) lagrange_1d(X[d * N + j], t->lo[d], t->hi[d], p, L[d]);
      for (int a = 0; a < 3; ++a) {
        g[a] = F[a * N + j] * W[j];                  /* f_a w   (SL) */
        g[3 + a] = Nr[a * N + j] * W[j];             /* n_a w   (SL, DL) */
        for (int cc = 0; cc < 3; ++cc) g[6 + 3 * a + cc] = Q[a * N + j] * Nr[cc * N + j] * W[j];  /* q_a n_c w */
      }
      for (int k1 = 0; k1 < P1; ++k1)
        for (int k2 = 0; k2 < P1; ++k2)
          for (int k3 = 0; k3 < P1; ++k3) {
            const double Lk = L[0][k1] * L[1][k2] * L[2][k3];
            double* Gk = G + ((size_t)(k1 * P1 + k2) * P1 + k3) * TC_CH;
            for (int ch = 0; ch < TC_CH; ++ch) Gk[ch] += Lk * g[ch];
          }
    }
  }
  /* 3. per target traversal */
  const double delta[3] = {rho[0] * h, rho[1] * h, rho[2] * h};
  const double cutoff = sharp ? 7.0 : ORACLE_CUTOFF;  /* R15 for s# */
  const double rc2 = (cutoff * delta[2]) * (cutoff * delta[2]);
  /* R23 guard margin: a cluster whose box gap is within rounding of the cutoff is
   * never approximated, so no pair the near rule (r^2 <= rc2) owns can be */
  const double rc2_guard = rc2 * (1.0 + 1e-9);
  const int nd = sharp ? 1 : 3;
  double* ud = (double*)malloc(sizeof(double) * 9 * (size_t)(M > 0 ? M : 1));
  double* vd = (double*)malloc(sizeof(double) * 9 * (size_t)(M > 0 ? M : 1));
  double n_acc = 0.0, n_dir = 0.0;
#ifdef _OPENMP
  if (nthreads > 0) omp_set_num_threads(nthreads);
#endif
#pragma omp parallel for schedule(dynamic, 4) reduction(+ : n_acc, n_dir)
  for (int64_t tg = 0; tg < M; ++tg) {
    double y[3], n0[3], f0[3], q0[3], x0[3], alpha = 0.0;
    for (int i = 0; i < 3; ++i) {
      y[i] = tgt_xyz[i * M + tg];
      n0[i] = tgt_x0_density[i * M + tg];
      f0[i] = tgt_x0_density[(3 + i) * M + tg];
      q0[i] = tgt_x0_density[(6 + i) * M + tg];
    }
    const double b = tgt_b[tg];
    for (int i = 0; i < 3; ++i) x0[i] = y[i] - b * n0[i];
    for (int i = 0; i < 3; ++i) alpha += f0[i] * n0[i];
    nsum Us[3][3], Vs[3][3], Uf[3], Vf[3];
    memset(Us, 0, sizeof(Us)); memset(Vs, 0, sizeof(Vs));
    memset(Uf, 0, sizeof(Uf)); memset(Vf, 0, sizeof(Vf));
    int stack[4096], sp = 0;
    stack[sp++] = 0;
    while (sp > 0) {
      const int c = stack[--sp];
      const tnode* t = &T.nodes[c];
      /* R23: MAC (eq. 28) and the regularization guard, plain FP64 */
      const double dx = y[0] - t->c[0], dy = y[1] - t->c[1], dz = y[2] - t->c[2];
      volatile double R2 = dx * dx;
      R2 = R2 + dy * dy;
      R2 = R2 + dz * dz;
      volatile double g2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        double gap = t->lo[d] - y[d];
        if (y[d] - t->hi[d] > gap) gap = y[d] - t->hi[d];
        if (gap < 0.0) gap = 0.0;
        g2 = g2 + gap * gap;
      }
      const int accept = (t->rc <= theta * sqrt(R2)) && (g2 > rc2_guard);
      if (accept && t->end - t->begin > NP) { /* eq. (31): unregularized kernels at the Chebyshev points */
        n_acc += 1.0;
        const double* G = T.mw + (size_t)c * NP * TC_CH;
        double cs[3][64];
        for (int d = 0; d < 3; ++d)
          for (int k = 0; k <= p; ++k)
            cs[d][k] = 0.5 * (t->lo[d] + t->hi[d]) + 0.5 * (t->hi[d] - t->lo[d]) * cos(k * ORACLE_PI / p);
        for (int k1 = 0; k1 < P1; ++k1)
          for (int k2 = 0; k2 < P1; ++k2)
            for (int k3 = 0; k3 < P1; ++k3) {
              const double* Gk = G + ((size_t)(k1 * P1 + k2) * P1 + k3) * TC_CH;
              double yh[3] = {y[0] - cs[0][k1], y[1] - cs[1][k2], y[2] - cs[2][k3]};
              const double r2 = yh[0] * yh[0] + yh[1] * yh[1] + yh[2] * yh[2];
              const double r = sqrt(r2), r3 = r2 * r, r5 = r3 * r2;
              if (mode & 1)
                for (int i = 0; i < 3; ++i)
                  for (int a = 0; a < 3; ++a) {
                    const double S = (i == a ? 1.0 / r : 0.0) + yh[i] * yh[a] / r3;   /* eq. (3) */
                    nadd(&Uf[i], S * (Gk[a] - alpha * Gk[3 + a]));                   /* R25 */
                  }
              if (mode & 2)
                for (int i = 0; i < 3; ++i)
                  for (int a = 0; a < 3; ++a)
                    for (int cc = 0; cc < 3; ++cc) {
                      const double Tt = -6.0 * yh[i] * yh[a] * yh[cc] / r5;             /* eq. (4) */
                      nadd(&Vf[i], Tt * (Gk[6 + 3 * a + cc] - q0[a] * Gk[3 + cc]));   /* R25 */
                    }
            }
      } else if (accept || t->nchild == 0) {
        /* a leaf that fails, or an accepted cluster with no more points than
         * Chebyshev points (R26): direct sum, localized regularization */
        n_dir += (double)(t->end - t->begin);
        accum_pairs(X, Nr, W, F, Q, N, t->begin, t->end, y, b, n0, x0, alpha, q0, delta, nd, mode, 1, sharp, rc2,
                    Us, Vs, Uf, Vf);
      } else {
        for (int k = t->nchild - 1; k >= 0; --k) stack[sp++] = t->first_child + k;  /* octant order */
      }
    }
    double U[3][3], V[3][3];
    finish_target(b, q0, nd, Us, Vs, Uf, Vf, U, V);
    for (int k = 0; k < nd; ++k)
      for (int i = 0; i < 3; ++i) {
        ud[(k * 3 + i) * M + tg] = U[k][i];
        vd[(k * 3 + i) * M + tg] = V[k][i];
      }
  }
  int rc = 0;
  if (sharp) { /* single delta: u^delta itself */
    for (int64_t tg = 0; tg < M; ++tg)
      for (int i = 0; i < 3; ++i) {
        if (out_u && (mode & 1)) out_u[i * M + tg] = ud[i * M + tg];
        if (out_v && (mode & 2)) out_v[i * M + tg] = vd[i * M + tg];
      }
  } else {
    if (M > 0 && (mode & 1)) rc = oracle_extrapolate(tgt_b, M, h, rho, ud, 3, out_u);
    if (!rc && M > 0 && (mode & 2)) rc = oracle_extrapolate(tgt_b, M, h, rho, vd, 3, out_v);
  }
  if (out_stats) {
    out_stats[0] = T.nnodes;
    out_stats[1] = n_acc;
    out_stats[2] = n_dir;
  }
  free(ud); free(vd); free(X); free(Nr); free(W); free(F); free(Q);
  free(T.nodes); free(T.perm); free(T.mw);
  return rc;
}

int oracle_eval_tree(const double* src_xyz, const double* src_normal, const double* src_weight,
                     const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                     const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho[3],
                     int mode, int64_t N0, int p, double theta, int nthreads, double* out_u, double* out_v,
                     double* out_stats) {
  return eval_tree_impl(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, mode,
                        N0, p, theta, nthreads, 0, out_u, out_v, out_stats);
}

int oracle_eval_tree_sharp(const double* src_xyz, const double* src_normal, const double* src_weight,
                           const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                           const double* tgt_x0_density, int64_t M, int64_t N, double delta, int mode, int64_t N0,
                           int p, double theta, int nthreads, double* out_u, double* out_v, double* out_stats) {
  return eval_tree_impl(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, delta, NULL,
                        mode, N0, p, theta, nthreads, 1, out_u, out_v, out_stats);
}
