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

  for (int64_t s = 0; s < N; ++s) {
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
