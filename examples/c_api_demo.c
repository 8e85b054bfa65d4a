/* c_api_demo.c -- the C ABI of include/stokes_er.h used from plain C (no Python):
 * the single layer of a constant density F on the unit sphere, evaluated at
 * targets on, inside and outside the sphere, against the closed form
 *   (1/8pi) int S F dS = (2/3) F            |y| <= 1 (Stokes' translating sphere)
 * Nodes: a Fibonacci lattice with equal weights 4 pi / N (a plain demo
 * quadrature, not the paper's); the extrapolated value still lands near the
 * closed form.  Build:
 *   gcc -O2 -I include -I /usr/local/cuda/include examples/c_api_demo.c -L paper_2507_00156_b200 -lstokes_er \
 *       -L /usr/local/cuda/lib64 -lcudart -lm -Wl,-rpath,$PWD/paper_2507_00156_b200 -o c_api_demo
 */
#include <cuda_runtime.h>
#include <math.h>
#include <stdio.h>
#include <stdlib.h>

#include "stokes_er.h"

#define CHECK(x)                                                                  \
  do {                                                                            \
    int st_ = (x);                                                                \
    if (st_) {                                                                    \
      fprintf(stderr, "%s failed: %s\n", #x, stokes_er_status_string(st_));       \
      return 1;                                                                   \
    }                                                                             \
  } while (0)

int main(void) {
  const int64_t N = 20000, M = 3;
  const double PI = 3.14159265358979323846, F[3] = {1.0, -0.5, 0.25};
  const double h = sqrt(4.0 * PI / N), rho[3] = {2.0, 3.0, 4.0};
  double *x = malloc(sizeof(double) * 3 * N), *w = malloc(sizeof(double) * N), *f = malloc(sizeof(double) * 3 * N);
  for (int64_t j = 0; j < N; ++j) {  /* Fibonacci lattice */
    const double z = 1.0 - (2.0 * j + 1.0) / N, r = sqrt(1.0 - z * z), phi = j * PI * (3.0 - sqrt(5.0));
    x[j] = r * cos(phi);
    x[N + j] = r * sin(phi);
    x[2 * N + j] = z;
    w[j] = 4.0 * PI / N;
    for (int d = 0; d < 3; ++d) f[d * N + j] = F[d];
  }
  /* targets y = x0 + b n0 with x0 = n0 = (0,0,1) and b = 0, -0.3, +0.5 */
  const double bs[3] = {0.0, -0.3, 0.5};
  double y[9], b[3], x0d[27];
  for (int t = 0; t < 3; ++t) {
    b[t] = bs[t];
    y[t] = 0.0;
    y[M + t] = 0.0;
    y[2 * M + t] = 1.0 + bs[t];
    for (int d = 0; d < 3; ++d) {
      x0d[d * M + t] = (d == 2);      /* n0 */
      x0d[(3 + d) * M + t] = F[d];    /* f(x0) */
      x0d[(6 + d) * M + t] = 0.0;     /* q(x0), unused in SL mode */
    }
  }
  double *dx, *dn, *dw, *df, *dy, *db, *dx0, *du;
  void* ws;
  const size_t wsb = stokes_er_workspace_bytes(M, N, STOKES_ER_SL);
  if (cudaMalloc((void**)&dx, 24 * N) || cudaMalloc((void**)&dn, 24 * N) || cudaMalloc((void**)&dw, 8 * N) ||
      cudaMalloc((void**)&df, 24 * N) || cudaMalloc((void**)&dy, 72) || cudaMalloc((void**)&db, 24) ||
      cudaMalloc((void**)&dx0, 216) || cudaMalloc((void**)&du, 72) || cudaMalloc(&ws, wsb)) {
    fprintf(stderr, "cudaMalloc failed (no GPU?)\n");
    return 2;
  }
  cudaMemcpy(dx, x, 24 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dn, x, 24 * N, cudaMemcpyHostToDevice); /* unit sphere: n = x */
  cudaMemcpy(dw, w, 8 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(df, f, 24 * N, cudaMemcpyHostToDevice);
  cudaMemcpy(dy, y, 72, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b, 24, cudaMemcpyHostToDevice);
  cudaMemcpy(dx0, x0d, 216, cudaMemcpyHostToDevice);
  CHECK(stokes_er_eval(dx, dn, dw, df, NULL, dy, db, dx0, M, N, h, rho, STOKES_ER_SL, du, NULL, ws, wsb, NULL));
  double u[9];
  if (cudaMemcpy(u, du, 72, cudaMemcpyDeviceToHost)) return 3;
  double err = 0.0;
  for (int t = 0; t < 2; ++t) /* on and inside: (2/3) F */
    for (int d = 0; d < 3; ++d) err = fmax(err, fabs(u[d * M + t] - 2.0 / 3.0 * F[d]));
  printf("c_api_demo: N=%lld h=%.4f u(on)=(%.6f %.6f %.6f) max |u - 2F/3| on/inside = %.2e\n", (long long)N, h, u[0],
         u[M], u[2 * M], err);
  return err < 1e-3 ? 0 : 4;
}
