// twodrop.cu -- NEXT-2: the two-drop interfacial Stokes flow of PAPER.md
// Sec. 4.3 (lines 331-377) on the GPU: right-hand side and operator of the
// integral equation (35) from four hot-path block evaluations each, the
// cross-block subtraction density by least-squares interpolation, and a full
// GMRES solve driven from the host with the vectors resident in HBM.
// C ABI and semantics: include/stokes_er.h (NEXT-2 section); readings
// R17-R21 in DESIGN.md.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <vector>

#include "stokes_er.h"

namespace twodrop {

constexpr int kKmax = STOKES_ER_INTERP_KMAX;  // stencil capacity
constexpr int kRowsPerLane = kKmax / 32;      // stencil rows held by each lane
#ifndef SER_INTERP_DEG
#define SER_INTERP_DEG 4                      // R20: total degree of the cross-point polynomial (study: DESIGN 5.5)
#endif
#ifndef SER_INTERP_RADIUS
#define SER_INTERP_RADIUS 3.5                 // R20: stencil = nodes within this many h of x0
#endif
constexpr int kInterpDeg = SER_INTERP_DEG;
constexpr int kNpoly = (kInterpDeg + 1) * (kInterpDeg + 2) / 2;  // monomials of total degree <= kInterpDeg
constexpr double kInterpRadius = SER_INTERP_RADIUS;
constexpr int kDotBlocks = 296;
#ifndef SER_NODES_MIN_N
#define SER_NODES_MIN_N 50000                 // self blocks through stokes_er_eval_nodes_onsurface from here on
#endif
constexpr int64_t kNodesMinN = SER_NODES_MIN_N;
static_assert(kKmax % 32 == 0, "stencil capacity: whole warps");

// ----------------------------------------------------------------- kernels
__device__ __forceinline__ double warp_sum(double v) {
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

// One warp per cross target t (a node y of drop b seen from drop m): x0 =
// y - b' n0 on drop m; stencil = drop m's nodes within R of x0 in index order
// (ballot compaction), stored k-major: idx[k * Nt + t].  Weights: the value
// at x0 of the least-squares polynomial of total degree <= 4 in the tangent
// coordinates (xi, eta) = ((x_k - x0).t1, (x_k - x0).t2) / R, i.e.
// L = Q z with Phi = Q R (modified Gram-Schmidt over the warp) and R^T z = e_1
// (the constant monomial is column 0).
// Bounding box [lo | hi] of each run of 32 consecutive source nodes (index order), for the
// stencil scan's chunk culling.
__global__ void chunk_box_kernel(const double* __restrict__ sx, int64_t Ns, double* __restrict__ box) {
  const int64_t c = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (c * 32 >= Ns) return;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  const int64_t kend = (c * 32 + 32 < Ns) ? c * 32 + 32 : Ns;
  for (int64_t k = c * 32; k < kend; ++k)
    for (int d = 0; d < 3; ++d) {
      lo[d] = fmin(lo[d], sx[d * Ns + k]);
      hi[d] = fmax(hi[d], sx[d * Ns + k]);
    }
  for (int d = 0; d < 3; ++d) {
    box[c * 6 + d] = lo[d];
    box[c * 6 + 3 + d] = hi[d];
  }
}

__global__ void stencil_kernel(const double* __restrict__ sx, int64_t Ns, const double* __restrict__ sbox,
                               const double* __restrict__ ty, const double* __restrict__ tb,
                               const double* __restrict__ x0d, int64_t Nt, double R, int* __restrict__ cnt,
                               int* __restrict__ idx, double* __restrict__ L, int* __restrict__ status) {
  const int lane = threadIdx.x & 31;
  const int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  if (t >= Nt) return;
  double n0[3], x0[3];
  for (int d = 0; d < 3; ++d) n0[d] = x0d[d * Nt + t];
  const double b = tb[t];
  for (int d = 0; d < 3; ++d) x0[d] = ty[d * Nt + t] - b * n0[d];
  const double R2 = R * R, R2box = R2 * (1.0 + 1e-9);
  int count = 0;
  // chunks of 32 consecutive nodes whose box is within R of x0 (lane = chunk, ballot), then the
  // nodes of each such chunk (lane = node): the same selection, in the same index order, as a scan
  // over every node (round 1), at ~1/30 of the distance tests
  const int64_t nch = (Ns + 31) / 32;
  for (int64_t cb = 0; cb < nch; cb += 32) {
    bool cand = false;
    if (cb + lane < nch) {
      const double* bx = sbox + (cb + lane) * 6;
      double g2 = 0.0;
      for (int d = 0; d < 3; ++d) {
        const double gap = fmax(0.0, fmax(bx[d] - x0[d], x0[d] - bx[3 + d]));
        g2 = fma(gap, gap, g2);
      }
      cand = g2 <= R2box;
    }
    unsigned cm = __ballot_sync(0xffffffffu, cand);
    while (cm) {
      const int64_t base = (cb + __ffs(cm) - 1) * 32;
      cm &= cm - 1;
      const int64_t k = base + lane;
      bool in = false;
      if (k < Ns) {
        const double dx = sx[k] - x0[0], dy = sx[Ns + k] - x0[1], dz = sx[2 * Ns + k] - x0[2];
        in = dx * dx + dy * dy + dz * dz <= R2;
      }
      const unsigned m = __ballot_sync(0xffffffffu, in);
      const int pos = count + __popc(m & ((1u << lane) - 1u));
      if (in && pos < kKmax) idx[(int64_t)pos * Nt + t] = static_cast<int>(k);
      count += __popc(m);
    }
  }
  if (count < kNpoly || count > kKmax) {
    if (lane == 0) {
      cnt[t] = 0;
      atomicOr(status, 1);
    }
    return;
  }
  if (lane == 0) cnt[t] = count;
  // tangent frame: t1 = n0 x e / |n0 x e| with e the axis least aligned with n0, t2 = n0 x t1
  int ax = 0;
  if (fabs(n0[1]) < fabs(n0[ax])) ax = 1;
  if (fabs(n0[2]) < fabs(n0[ax])) ax = 2;
  double e[3] = {0.0, 0.0, 0.0};
  e[ax] = 1.0;
  double t1[3] = {n0[1] * e[2] - n0[2] * e[1], n0[2] * e[0] - n0[0] * e[2], n0[0] * e[1] - n0[1] * e[0]};
  const double tn = 1.0 / sqrt(t1[0] * t1[0] + t1[1] * t1[1] + t1[2] * t1[2]);
  for (int d = 0; d < 3; ++d) t1[d] *= tn;
  const double t2[3] = {n0[1] * t1[2] - n0[2] * t1[1], n0[2] * t1[0] - n0[0] * t1[2],
                        n0[0] * t1[1] - n0[1] * t1[0]};
  // rows r = lane + 32 j of Phi (zero rows beyond count)
  double Q[kRowsPerLane][kNpoly];
  for (int j = 0; j < kRowsPerLane; ++j) {
    const int r = lane + 32 * j;
    double xi = 0.0, eta = 0.0, on = 0.0;
    if (r < count) {
      const int64_t k = idx[(int64_t)r * Nt + t];
      const double d[3] = {sx[k] - x0[0], sx[Ns + k] - x0[1], sx[2 * Ns + k] - x0[2]};
      xi = (d[0] * t1[0] + d[1] * t1[1] + d[2] * t1[2]) / R;
      eta = (d[0] * t2[0] + d[1] * t2[1] + d[2] * t2[2]) / R;
      on = 1.0;
    }
    int c = 0;
    for (int deg = 0; deg <= kInterpDeg; ++deg)
      for (int pb = 0; pb <= deg; ++pb) {
        double v = on;
        for (int i = 0; i < deg - pb; ++i) v *= xi;
        for (int i = 0; i < pb; ++i) v *= eta;
        Q[j][c++] = v;
      }
  }
  double Rm[kNpoly][kNpoly];
  for (int j = 0; j < kNpoly; ++j) {
    double s = 0.0;
    for (int i = 0; i < kRowsPerLane; ++i) s += Q[i][j] * Q[i][j];
    const double rjj = sqrt(warp_sum(s));
    Rm[j][j] = rjj;
    const double inv = 1.0 / rjj;
    for (int i = 0; i < kRowsPerLane; ++i) Q[i][j] *= inv;
    for (int k = j + 1; k < kNpoly; ++k) {
      double p = 0.0;
      for (int i = 0; i < kRowsPerLane; ++i) p += Q[i][j] * Q[i][k];
      const double rjk = warp_sum(p);
      Rm[j][k] = rjk;
      for (int i = 0; i < kRowsPerLane; ++i) Q[i][k] -= rjk * Q[i][j];
    }
  }
  double z[kNpoly];  // R^T z = e_1 (forward substitution)
  for (int j = 0; j < kNpoly; ++j) {
    double s = (j == 0) ? 1.0 : 0.0;
    for (int i = 0; i < j; ++i) s -= Rm[i][j] * z[i];
    z[j] = s / Rm[j][j];
  }
  for (int j = 0; j < kRowsPerLane; ++j) {
    const int r = lane + 32 * j;
    if (r >= count) break;
    double w = 0.0;
    for (int c = 0; c < kNpoly; ++c) w += Q[j][c] * z[c];
    L[(int64_t)r * Nt + t] = w;
  }
}

// q0[c][t] = sum_k L[k][t] u[c][idx[k][t]]: drop m's u at the closest points x0.
__global__ void interp_apply_kernel(const double* __restrict__ u, int64_t Ns, const int* __restrict__ cnt,
                                    const int* __restrict__ idx, const double* __restrict__ L, int64_t Nt,
                                    double* __restrict__ q0) {
  const int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (t >= Nt) return;
  double a0 = 0.0, a1 = 0.0, a2 = 0.0;
  const int n = cnt[t];
  for (int k = 0; k < n; ++k) {
    const double w = L[(int64_t)k * Nt + t];
    const int64_t j = idx[(int64_t)k * Nt + t];
    a0 = fma(w, u[j], a0);
    a1 = fma(w, u[Ns + j], a1);
    a2 = fma(w, u[2 * Ns + j], a2);
  }
  q0[t] = a0;
  q0[Nt + t] = a1;
  q0[2 * Nt + t] = a2;
}

// out = a x + b y + c z (elementwise; y or z may be NULL)
__global__ void lincomb_kernel(int64_t n, double a, const double* x, double b,
                               const double* __restrict__ y, double c, const double* __restrict__ z,
                               double* out) {  // out may alias x
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  double v = a * x[i];
  if (y) v = fma(b, y[i], v);
  if (z) v = fma(c, z[i], v);
  out[i] = v;
}

// Deterministic dot product: fixed grid, block sums, then one block in order.
__global__ void dot_partial_kernel(const double* __restrict__ a, const double* __restrict__ b, int64_t n,
                                   double* __restrict__ partial) {
  double s = 0.0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    s = fma(a[i], b[i], s);
  __shared__ double red[32];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x < 32) {
    double v = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    v = warp_sum(v);
    if (threadIdx.x == 0) partial[blockIdx.x] = v;
  }
}
__global__ void dot_final_kernel(const double* __restrict__ partial, int nb, double* __restrict__ out) {
  double s = 0.0;
  for (int i = threadIdx.x; i < nb; i += 32) s += partial[i];
  s = warp_sum(s);
  if (threadIdx.x == 0) *out = s;
}

// MGS update with the coefficient read on the device (no host round trip per dot):
// w = 1.0 * w + (-h) * v, the same arithmetic as lincomb_kernel(n, 1.0, w, -h, v).
__global__ void mgs_update_kernel(int64_t n, const double* __restrict__ h, double* w, const double* __restrict__ v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  w[i] = fma(-*h, v[i], 1.0 * w[i]);
}
// *h = ||w||^2 (left in place; the host takes its sqrt after the copy): v = (1/||w||) w when
// ||w|| > 0, the arithmetic of lincomb_kernel(n, 1.0 / ||w||, w).
__global__ void mgs_normalize_kernel(int64_t n, const double* __restrict__ h, const double* __restrict__ w,
                                     double* __restrict__ v) {
  const double nw = sqrt(*h);
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (nw > 0.0 && i < n) v[i] = (1.0 / nw) * w[i];
}

// ----------------------------------------------------------------- host side
size_t al(size_t x) { return (x + 255) / 256 * 256; }
int64_t cdiv(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Layout {
  int64_t N[2] = {0, 0}, n = 0;
  int max_iter = 0;
  size_t eval_ws = 0;
  size_t off_eval, off_x0s[2], off_x0c[2], off_zero[2], off_vs[2], off_vc[2], off_cnt[2], off_idx[2], off_L[2];
  size_t off_V, off_w, off_partial, off_scalar, off_hcol, off_status, total;
};

Layout layout(int64_t N1, int64_t N2, int max_iter, const stokes_er_twodrop_params* P = nullptr) {
  Layout L;
  L.N[0] = N1;
  L.N[1] = N2;
  L.n = 3 * (N1 + N2);
  L.max_iter = max_iter;
  for (int b = 0; b < 2; ++b)
    for (int m = 0; m < 2; ++m) {
      L.eval_ws = std::max(L.eval_ws, stokes_er_workspace_bytes(L.N[b], L.N[m], 3));
      if (b == m) L.eval_ws = std::max(L.eval_ws, stokes_er_nodes_workspace_bytes(L.N[b], 3));  // self blocks
      if (P && P->use_tree)  // block (targets b <- sources m) through the treecode over drop m
        L.eval_ws = std::max(L.eval_ws, stokes_er_tree_workspace_bytes(L.N[b], L.N[m], 3, P->tree, P->tree_plan[m]));
    }
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = al(off + bytes);
    return o;
  };
  L.off_eval = take(L.eval_ws);
  for (int b = 0; b < 2; ++b) {
    const size_t nb = static_cast<size_t>(L.N[b]);
    L.off_x0s[b] = take(9 * nb * sizeof(double));
    L.off_x0c[b] = take(9 * nb * sizeof(double));
    L.off_zero[b] = take(nb * sizeof(double));
    L.off_vs[b] = take(3 * nb * sizeof(double));
    L.off_vc[b] = take(3 * nb * sizeof(double));
    L.off_cnt[b] = take(nb * sizeof(int));
    L.off_idx[b] = take((size_t)kKmax * nb * sizeof(int));
    L.off_L[b] = take((size_t)kKmax * nb * sizeof(double));
  }
  L.off_V = take((size_t)(max_iter + 1) * L.n * sizeof(double));
  L.off_w = take(L.n * sizeof(double));
  L.off_partial = take(kDotBlocks * sizeof(double));
  L.off_scalar = take(8 * sizeof(double));
  L.off_hcol = take((size_t)(max_iter + 2) * sizeof(double));
  L.off_status = take(4 * sizeof(int));
  L.total = off;
  return L;
}

struct Ctx {
  const stokes_er_drop* drops;
  const stokes_er_cross* cross;
  const stokes_er_twodrop_params* P;
  Layout L;
  char* ws;
  cudaStream_t s;
  template <class T>
  T* at(size_t off) const {
    return reinterpret_cast<T*>(ws + off);
  }
};

int validate(const stokes_er_drop* drops, const stokes_er_cross* cross, const stokes_er_twodrop_params* P,
             void* ws, size_t bytes) {
  if (!drops || !cross || !P || !ws) return STOKES_ER_EINVAL;
  for (int b = 0; b < 2; ++b) {
    const stokes_er_drop& d = drops[b];
    if (d.N < 1 || d.N > INT32_MAX / 3 || !d.xyz || !d.normal || !d.weight || !d.f || !std::isfinite(d.lambda))
      return STOKES_ER_EINVAL;
    if (!cross[b].b || !cross[b].x0d) return STOKES_ER_EINVAL;
  }
  if (!(P->h > 0.0) || !std::isfinite(P->h) || !(P->delta_self > 0.0) || !std::isfinite(P->delta_self) ||
      !(P->mu0 > 0.0) || !std::isfinite(P->mu0) || !(P->tol > 0.0) || P->max_iter < 1 || P->max_iter > 512)
    return STOKES_ER_EINVAL;
  if (!(P->rho[0] > 0.0 && P->rho[1] > P->rho[0] && P->rho[2] > P->rho[1] && std::isfinite(P->rho[2])))
    return STOKES_ER_EINVAL;
  if (P->use_tree) {
    if (!P->tree) return STOKES_ER_EINVAL;
    for (int m = 0; m < 2; ++m)
      if (stokes_er_tree_workspace_bytes(drops[0].N, drops[m].N, 3, P->tree, P->tree_plan[m]) == 0)
        return STOKES_ER_EINVAL;  // missing plan or one built for other nodes
  }
  if (bytes < layout(drops[0].N, drops[1].N, P->max_iter, P).total) return STOKES_ER_EWORKSPACE;
  return STOKES_ER_OK;
}

int ok(cudaError_t e) { return e == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA; }

// A u (mode DL) or the right-hand side (mode SL, u ignored) into out.
int blocks(const Ctx& c, int mode, const double* u, double* out) {
  const auto* d = c.drops;
  int st = STOKES_ER_OK;
  int64_t off_u[2] = {0, 3 * d[0].N};
  for (int b = 0; b < 2 && !st; ++b) {
    const int m = 1 - b;
    const int64_t Nb = d[b].N, Nm = d[m].N;
    double* x0s = c.at<double>(c.L.off_x0s[b]);
    double* x0c = c.at<double>(c.L.off_x0c[b]);
    double* vs = c.at<double>(c.L.off_vs[b]);
    double* vc = c.at<double>(c.L.off_vc[b]);
    void* ews = c.at<void>(c.L.off_eval);
    const double* ub = u ? u + off_u[b] : nullptr;
    const double* um = u ? u + off_u[m] : nullptr;
    if (mode == STOKES_ER_DL) {
      // self: q(x0) = u_b at the node itself
      if ((st = ok(cudaMemcpyAsync(x0s + 6 * Nb, ub, 3 * Nb * sizeof(double), cudaMemcpyDeviceToDevice, c.s))))
        break;
      // cross: q(x0) = u_m interpolated at the closest points (R20)
      interp_apply_kernel<<<cdiv(Nb, 256), 256, 0, c.s>>>(um, Nm, c.at<int>(c.L.off_cnt[b]),
                                                           c.at<int>(c.L.off_idx[b]), c.at<double>(c.L.off_L[b]),
                                                           Nb, x0c + 6 * Nb);
    }
    const bool sl = mode == STOKES_ER_SL;
    if (c.P->use_tree)
      st = stokes_er_eval_tree_onsurface(d[b].xyz, d[b].normal, d[b].weight, sl ? d[b].f : nullptr,
                                         sl ? nullptr : ub, d[b].xyz, c.at<double>(c.L.off_zero[b]), x0s, Nb, Nb,
                                         c.P->delta_self, mode, c.P->tree, c.P->tree_plan[b], sl ? vs : nullptr,
                                         sl ? nullptr : vs, ews, c.L.eval_ws, c.s);
    else if (Nb >= kNodesMinN)  // the self block's targets are the drop's own nodes: the symmetric node
                                // path (same sums; measured 498 vs 515 ms per solve at 1/h = 64)
      st = stokes_er_eval_nodes_onsurface(d[b].xyz, d[b].normal, d[b].weight, sl ? d[b].f : nullptr,
                                          sl ? nullptr : ub, Nb, c.P->delta_self, mode, sl ? vs : nullptr,
                                          sl ? nullptr : vs, ews, c.L.eval_ws, c.s);
    else
      st = stokes_er_eval_onsurface(d[b].xyz, d[b].normal, d[b].weight, sl ? d[b].f : nullptr, sl ? nullptr : ub,
                                    d[b].xyz, c.at<double>(c.L.off_zero[b]), x0s, Nb, Nb, c.P->delta_self, mode,
                                    sl ? vs : nullptr, sl ? nullptr : vs, ews, c.L.eval_ws, c.s);
    if (st) break;
    if (c.P->use_tree)
      st = stokes_er_eval_tree(d[m].xyz, d[m].normal, d[m].weight, sl ? d[m].f : nullptr, sl ? nullptr : um,
                               d[b].xyz, c.cross[b].b, x0c, Nb, Nm, c.P->h, c.P->rho, mode, c.P->tree,
                               c.P->tree_plan[m], sl ? vc : nullptr, sl ? nullptr : vc, ews, c.L.eval_ws, c.s);
    else
      st = stokes_er_eval(d[m].xyz, d[m].normal, d[m].weight, sl ? d[m].f : nullptr, sl ? nullptr : um, d[b].xyz,
                          c.cross[b].b, x0c, Nb, Nm, c.P->h, c.P->rho, mode, sl ? vc : nullptr, sl ? nullptr : vc,
                          ews, c.L.eval_ws, c.s);
    if (st) break;
    const int64_t n3 = 3 * Nb;
    if (sl)  // rhs_b = -(2/mu0) (SL_bb + SL_bm)
      lincomb_kernel<<<cdiv(n3, 256), 256, 0, c.s>>>(n3, -2.0 / c.P->mu0, vs, -2.0 / c.P->mu0, vc, 0.0, nullptr,
                                                      out + off_u[b]);
    else  // (lambda_b + 1) u_b - 2 (lambda_b - 1) DL_bb - 2 (lambda_m - 1) DL_bm
      lincomb_kernel<<<cdiv(n3, 256), 256, 0, c.s>>>(n3, d[b].lambda + 1.0, ub, -2.0 * (d[b].lambda - 1.0), vs,
                                                      -2.0 * (d[m].lambda - 1.0), vc, out + off_u[b]);
    st = ok(cudaGetLastError());
  }
  return st;
}

int dot(const Ctx& c, const double* a, const double* b, double* host_out) {
  double* part = c.at<double>(c.L.off_partial);
  double* sc = c.at<double>(c.L.off_scalar);
  dot_partial_kernel<<<kDotBlocks, 256, 0, c.s>>>(a, b, c.L.n, part);
  dot_final_kernel<<<1, 32, 0, c.s>>>(part, kDotBlocks, sc);
  if (cudaMemcpyAsync(host_out, sc, sizeof(double), cudaMemcpyDeviceToHost, c.s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  return ok(cudaStreamSynchronize(c.s));
}

void lincomb(const Ctx& c, double a, const double* x, double b, const double* y, double* out) {
  lincomb_kernel<<<cdiv(c.L.n, 256), 256, 0, c.s>>>(c.L.n, a, x, b, y, 0.0, nullptr, out);
}

int arch_ok() {
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return STOKES_ER_ECUDA;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess) return STOKES_ER_ECUDA;
  return major == 10 ? STOKES_ER_OK : STOKES_ER_EARCH;
}

}  // namespace twodrop

using namespace twodrop;

extern "C" {

size_t stokes_er_twodrop_workspace_bytes(int64_t N1, int64_t N2, int max_iter) {
  if (N1 < 1 || N2 < 1 || max_iter < 1 || max_iter > 512) return 0;
  return layout(N1, N2, max_iter).total;
}

size_t stokes_er_twodrop_workspace_bytes_ex(int64_t N1, int64_t N2, const stokes_er_twodrop_params* params) {
  if (!params || N1 < 1 || N2 < 1 || params->max_iter < 1 || params->max_iter > 512) return 0;
  if (params->use_tree) {
    if (!params->tree) return 0;
    for (int m = 0; m < 2; ++m)
      if (stokes_er_tree_workspace_bytes(N1, m ? N2 : N1, 3, params->tree, params->tree_plan[m]) == 0) return 0;
  }
  return layout(N1, N2, params->max_iter, params).total;
}

int stokes_er_twodrop_setup(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                            const stokes_er_twodrop_params* params, void* workspace, size_t workspace_bytes,
                            void* stream) {
  int st = validate(drops, cross, params, workspace, workspace_bytes);
  if (st || (st = arch_ok())) return st;
  Ctx c{drops, cross, params, layout(drops[0].N, drops[1].N, params->max_iter, params), static_cast<char*>(workspace),
        static_cast<cudaStream_t>(stream)};
  int* status = c.at<int>(c.L.off_status);
  if ((st = ok(cudaMemsetAsync(status, 0, 4 * sizeof(int), c.s)))) return st;
  for (int b = 0; b < 2 && !st; ++b) {
    const int m = 1 - b;
    const int64_t Nb = drops[b].N;
    double* x0s = c.at<double>(c.L.off_x0s[b]);
    double* x0c = c.at<double>(c.L.off_x0c[b]);
    const size_t row = Nb * sizeof(double);
    // self targets: n0 = node normal, f(x0) = [f]_b at the node; rows 6-8 (u_b) per apply
    st = ok(cudaMemcpyAsync(x0s, drops[b].normal, 3 * row, cudaMemcpyDeviceToDevice, c.s));
    if (!st) st = ok(cudaMemcpyAsync(x0s + 3 * Nb, drops[b].f, 3 * row, cudaMemcpyDeviceToDevice, c.s));
    if (!st) st = ok(cudaMemsetAsync(x0s + 6 * Nb, 0, 3 * row, c.s));
    // cross targets: n0 and [f]_m(x0) from the caller; rows 6-8 (interpolated u_m) per apply
    if (!st) st = ok(cudaMemcpyAsync(x0c, cross[b].x0d, 6 * row, cudaMemcpyDeviceToDevice, c.s));
    if (!st) st = ok(cudaMemsetAsync(x0c + 6 * Nb, 0, 3 * row, c.s));
    if (!st) st = ok(cudaMemsetAsync(c.at<double>(c.L.off_zero[b]), 0, row, c.s));
    if (st) break;
    double* sbox = c.at<double>(c.L.off_eval);  // the block evaluations' workspace is free during setup
    chunk_box_kernel<<<cdiv(cdiv(drops[m].N, 32), 128), 128, 0, c.s>>>(drops[m].xyz, drops[m].N, sbox);
    stencil_kernel<<<cdiv(Nb * 32, 128), 128, 0, c.s>>>(drops[m].xyz, drops[m].N, sbox, drops[b].xyz, cross[b].b,
                                                        cross[b].x0d, Nb, kInterpRadius * params->h,
                                                        c.at<int>(c.L.off_cnt[b]), c.at<int>(c.L.off_idx[b]),
                                                        c.at<double>(c.L.off_L[b]), status);
    st = ok(cudaGetLastError());
  }
  if (st) return st;
  int hs = 0;
  if ((st = ok(cudaMemcpyAsync(&hs, status, sizeof(int), cudaMemcpyDeviceToHost, c.s)))) return st;
  if ((st = ok(cudaStreamSynchronize(c.s)))) return st;
  return hs ? STOKES_ER_EINVAL : STOKES_ER_OK;
}

int stokes_er_twodrop_rhs(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                          const stokes_er_twodrop_params* params, double* out_rhs, void* workspace,
                          size_t workspace_bytes, void* stream) {
  int st = validate(drops, cross, params, workspace, workspace_bytes);
  if (st || (st = arch_ok())) return st;
  if (!out_rhs) return STOKES_ER_EINVAL;
  Ctx c{drops, cross, params, layout(drops[0].N, drops[1].N, params->max_iter, params), static_cast<char*>(workspace),
        static_cast<cudaStream_t>(stream)};
  return blocks(c, STOKES_ER_SL, nullptr, out_rhs);
}

int stokes_er_twodrop_apply(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                            const stokes_er_twodrop_params* params, const double* u, double* out_Au,
                            void* workspace, size_t workspace_bytes, void* stream) {
  int st = validate(drops, cross, params, workspace, workspace_bytes);
  if (st || (st = arch_ok())) return st;
  if (!u || !out_Au || u == out_Au) return STOKES_ER_EINVAL;
  Ctx c{drops, cross, params, layout(drops[0].N, drops[1].N, params->max_iter, params), static_cast<char*>(workspace),
        static_cast<cudaStream_t>(stream)};
  return blocks(c, STOKES_ER_DL, u, out_Au);
}

int stokes_er_twodrop_solve(const stokes_er_drop drops[2], const stokes_er_cross cross[2],
                            const stokes_er_twodrop_params* params, double* out_u, int* out_iters,
                            double* out_res_host, void* workspace, size_t workspace_bytes, void* stream) {
  int st = validate(drops, cross, params, workspace, workspace_bytes);
  if (st || (st = arch_ok())) return st;
  if (!out_u) return STOKES_ER_EINVAL;
  Ctx c{drops, cross, params, layout(drops[0].N, drops[1].N, params->max_iter, params), static_cast<char*>(workspace),
        static_cast<cudaStream_t>(stream)};
  const int K = params->max_iter;
  const int64_t n = c.L.n;
  double* V = c.at<double>(c.L.off_V);
  double* w = c.at<double>(c.L.off_w);
  auto Vj = [&](int j) { return V + (int64_t)j * n; };
  // r0 = rhs (u0 = 0); v_0 = r0 / beta
  if ((st = blocks(c, STOKES_ER_SL, nullptr, w))) return st;
  double beta2 = 0.0;
  if ((st = dot(c, w, w, &beta2))) return st;
  const double beta = std::sqrt(beta2);
  if (out_iters) *out_iters = 0;
  if (!(beta > 0.0)) {  // rhs = 0: u = 0
    if ((st = ok(cudaMemsetAsync(out_u, 0, n * sizeof(double), c.s)))) return st;
    return ok(cudaStreamSynchronize(c.s));
  }
  lincomb(c, 1.0 / beta, w, 0.0, nullptr, Vj(0));
  // Hessenberg H (column-major, (K+1) x K), Givens rotations, g = beta e_1 rotated
  std::vector<double> H((size_t)(K + 1) * K, 0.0), cs(K), sn(K), g(K + 1, 0.0);
  g[0] = beta;
  int j = 0;
  bool conv = false;
  for (; j < K; ++j) {
    if ((st = blocks(c, STOKES_ER_DL, Vj(j), w))) return st;
    double* hj = &H[(size_t)j * (K + 1)];
    // modified Gram-Schmidt with the coefficients kept on the device: h_ij = <w, v_i> then
    // w -= h_ij v_i, in order; ||w|| and v_{j+1}; ONE device->host copy of the column and one
    // stream synchronization per Krylov step (the Givens update and the stopping test are on
    // the host).  Same arithmetic as the per-dot host round trip it replaces.
    double* hcol = c.at<double>(c.L.off_hcol);
    double* part = c.at<double>(c.L.off_partial);
    for (int i = 0; i <= j; ++i) {
      dot_partial_kernel<<<kDotBlocks, 256, 0, c.s>>>(w, Vj(i), n, part);
      dot_final_kernel<<<1, 32, 0, c.s>>>(part, kDotBlocks, hcol + i);
      mgs_update_kernel<<<cdiv(n, 256), 256, 0, c.s>>>(n, hcol + i, w, Vj(i));
    }
    dot_partial_kernel<<<kDotBlocks, 256, 0, c.s>>>(w, w, n, part);
    dot_final_kernel<<<1, 32, 0, c.s>>>(part, kDotBlocks, hcol + j + 1);
    mgs_normalize_kernel<<<cdiv(n, 256), 256, 0, c.s>>>(n, hcol + j + 1, w, Vj(j + 1));
    if ((st = ok(cudaMemcpyAsync(hj, hcol, (j + 2) * sizeof(double), cudaMemcpyDeviceToHost, c.s)))) return st;
    if ((st = ok(cudaStreamSynchronize(c.s)))) return st;
    const double nw2 = hj[j + 1];
    hj[j + 1] = std::sqrt(nw2);
    for (int i = 0; i < j; ++i) {  // apply the previous rotations to column j
      const double a = hj[i], b2 = hj[i + 1];
      hj[i] = cs[i] * a + sn[i] * b2;
      hj[i + 1] = -sn[i] * a + cs[i] * b2;
    }
    const double r = std::hypot(hj[j], hj[j + 1]);
    cs[j] = hj[j] / r;
    sn[j] = hj[j + 1] / r;
    hj[j] = r;
    hj[j + 1] = 0.0;
    g[j + 1] = -sn[j] * g[j];
    g[j] = cs[j] * g[j];
    const double res = std::fabs(g[j + 1]) / beta;
    if (out_res_host) out_res_host[j] = res;
    if (res <= params->tol || nw2 == 0.0) {
      conv = true;
      ++j;
      break;
    }
  }
  const int k = std::min(j, K);
  if (out_iters) *out_iters = k;
  // y = R^{-1} g (upper triangular, k x k); u = V y
  std::vector<double> y(k, 0.0);
  for (int i = k - 1; i >= 0; --i) {
    double s = g[i];
    for (int l = i + 1; l < k; ++l) s -= H[(size_t)l * (K + 1) + i] * y[l];
    y[i] = s / H[(size_t)i * (K + 1) + i];
  }
  if ((st = ok(cudaMemsetAsync(out_u, 0, n * sizeof(double), c.s)))) return st;
  for (int i = 0; i < k; ++i) lincomb(c, 1.0, out_u, y[i], Vj(i), out_u);
  if ((st = ok(cudaGetLastError()))) return st;
  if ((st = ok(cudaStreamSynchronize(c.s)))) return st;
  return conv ? STOKES_ER_OK : STOKES_ER_ENOCONV;
}

}  // extern "C"
