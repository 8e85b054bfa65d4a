// treecode.cuh -- NEXT-3: the kernel-independent treecode of PAPER.md Sec. 3.4
// (lines 194-233) for the far part of the localized sums, on sm_100a.
//
//   host   : octree over the sources (stokes_er_tree_build, readings R22)
//   KW     : modified weights, eq. (32), at the (p+1)^3 second-kind Chebyshev
//            points of every cluster box (R24), 12 channels: f w, n w (SL) and the
//            symmetric part of q_a n_c w (DL: T contracts it with d_a d_c; the DL n w
//            channel is the SL one): leaves from their
//            sources (tree_p2m_kernel), internal nodes from their children level by
//            level (tree_m2m_kernel, separable; exact for degree-p interpolants)
//   KT     : far part per target: a warp of 32 Morton-consecutive targets walks
//            the tree depth-first with a warp-uniform stack of (cluster, lane
//            mask); each lane decides MAC + regularization guard for its own
//            target (R23, plain FP64 in the oracle's order, so the decisions are
//            the oracle's); accepted lanes add eq. (31) at the cluster's
//            Chebyshev points (or, R26, its far pairs directly when it has at most
//            (p+1)^3 points), lanes that reject a leaf add its far pairs directly
//            (near pairs masked)                                -- tree_far_kernel
//   K3     : the near pairs, all in directly summed leaves (R23), by the near
//            units of the direct path over the tree-ordered sources
//   K2     : finalize (far partial + near phases, 1/(8pi), -6, chi q0)
// Included by stokes_er.cu (one translation unit with kernels.cuh).
#pragma once

#include <cmath>
#include <vector>

namespace ser {

constexpr int kTreeMaxDegree = 16;
constexpr int kTreeCh = 12;               // fw(3) nw(3) symmetric part of q_a n_c w (6)
constexpr int kTreeStack = 512;           // DFS stack entries per warp (depth <= 63)
constexpr int kTreeWarps = 4;             // warps per CTA of tree_far_kernel
#ifndef SER_TREE_MINB
#define SER_TREE_MINB 3  // 12 warps/SM at 168 registers with the two-proxy loop (4: 128 registers, spills)
#endif
#ifndef SER_TREE_FUSED_NEAR
#define SER_TREE_FUSED_NEAR 1  // near units interleaved in the walk kernel's queue (0: separate near_kernel)
#endif
constexpr uint64_t kTreeMagic = 0x53455254524545ULL;  // "SERTREE"

struct TreeNode {  // POD, identical on host and device
  double lo[3], hi[3], c[3], rc;
  int32_t begin, end, first_child, nchild, level, pad;
};

struct TreePlanHeader {
  uint64_t magic;
  int64_t N;
  int32_t nnodes, max_nodes, leaf_size, depth;
  int64_t off_nodes, off_perm;  // byte offsets inside the plan
};

inline int64_t tree_max_nodes(int64_t N, int64_t N0) { return 8 * (N / N0) + 4096; }

inline size_t tree_plan_bytes(int64_t N, int64_t N0) {
  return sizeof(TreePlanHeader) + 64 + (size_t)tree_max_nodes(N, N0) * sizeof(TreeNode) + (size_t)N * 4 + 64;
}

// ---------------------------------------------------------------- host build (R22)
struct TreeBuilder {
  const double* x;  // [3][N] host
  int64_t N, N0;
  std::vector<int32_t> idx, tmp;
  std::vector<TreeNode> nodes;
  int64_t max_nodes;
  int depth = 0;

  void tight_box(TreeNode& t) const {
    for (int d = 0; d < 3; ++d) { t.lo[d] = INFINITY; t.hi[d] = -INFINITY; }
    for (int64_t j = t.begin; j < t.end; ++j)
      for (int d = 0; d < 3; ++d) {
        const double v = x[d * N + idx[j]];
        if (v < t.lo[d]) t.lo[d] = v;
        if (v > t.hi[d]) t.hi[d] = v;
      }
    double s = 0.0;
    for (int d = 0; d < 3; ++d) {
      const double w = t.hi[d] - t.lo[d];
      t.c[d] = 0.5 * (t.lo[d] + t.hi[d]);
      s = s + w * w;
    }
    t.rc = 0.5 * std::sqrt(s);
  }

  bool split(int self, int level) {
    if (level > depth) depth = level;
    if (level >= 63) return false;
    TreeNode t = nodes[self];
    nodes[self].first_child = -1;
    nodes[self].nchild = 0;
    const int64_t n = t.end - t.begin;
    int axes = 0;
    for (int d = 0; d < 3; ++d)
      if (t.hi[d] > t.lo[d]) axes |= 1 << d;
    if (n <= N0 || !axes) return true;
    double mid[3];
    for (int d = 0; d < 3; ++d) mid[d] = 0.5 * (t.lo[d] + t.hi[d]);
    auto oct = [&](int32_t j) {
      int o = 0;
      for (int d = 0; d < 3; ++d)
        if ((axes >> d & 1) && x[d * N + j] >= mid[d]) o |= 1 << d;
      return o;
    };
    int64_t cnt[8] = {0, 0, 0, 0, 0, 0, 0, 0}, start[8], pos[8];
    for (int64_t j = t.begin; j < t.end; ++j) cnt[oct(idx[j])]++;
    start[0] = t.begin;
    for (int o = 1; o < 8; ++o) start[o] = start[o - 1] + cnt[o - 1];
    for (int o = 0; o < 8; ++o) pos[o] = start[o];
    for (int64_t j = t.begin; j < t.end; ++j) tmp[pos[oct(idx[j])]++] = idx[j];  // stable per octant
    for (int64_t j = t.begin; j < t.end; ++j) idx[j] = tmp[j];
    int nc = 0;
    for (int o = 0; o < 8; ++o) nc += cnt[o] > 0;
    if ((int64_t)nodes.size() + nc > max_nodes) return false;
    const int first = static_cast<int>(nodes.size());
    nodes[self].first_child = first;
    nodes[self].nchild = nc;
    for (int o = 0; o < 8; ++o) {
      if (!cnt[o]) continue;
      TreeNode ch{};
      ch.level = level + 1;
      ch.begin = static_cast<int32_t>(start[o]);
      ch.end = static_cast<int32_t>(start[o] + cnt[o]);
      tight_box(ch);
      nodes.push_back(ch);
    }
    for (int k = first; k < first + nc; ++k)
      if (!split(k, level + 1)) return false;
    return true;
  }
};

// ---------------------------------------------------------------- device helpers
// 1-D barycentric Lagrange basis on the second-kind Chebyshev points of [lo, hi] (R24).
__device__ __forceinline__ void tree_lagrange(double x, double lo, double hi, int p, const double* __restrict__ cosk,
                                              double* L) {
  const double w = hi - lo;
  for (int k = 0; k <= p; ++k) L[k] = 0.0;
  if (!(w > 0.0)) { L[0] = 1.0; return; }
  const double c = 0.5 * (lo + hi), half = 0.5 * w;
  int hit = -1;
  double den = 0.0;
  for (int k = 0; k <= p; ++k) {
    const double s = c + half * cosk[k];
    const double dx = x - s;
    if (hit < 0 && fabs(dx) <= 1e-14 * w) hit = k;
    const double bw = ((k & 1) ? -1.0 : 1.0) * ((k == 0 || k == p) ? 0.5 : 1.0);
    L[k] = bw / dx;
    den += L[k];
  }
  if (hit >= 0) {
    for (int k = 0; k <= p; ++k) L[k] = 0.0;
    L[hit] = 1.0;
    return;
  }
  const double inv = 1.0 / den;
  for (int k = 0; k <= p; ++k) L[k] *= inv;
}

// KW1 (leaves): modified weights, eq. (32): G[node][k][ch] = sum_j L_k(x_j) g_ch(x_j),
// sources j of the leaf in tree order.  One CTA per leaf (ids[blockIdx.x]);
// threads own proxy points.
constexpr int kTwChunk = 32;
template <int MODE>
__global__ void __launch_bounds__(256) tree_p2m_kernel(const TreeNode* __restrict__ nodes,
                                                       const int* __restrict__ ids, const double* __restrict__ src,
                                                       int p, double* __restrict__ G) {
  __shared__ double sL[kTwChunk][3][kTreeMaxDegree + 1];
  __shared__ double sg[kTwChunk][kTreeCh];
  __shared__ double cosk[kTreeMaxDegree + 1];
  const int node = ids[blockIdx.x];
  const TreeNode nd = nodes[node];
  const int P1 = p + 1, NP = P1 * P1 * P1;
  if (threadIdx.x <= p) cosk[threadIdx.x] = cos(threadIdx.x * kPi / p);
  double* Gn = G + (size_t)node * NP * kTreeCh;
  for (int k0 = 0; k0 < NP; k0 += blockDim.x) {
    const int k = k0 + threadIdx.x;
    const int k1 = k / (P1 * P1), k2 = (k / P1) % P1, k3 = k % P1;
    double acc[kTreeCh];
#pragma unroll
    for (int c = 0; c < kTreeCh; ++c) acc[c] = 0.0;
    for (int j0 = nd.begin; j0 < nd.end; j0 += kTwChunk) {
      __syncthreads();  // previous chunk consumed (and cosk written)
      const int nj = min(kTwChunk, nd.end - j0);
      if (threadIdx.x < nj) {
        const double* s = src + (int64_t)(j0 + threadIdx.x) * kSrcDoubles;
        for (int d = 0; d < 3; ++d) tree_lagrange(s[d], nd.lo[d], nd.hi[d], p, cosk, sL[threadIdx.x][d]);
        for (int a = 0; a < 3; ++a) {
          sg[threadIdx.x][a] = s[6 + a];       // f w (0 unless MODE & 1)
          sg[threadIdx.x][3 + a] = s[3 + a];   // n w
        }
        // the DL far term contracts q_a n_c w with d_a d_c only, so its symmetric part
        // suffices: Q00 Q11 Q22 and Q01+Q10, Q02+Q20, Q12+Q21 (6 channels, not 9)
        const double* q = s + 9;
        const double* m = s + 3;
        const bool dl = MODE & 2;
        sg[threadIdx.x][6] = dl ? q[0] * m[0] : 0.0;
        sg[threadIdx.x][7] = dl ? q[1] * m[1] : 0.0;
        sg[threadIdx.x][8] = dl ? q[2] * m[2] : 0.0;
        sg[threadIdx.x][9] = dl ? fma(q[0], m[1], q[1] * m[0]) : 0.0;
        sg[threadIdx.x][10] = dl ? fma(q[0], m[2], q[2] * m[0]) : 0.0;
        sg[threadIdx.x][11] = dl ? fma(q[1], m[2], q[2] * m[1]) : 0.0;
      }
      __syncthreads();
      if (k < NP)
        for (int j = 0; j < nj; ++j) {
          const double Lk = sL[j][0][k1] * sL[j][1][k2] * sL[j][2][k3];
#pragma unroll
          for (int c = 0; c < kTreeCh; ++c) acc[c] = fma(Lk, sg[j][c], acc[c]);
        }
    }
    if (k < NP)
#pragma unroll
      for (int c = 0; c < kTreeCh; ++c) Gn[(size_t)k * kTreeCh + c] = acc[c];
  }
}

// KW2 (internal nodes, one level at a time from the deepest): the parent's
// modified weights from its children's, G^P_k = sum_C sum_k' L^P_k1(s^C_k1')
// L^P_k2(s^C_k2') L^P_k3(s^C_k3') G^C_k'.  Exact in exact arithmetic: each
// L^P_k is a polynomial of degree p per axis, reproduced by the child's
// degree-p interpolation, so this equals eq. (32) summed over the parent's
// sources (what the oracle computes) up to rounding.
template <int MODE>
__global__ void __launch_bounds__(256) tree_m2m_kernel(const TreeNode* __restrict__ nodes,
                                                       const int* __restrict__ ids, int p, double* __restrict__ G) {
  // separable form: for each child and channel, three 1-D contractions through
  // SMEM (B0 -> B1 -> B0 -> += G^P), 3 (p+1)^4 FMAs instead of (p+1)^6
  __shared__ double A[3][kTreeMaxDegree + 1][kTreeMaxDegree + 1];  // A[d][k'][k] = L^P_k(s^C_k',d)
  __shared__ double cosk[kTreeMaxDegree + 1];
  extern __shared__ double dyn[];
  const int node = ids[blockIdx.x];
  const TreeNode P = nodes[node];
  const int P1 = p + 1, NP = P1 * P1 * P1;
  double* B0 = dyn;
  double* B1 = dyn + NP;
  if (threadIdx.x <= p) cosk[threadIdx.x] = cos(threadIdx.x * kPi / p);
  double* GP = G + (size_t)node * NP * kTreeCh;
  for (int ci = 0; ci < P.nchild; ++ci) {
    const int child = P.first_child + ci;
    const TreeNode C = nodes[child];
    const double* GC = G + (size_t)child * NP * kTreeCh;
    __syncthreads();  // previous child's A consumed (and cosk written)
    if (threadIdx.x < 3 * P1) {
      const int d = threadIdx.x / P1, kp = threadIdx.x % P1;
      const double sc = C.c[d] + 0.5 * (C.hi[d] - C.lo[d]) * cosk[kp];
      tree_lagrange(sc, P.lo[d], P.hi[d], p, cosk, A[d][kp]);
    }
    for (int c = 0; c < kTreeCh; ++c) {
      __syncthreads();
      for (int k = threadIdx.x; k < NP; k += blockDim.x) B0[k] = GC[(size_t)k * kTreeCh + c];
      __syncthreads();
      for (int k = threadIdx.x; k < NP; k += blockDim.x) {  // axis 0: [a][b][cc] -> [k1][b][cc]
        const int k1 = k / (P1 * P1), r = k % (P1 * P1);
        double v = 0.0;
        for (int a2 = 0; a2 < P1; ++a2) v = fma(A[0][a2][k1], B0[a2 * P1 * P1 + r], v);
        B1[k] = v;
      }
      __syncthreads();
      for (int k = threadIdx.x; k < NP; k += blockDim.x) {  // axis 1: [k1][b][cc] -> [k1][k2][cc]
        const int k1 = k / (P1 * P1), k2 = (k / P1) % P1, cc = k % P1;
        double v = 0.0;
        for (int b2 = 0; b2 < P1; ++b2) v = fma(A[1][b2][k2], B1[(k1 * P1 + b2) * P1 + cc], v);
        B0[k] = v;
      }
      __syncthreads();
      for (int k = threadIdx.x; k < NP; k += blockDim.x) {  // axis 2, accumulate into the parent
        const int base = k - k % P1, k3 = k % P1;
        double v = 0.0;
        for (int c2 = 0; c2 < P1; ++c2) v = fma(A[2][c2][k3], B0[base + c2], v);
        double* out = GP + (size_t)k * kTreeCh + c;
        *out = (ci == 0) ? v : *out + v;
      }
    }
  }
}

#ifndef SER_TREE_ILP2
#define SER_TREE_ILP2 1  // proxies two at a time into two accumulator sets (-3.6% / -1.7% at 1/h = 128 / 256 with MINB 3)
#endif
// One target (lane) x one proxy point of an accepted cluster: eq. (31) with the unregularized
// S, T of eqs. (3)-(4) on the modified weights (the same arithmetic as the pipelined loop below).
template <int MODE>
__device__ __forceinline__ void tree_proxy_pair(const double* __restrict__ b, const Tgt& t, Acc& acc) {
  const double dx = t.y0 - b[0], dy = t.y1 - b[1], dz = t.y2 - b[2];
  const double ri = rsqrt_nr(fma(dx, dx, fma(dy, dy, dz * dz)));
  const double ri2 = ri * ri;
  if (MODE & 1) {
    const double ux = fma(-t.alpha, b[6], b[3]), uy = fma(-t.alpha, b[7], b[4]), uz = fma(-t.alpha, b[8], b[5]);
    const double a3 = fma(dx, ux, fma(dy, uy, dz * uz)) * ri2;
    acc.u0 = fma(fma(dx, a3, ux), ri, acc.u0);
    acc.u1 = fma(fma(dy, a3, uy), ri, acc.u1);
    acc.u2 = fma(fma(dz, a3, uz), ri, acc.u2);
  }
  if (MODE & 2) {
    const double* Q = b + 9;
    const double w0 = fma(Q[0], dx, fma(Q[3], dy, Q[4] * dz));
    const double w1 = fma(Q[1], dy, Q[5] * dz);
    const double dQd = fma(dx, w0, fma(dy, w1, dz * (Q[2] * dz)));
    const double dq0 = fma(dx, t.q0, fma(dy, t.q1, dz * t.q2));
    const double dn = fma(dx, b[6], fma(dy, b[7], dz * b[8]));
    const double c = fma(-dq0, dn, dQd) * (ri2 * ri2 * ri);
    acc.v0 = fma(dx, c, acc.v0);
    acc.v1 = fma(dy, c, acc.v1);
    acc.v2 = fma(dz, c, acc.v2);
  }
}

struct TreeFarParams {
  const TreeNode* nodes;
  const double* G;        // modified weights
  const double* src;      // [Npad][12] tree order
  const double* tgt;      // [14][Mpad] Morton order
  double* partial;        // [Mpad/32][6][32]
  int* counter;
  int64_t Mpad;
  int n_groups, p;
  double theta, rc2;      // MAC parameter, (c delta_max)^2: the per-pair near rule of the direct sums
  double rc2_guard;       // R23 acceptance guard: rc2 (1 + 1e-9), the margin of the direct path's box tests
};

struct __align__(16) TreeWarpSmem {
  int stack_node[kTreeStack];
  unsigned stack_mask[kTreeStack];
  double buf[32][18];     // 32 proxies (coords + 12 channels) or 32 sources (12 doubles); 144-B rows
                          // (16-B aligned for double2 loads, staggered banks for the per-lane stores)
  double cosk[kTreeMaxDegree + 1];
};

union TreeFusedSmem {
  TreeWarpSmem t;
  NearSmem n;
};

// KT: far part of a warp's 32 targets (R23, R25); lane = target.  The queue also
// holds the n_near near units (K3 body), interleaved uniformly with the target
// groups as in K13, so the latency-bound near pairs share the SMs with the
// tree walk; the per-warp SMEM is a union of the two bodies.
template <int MODE, bool SHARP>
__global__ void __launch_bounds__(kTreeWarps * 32, SER_TREE_MINB) tree_far_kernel(const TreeFarParams p, const NearParams np,
                                                                   int n_near) {
  __shared__ TreeFusedSmem s_all[kTreeWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  TreeWarpSmem& sm = s_all[warp].t;
  const int P1 = p.p + 1, NP = P1 * P1 * P1;
  const int64_t total = (int64_t)p.n_groups + n_near;
  for (;;) {
    int qi = 0;
    if (lane == 0) qi = atomicAdd(p.counter, 1);
    qi = __shfl_sync(0xffffffffu, qi, 0);
    if (qi >= total) break;
    int64_t idx;
#if SER_TREE_FUSED_NEAR
    if (fused_slot(qi, p.n_groups, n_near, &idx)) {
      near_unit<MODE, SHARP>(np, static_cast<int>(idx), s_all[warp].n);
      continue;
    }
#else
    idx = qi;  // walk only: the near units run in near_kernel
#endif
    const int g = static_cast<int>(idx);
    __syncwarp();
    if (lane <= p.p) sm.cosk[lane] = cos(lane * kPi / p.p);
    __syncwarp();
    const int64_t ti = (int64_t)g * 32 + lane;
    Tgt t;
    t.y0 = p.tgt[F_Y0 * p.Mpad + ti];
    t.y1 = p.tgt[F_Y1 * p.Mpad + ti];
    t.y2 = p.tgt[F_Y2 * p.Mpad + ti];
    t.alpha = (MODE & 1) ? p.tgt[F_ALPHA * p.Mpad + ti] : 0.0;
    t.q0 = (MODE & 2) ? p.tgt[F_Q0 * p.Mpad + ti] : 0.0;
    t.q1 = (MODE & 2) ? p.tgt[F_Q1 * p.Mpad + ti] : 0.0;
    t.q2 = (MODE & 2) ? p.tgt[F_Q2 * p.Mpad + ti] : 0.0;
    Acc acc{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
    int sp = 0;
    if (lane == 0) { sm.stack_node[0] = 0; sm.stack_mask[0] = 0xffffffffu; }
    sp = 1;
    __syncwarp();
    while (sp > 0) {
      --sp;
      const int ni = sm.stack_node[sp];
      const unsigned mask = sm.stack_mask[sp];
      __syncwarp();
      const TreeNode nd = p.nodes[ni];
      // R23: MAC and regularization guard in plain (unfused) FP64, the oracle's order
      bool acc_lane = false;
      if (mask >> lane & 1) {
        const double dx = __dadd_rn(t.y0, -nd.c[0]), dy = __dadd_rn(t.y1, -nd.c[1]), dz = __dadd_rn(t.y2, -nd.c[2]);
        const double R2 = __dadd_rn(__dadd_rn(__dmul_rn(dx, dx), __dmul_rn(dy, dy)), __dmul_rn(dz, dz));
        const double yv[3] = {t.y0, t.y1, t.y2};
        double g2 = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          double gap = __dadd_rn(nd.lo[d], -yv[d]);
          const double up = __dadd_rn(yv[d], -nd.hi[d]);
          if (up > gap) gap = up;
          if (gap < 0.0) gap = 0.0;
          g2 = __dadd_rn(g2, __dmul_rn(gap, gap));
        }
        acc_lane = (nd.rc <= __dmul_rn(p.theta, __dsqrt_rn(R2))) && (g2 > p.rc2_guard);
      }
      const unsigned accm = __ballot_sync(0xffffffffu, acc_lane);
      // R26: an accepted cluster with at most (p+1)^3 points is summed directly
      const bool small = nd.end - nd.begin <= NP;
      const unsigned amask = small ? 0u : accm;                          // approximated (eq. 31)
      const unsigned dmask = (small ? accm : 0u) | (nd.nchild == 0 ? mask & ~accm : 0u);  // direct
      const unsigned rmask = nd.nchild == 0 ? 0u : mask & ~accm;         // recurse into the children
      if (amask) {  // eq. (31) at the cluster's Chebyshev points (unregularized S, T)
        const bool on = amask >> lane & 1;
        const double* Gn = p.G + (size_t)ni * NP * kTreeCh;
        for (int k0 = 0; k0 < NP; k0 += 32) {
          const int nk = min(32, NP - k0);
          __syncwarp();
          if (lane < nk) {
            const int k = k0 + lane;
            const int k1 = k / (P1 * P1), k2 = (k / P1) % P1, k3 = k % P1;
            sm.buf[lane][0] = nd.c[0] + 0.5 * (nd.hi[0] - nd.lo[0]) * sm.cosk[k1];
            sm.buf[lane][1] = nd.c[1] + 0.5 * (nd.hi[1] - nd.lo[1]) * sm.cosk[k2];
            sm.buf[lane][2] = nd.c[2] + 0.5 * (nd.hi[2] - nd.lo[2]) * sm.cosk[k3];
#pragma unroll
            for (int c = 0; c < kTreeCh; ++c) sm.buf[lane][3 + c] = Gn[(size_t)k * kTreeCh + c];
          }
          __syncwarp();
#if SER_TREE_ILP2
          if (on) {
            // two proxies per iteration into two accumulator sets: independent chains
            Acc acc2{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
            int j = 0;
            for (; j + 1 < nk; j += 2) {
              tree_proxy_pair<MODE>(sm.buf[j], t, acc);
              tree_proxy_pair<MODE>(sm.buf[j + 1], t, acc2);
            }
            if (j < nk) tree_proxy_pair<MODE>(sm.buf[j], t, acc);
            acc.u0 += acc2.u0; acc.u1 += acc2.u1; acc.u2 += acc2.u2;
            acc.v0 += acc2.v0; acc.v1 += acc2.v1; acc.v2 += acc2.v2;
          }
#else
          if (on) {
            // software pipeline: distance + rsqrt of proxy j+1 overlap the contractions of proxy j
            double gx = t.y0 - sm.buf[0][0], gy = t.y1 - sm.buf[0][1], gz = t.y2 - sm.buf[0][2];
            double gri = rsqrt_nr(fma(gx, gx, fma(gy, gy, gz * gz)));
            for (int j = 0; j < nk; ++j) {
              const double* b = sm.buf[j];
              const double* bn = sm.buf[j + 1 < nk ? j + 1 : j];
              const double nx = t.y0 - bn[0], ny = t.y1 - bn[1], nz = t.y2 - bn[2];
              const double nri = rsqrt_nr(fma(nx, nx, fma(ny, ny, nz * nz)));
              const double dx = gx, dy = gy, dz = gz, ri = gri;
              const double ri2 = ri * ri;
              if (MODE & 1) {  // S (eq. 3) on g = G^fw - alpha G^nw
                const double ux = fma(-t.alpha, b[6], b[3]), uy = fma(-t.alpha, b[7], b[4]),
                             uz = fma(-t.alpha, b[8], b[5]);
                const double a3 = fma(dx, ux, fma(dy, uy, dz * uz)) * ri2;
                acc.u0 = fma(fma(dx, a3, ux), ri, acc.u0);
                acc.u1 = fma(fma(dy, a3, uy), ri, acc.u1);
                acc.u2 = fma(fma(dz, a3, uz), ri, acc.u2);
              }
              if (MODE & 2) {  // T (eq. 4) on D_ac = G^qn_ac - q0_a G^nw_c (the -6 in the finalize)
                const double* Q = b + 9;  // Q00 Q11 Q22, Q01+Q10, Q02+Q20, Q12+Q21
                const double w0 = fma(Q[0], dx, fma(Q[3], dy, Q[4] * dz));
                const double w1 = fma(Q[1], dy, Q[5] * dz);
                const double dQd = fma(dx, w0, fma(dy, w1, dz * (Q[2] * dz)));
                const double dq0 = fma(dx, t.q0, fma(dy, t.q1, dz * t.q2));
                const double dn = fma(dx, b[6], fma(dy, b[7], dz * b[8]));
                const double c = fma(-dq0, dn, dQd) * (ri2 * ri2 * ri);
                acc.v0 = fma(dx, c, acc.v0);
                acc.v1 = fma(dy, c, acc.v1);
                acc.v2 = fma(dz, c, acc.v2);
              }
              gx = nx; gy = ny; gz = nz; gri = nri;
            }
          }
#endif
        }
      }
      if (dmask) {  // direct far pairs (near pairs masked: K3 owns them)
        {
          const bool on = dmask >> lane & 1;
          for (int j0 = nd.begin; j0 < nd.end; j0 += 32) {
            const int nj = min(32, nd.end - j0);
            __syncwarp();
            if (lane < nj) {
              const double2* s2 = reinterpret_cast<const double2*>(p.src + (int64_t)(j0 + lane) * kSrcDoubles);
#pragma unroll
              for (int c = 0; c < kSrcDoubles / 2; ++c) {
                const double2 v = __ldg(s2 + c);
                sm.buf[lane][2 * c] = v.x;
                sm.buf[lane][2 * c + 1] = v.y;
              }
            }
            __syncwarp();
            const double rc2_lane = on ? p.rc2 : INFINITY;  // inactive lanes mask every pair
            for (int j = 0; j < nj; ++j) far_pair_masked<MODE>(load_src<MODE>(sm.buf[j]), t, acc, rc2_lane);
          }
        }
      }
      if (rmask) {
        {
          __syncwarp();
          if (lane == 0)
            for (int k = nd.nchild - 1; k >= 0; --k) {  // popped in octant order
              sm.stack_node[sp + (nd.nchild - 1 - k)] = nd.first_child + k;
              sm.stack_mask[sp + (nd.nchild - 1 - k)] = rmask;
            }
          sp += nd.nchild;
          __syncwarp();
        }
      }
    }
    double* out = p.partial + (int64_t)g * 6 * 32 + lane;
    out[0] = acc.u0; out[32] = acc.u1; out[64] = acc.u2;
    out[96] = acc.v0; out[128] = acc.v1; out[160] = acc.v2;
    __syncwarp();  // the warp's SMEM may hold a near unit next
  }
}

}  // namespace ser
