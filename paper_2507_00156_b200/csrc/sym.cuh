// sym.cuh -- the node-target path (stokes_er_eval_nodes): every quadrature node
// is also a target (b = 0, x0 = the node, n0 = its normal, f(x0) = f and
// q(x0) = q at the node).  The pair sum is then symmetric in geometry: the far
// pair (i <- j) and (j <- i) share d = x_i - x_j, r^2, 1/r and its powers
// (eqs. (3)-(4): S is even in d, T odd), and for node targets even the
// stresslet's d.(q_j - q_i) is shared (q0_i = q_i).  One evaluation of the
// shared part serves both directions.
//
// Pipeline (after K0 sort/pack of the general path):
//   pack_node_soa      node records in 32-node tiles (x | m w | f w | q | alpha; 14-double
//                      AoS records by default, SoA [13][32] with SER_SYM_AOS=0) and the
//                      node-target fields
//   block_boxes        kBlk-node block boxes (union of the kSymT = 3 32-node boxes)
//   sym_kernel         K5: every unordered pair of kBlk-node (96-node) blocks (m < n) whose
//                      boxes are beyond the cutoff ("AF": all far) -- both
//                      directions of all 9216 pairs, far-field sums only
//   nbr_kernel         K6: per 32-target group, every source sub-tile of its own
//                      block or of a block that is not AF: far pairs (masked)
//                      and the near 3-delta pairs (the near unit's queue)
//   finalize_nodes     K7: sums the per-CTA accumulators (fixed order) and the
//                      K6 partials, applies 1/(8 pi), -6 and chi q0 = q/2 (b = 0; a shard other
//                      than 0 of a sharded call adds no chi term: the shards' sum has it once)
//
// Determinism: sym_kernel assigns items to CTAs statically (CTA g takes the g-th
// contiguous range of the c-major item list) and every CTA accumulates into its OWN
// slice of the workspace, in item order; finalize sums the slices in CTA order.
// No atomics on data.
#pragma once
#include "kernels.cuh"

namespace ser {

constexpr int kNodeFields = 13;  // x y z | mx my mz | fx fy fz | qx qy qz | alpha
enum NodeField { NX = 0, NY, NZ, NMX, NMY, NMZ, NFX, NFY, NFZ, NQX, NQY, NQZ, NALPHA };
#ifndef SER_SYM_AOS
#define SER_SYM_AOS 1  // node records of 14 doubles (13 + pad, 112 B) instead of SoA 32-node tiles
#endif
// AoS: lane-varying 16-byte reads of record (l + k) mod 32 are conflict-free (112 B = 28 banks:
// 8 consecutive records start on 8 distinct 4-bank groups), 7 LDS.128 per node instead of 13 LDS.64
constexpr int kNodeStride = SER_SYM_AOS ? 14 : kNodeFields;       // doubles per node in a tile
constexpr int kTileDoubles = 32 * kNodeStride;                     // one 32-node tile
__host__ __device__ constexpr int nfield(int l, int f) { return SER_SYM_AOS ? l * 14 + f : f * 32 + l; }
#ifndef SER_SYM_PIPE
#define SER_SYM_PIPE 0                                     // software-pipelined step (measured slower)
#endif
#ifndef SER_SYM_TR2
#define SER_SYM_TR2 0                                      // 2 R nodes per step (4 pairs): tuning macro
#endif
#ifndef SER_SYM_T
#define SER_SYM_T 3                                        // I nodes per lane = 32-node sub-tiles per block
                                                           // (3 at 8 warps: +2.9% over 2 at 12 warps; 4: -3%)
#endif
constexpr int kSymT = SER_SYM_T;
static_assert(kSymT >= 2 && kSymT <= 4, "I nodes per lane: 2, 3 or 4 (registers)");
static_assert(kSymT == 2 || !(SER_SYM_PIPE || SER_SYM_TR2), "the pipelined and two-R-node steps are written for T = 2");
constexpr int kBlk = 32 * kSymT;                           // nodes per symmetric block (96: 3 sub-tiles)
constexpr int kBlkTileBytes = kSymT * kTileDoubles * 8;    // one R block in SMEM (TMA unit)
#ifndef SER_SYM_WARPS
#define SER_SYM_WARPS 8
#endif
constexpr int kSymWarps = SER_SYM_WARPS;                   // I blocks per CTA (one per warp)
constexpr int kSymThreads = kSymWarps * 32;
#ifndef SER_SYM_STAGES
#define SER_SYM_STAGES 3
#endif
constexpr int kSymStages = SER_SYM_STAGES;                 // R-block TMA ring
#ifndef SER_SYM_UNROLL
#define SER_SYM_UNROLL 8                                   // steps per loop iteration (8: +0.6% over 4; 2, 1: -1%)
#endif
constexpr int kSymUnroll = SER_SYM_UNROLL;
#ifndef SER_SYM_MINB
#define SER_SYM_MINB 1                                     // resident CTAs per SM (tuning macro)
#endif
#ifndef SER_SYM_RSQ2
#define SER_SYM_RSQ2 0                                     // quadratic Newton rsqrt in sym_geo (tuning macro)
#endif
#ifndef SER_SYM_MAXK
#define SER_SYM_MAXK 3                                     // R blocks per item <= MAXK * warps (SMEM)
#endif

struct SymParams {
  const double* nsoa;     // [Npad/32][13][32]
  const double* blk_box;  // [nb][8] lo xyz, pad, hi xyz, pad
  double* pacc;           // [G][6][Npad] per-CTA accumulators (zeroed by the host)
  int64_t Npad;
  int nb;                 // kBlk-node blocks
  int nsb;                // superblocks of kSymWarps blocks
  int chunk;              // R blocks per item (a multiple of kSymWarps)
  int nchunks;
  int64_t n_items;
  int64_t item_begin, item_end;  // this call's items (a shard of [0, n_items), or all of them)
  double rc2_box;
};

// Box-level "all far" test between kBlk-node blocks, symmetric in (a, b): every
// pair has r^2 >= gap^2 > rc2 (1 + 1e-9).  The same expression decides which
// pairs sym_kernel owns and which nbr_kernel owns.
__device__ __forceinline__ bool blocks_far(const double* __restrict__ bb, int a, int b, double rc2_box) {
  const double* A = bb + (int64_t)a * 8;
  const double* B = bb + (int64_t)b * 8;
  double g2 = 0.0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double gap = fmax(0.0, fmax(__ldg(B + d) - __ldg(A + 4 + d), __ldg(A + d) - __ldg(B + 4 + d)));
    g2 = fma(gap, gap, g2);
  }
  return g2 > rc2_box;
}

// ---------------------------------------------------------------- K0 extras
// SoA node tiles + node-target fields (y = x, alpha = f.n, q0 = q, n0 = n, b = 0,
// extrapolation weights at lambda = 0) in Morton order; i >= N are padding
// copies of the last node with zero weight (they add exactly 0 as sources, and
// their target sums are dropped).
template <int MODE>
__global__ void pack_node_soa(const double* __restrict__ xyz, const double* __restrict__ nrm,
                              const double* __restrict__ wgt, const double* __restrict__ f,
                              const double* __restrict__ q, int64_t N, int64_t Npad, const int32_t* __restrict__ perm,
                              double h, Delta3 rho, bool sharp, double* __restrict__ nsoa,
                              double* __restrict__ tgt, int32_t* __restrict__ orig) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Npad) return;
  const bool pad = i >= N;
  const int64_t j = perm[pad ? N - 1 : i];
  const double w = pad ? 0.0 : wgt[j];
  double x[3], n[3], fv[3], qv[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    x[d] = xyz[d * N + j];
    n[d] = nrm[d * N + j];
    fv[d] = (MODE & 1) ? f[d * N + j] : 0.0;
    qv[d] = (MODE & 2) ? q[d * N + j] : 0.0;
  }
  const double alpha = fma(fv[0], n[0], fma(fv[1], n[1], fv[2] * n[2]));  // f(x0).n0
  double* t = nsoa + (i >> 5) * kTileDoubles;
  const int l = static_cast<int>(i & 31);
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    t[nfield(l, NX + d)] = x[d];
    t[nfield(l, NMX + d)] = n[d] * w;
    t[nfield(l, NFX + d)] = fv[d] * w;
    t[nfield(l, NQX + d)] = qv[d];
  }
  t[nfield(l, NALPHA)] = alpha;
  if (SER_SYM_AOS) t[nfield(l, 13)] = 0.0;
  double wk[3] = {1.0, 0.0, 0.0};  // NEXT-1 (s#): one delta, no extrapolation
  if (!sharp) extrap_weights(0.0, h, rho.rho, STOKES_ER_CUTOFF, wk);
  tgt[F_Y0 * Npad + i] = x[0];
  tgt[F_Y1 * Npad + i] = x[1];
  tgt[F_Y2 * Npad + i] = x[2];
  tgt[F_ALPHA * Npad + i] = alpha;
  tgt[F_Q0 * Npad + i] = qv[0];
  tgt[F_Q1 * Npad + i] = qv[1];
  tgt[F_Q2 * Npad + i] = qv[2];
  tgt[F_N0 * Npad + i] = n[0];
  tgt[F_N1 * Npad + i] = n[1];
  tgt[F_N2 * Npad + i] = n[2];
  tgt[F_B * Npad + i] = 0.0;
  tgt[F_W0 * Npad + i] = wk[0];
  tgt[F_W1 * Npad + i] = wk[1];
  tgt[F_W2 * Npad + i] = wk[2];
  orig[i] = static_cast<int32_t>(pad ? -1 : j);
}

__global__ void block_boxes(const double* __restrict__ box32, int nb, double* __restrict__ bb) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nb) return;
  const double* a = box32 + (int64_t)(kSymT * m) * 8;
  double* o = bb + (int64_t)m * 8;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double lo = a[d], hi = a[4 + d];
    for (int t = 1; t < kSymT; ++t) {
      lo = fmin(lo, a[t * 8 + d]);
      hi = fmax(hi, a[t * 8 + 4 + d]);
    }
    o[d] = lo;
    o[4 + d] = hi;
  }
  o[3] = 0.0;
  o[7] = 0.0;
}

// ---------------------------------------------------------------- K5
struct SymNode {
  double x, y, z, mx, my, mz, fx, fy, fz, qx, qy, qz, alpha;
};

template <int MODE>
__device__ __forceinline__ SymNode load_node(const double* __restrict__ t, int l) {
  SymNode n;
#if SER_SYM_AOS
  const double2* p = reinterpret_cast<const double2*>(t + l * kNodeStride);
  const double2 a = p[0], b = p[1], c = p[2];
  n.x = a.x; n.y = a.y; n.z = b.x; n.mx = b.y; n.my = c.x; n.mz = c.y;
  if (MODE & 1) {
    const double2 d = p[3], e = p[4], g = p[6];
    n.fx = d.x; n.fy = d.y; n.fz = e.x; n.alpha = g.x;
  } else {
    n.fx = n.fy = n.fz = n.alpha = 0.0;
  }
  if (MODE & 2) {
    const double2 e = p[4], f = p[5];
    n.qx = e.y; n.qy = f.x; n.qz = f.y;
  } else {
    n.qx = n.qy = n.qz = 0.0;
  }
#else
  n.x = t[NX * 32 + l]; n.y = t[NY * 32 + l]; n.z = t[NZ * 32 + l];
  n.mx = t[NMX * 32 + l]; n.my = t[NMY * 32 + l]; n.mz = t[NMZ * 32 + l];
  if (MODE & 1) {
    n.fx = t[NFX * 32 + l]; n.fy = t[NFY * 32 + l]; n.fz = t[NFZ * 32 + l];
    n.alpha = t[NALPHA * 32 + l];
  } else {
    n.fx = n.fy = n.fz = n.alpha = 0.0;
  }
  if (MODE & 2) {
    n.qx = t[NQX * 32 + l]; n.qy = t[NQY * 32 + l]; n.qz = t[NQZ * 32 + l];
  } else {
    n.qx = n.qy = n.qz = 0.0;
  }
#endif
  return n;
}

// Both directions of one far pair (node I, node R), d = x_I - x_R:
//   u_I += S(d) (f_R w_R - alpha_I m_R w_R),  u_R += S(-d) (f_I w_I - alpha_R m_I w_I)
//   v_I += T(d) (q_R - q_I) m_R w_R,           v_R += T(-d) (q_I - q_R) m_I w_I
// with S(d) g = g/r + d (d.g)/r^3 (eq. (3), even in d) and T(d) dq mw =
// d (d.dq)(d.mw)/r^5 (eq. (4) without the -6, odd in d: the two sign flips of the
// reverse direction cancel).  61 FP64 instructions for the two directed pairs (60 in the unit-vector
// form sym_acc_unit below, the default with both layers)
// (41 for one directed pair in far_pair).  Split in two halves for the software
// pipeline of sym_kernel: sym_geo (d and the MUFU + Newton 1/r, the long dependency
// chain) of step k+1 is issued before sym_acc (the contractions) of step k.
__device__ __forceinline__ Geo sym_geo(const SymNode& I, double rx, double ry, double rz) {
  Geo g;
  g.dx = I.x - rx;
  g.dy = I.y - ry;
  g.dz = I.z - rz;
#if SER_SYM_RSQ2
  // tuning variant: one quadratic Newton step from the MUFU seed (4 FP64 instructions instead of 5;
  // accurate only if the seed is; tools/probes/rsqrt_seed_probe.cu)
  const double x = fma(g.dx, g.dx, fma(g.dy, g.dy, g.dz * g.dz));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  g.ri = fma(y * 0.5, fma(-x, y * y, 1.0), y);
#else
  g.ri = rsqrt_nr(fma(g.dx, g.dx, fma(g.dy, g.dy, g.dz * g.dz)));
#endif
  return g;
}
template <int MODE>
__device__ __forceinline__ void sym_acc(const SymNode& I, const SymNode& R, const Geo& g, Acc& ai, Acc& ar) {
  const double dx = g.dx, dy = g.dy, dz = g.dz, ri = g.ri;
  const double ri2 = ri * ri;
  if (MODE & 1) {
    const double gx = fma(-I.alpha, R.mx, R.fx), gy = fma(-I.alpha, R.my, R.fy), gz = fma(-I.alpha, R.mz, R.fz);
    const double a3 = fma(dx, gx, fma(dy, gy, dz * gz)) * ri2;
    ai.u0 = fma(fma(dx, a3, gx), ri, ai.u0);
    ai.u1 = fma(fma(dy, a3, gy), ri, ai.u1);
    ai.u2 = fma(fma(dz, a3, gz), ri, ai.u2);
    const double hx = fma(-R.alpha, I.mx, I.fx), hy = fma(-R.alpha, I.my, I.fy), hz = fma(-R.alpha, I.mz, I.fz);
    const double b3 = fma(dx, hx, fma(dy, hy, dz * hz)) * ri2;
    ar.u0 = fma(fma(dx, b3, hx), ri, ar.u0);
    ar.u1 = fma(fma(dy, b3, hy), ri, ar.u1);
    ar.u2 = fma(fma(dz, b3, hz), ri, ar.u2);
  }
  if (MODE & 2) {
    const double qx = R.qx - I.qx, qy = R.qy - I.qy, qz = R.qz - I.qz;
    const double c = fma(dx, qx, fma(dy, qy, dz * qz)) * (ri2 * ri2 * ri);
    const double ci = c * fma(dx, R.mx, fma(dy, R.my, dz * R.mz));
    const double cr = c * fma(dx, I.mx, fma(dy, I.my, dz * I.mz));
    ai.v0 = fma(dx, ci, ai.v0);
    ai.v1 = fma(dy, ci, ai.v1);
    ai.v2 = fma(dz, ci, ai.v2);
    ar.v0 = fma(dx, cr, ar.v0);
    ar.v1 = fma(dy, cr, ar.v1);
    ar.v2 = fma(dz, cr, ar.v2);
  }
}
#ifndef SER_SYM_RED2
#define SER_SYM_RED2 1  // double-buffered per-R-block reduction buffer: one CTA barrier per R block (+0.2%)
#endif
constexpr int kSymRedBufs = SER_SYM_RED2 ? 2 : 1;
#ifndef SER_SYM_DHAT
#define SER_SYM_DHAT 1  // contractions on the unit vector d/r: 60 FP64 instructions instead of 61 (+1.3% at 1/h = 256)
#endif
// The same two directed pairs written on the unit vector e = d/r (3 DMUL): S(d) g = (g + e (e.g))/r and
// T(d) dq mw = e (e.dq)(e.mw)/r^2, so r^-3 and r^-5 are not formed (one FP64 instruction fewer with both
// layers; the dots then wait for 1/r).
template <int MODE>
__device__ __forceinline__ void sym_acc_unit(const SymNode& I, const SymNode& R, const Geo& g, Acc& ai, Acc& ar) {
  const double ri = g.ri, ex = g.dx * ri, ey = g.dy * ri, ez = g.dz * ri;
  if (MODE & 1) {
    const double gx = fma(-I.alpha, R.mx, R.fx), gy = fma(-I.alpha, R.my, R.fy), gz = fma(-I.alpha, R.mz, R.fz);
    const double a = fma(ex, gx, fma(ey, gy, ez * gz));
    ai.u0 = fma(fma(ex, a, gx), ri, ai.u0);
    ai.u1 = fma(fma(ey, a, gy), ri, ai.u1);
    ai.u2 = fma(fma(ez, a, gz), ri, ai.u2);
    const double hx = fma(-R.alpha, I.mx, I.fx), hy = fma(-R.alpha, I.my, I.fy), hz = fma(-R.alpha, I.mz, I.fz);
    const double b = fma(ex, hx, fma(ey, hy, ez * hz));
    ar.u0 = fma(fma(ex, b, hx), ri, ar.u0);
    ar.u1 = fma(fma(ey, b, hy), ri, ar.u1);
    ar.u2 = fma(fma(ez, b, hz), ri, ar.u2);
  }
  if (MODE & 2) {
    const double qx = R.qx - I.qx, qy = R.qy - I.qy, qz = R.qz - I.qz;
    const double c = fma(ex, qx, fma(ey, qy, ez * qz)) * (ri * ri);
    const double ci = c * fma(ex, R.mx, fma(ey, R.my, ez * R.mz));
    const double cr = c * fma(ex, I.mx, fma(ey, I.my, ez * I.mz));
    ai.v0 = fma(ex, ci, ai.v0);
    ai.v1 = fma(ey, ci, ai.v1);
    ai.v2 = fma(ez, ci, ai.v2);
    ar.v0 = fma(ex, cr, ar.v0);
    ar.v1 = fma(ey, cr, ar.v1);
    ar.v2 = fma(ez, cr, ar.v2);
  }
}
template <int MODE>
__device__ __forceinline__ void sym_pair(const SymNode& I, const SymNode& R, Acc& ai, Acc& ar) {
  if (SER_SYM_DHAT && MODE == 3)
    sym_acc_unit<MODE>(I, R, sym_geo(I, R.x, R.y, R.z), ai, ar);
  else
    sym_acc<MODE>(I, R, sym_geo(I, R.x, R.y, R.z), ai, ar);
}

__device__ __forceinline__ void shfl_acc(Acc& a, int src_lane) {
  a.u0 = __shfl_sync(0xffffffffu, a.u0, src_lane);
  a.u1 = __shfl_sync(0xffffffffu, a.u1, src_lane);
  a.u2 = __shfl_sync(0xffffffffu, a.u2, src_lane);
  a.v0 = __shfl_sync(0xffffffffu, a.v0, src_lane);
  a.v1 = __shfl_sync(0xffffffffu, a.v1, src_lane);
  a.v2 = __shfl_sync(0xffffffffu, a.v2, src_lane);
}

// item -> (chunk c, superblock s): chunk c pairs with superblocks s < (c + 1) k (k = chunk /
// kSymWarps superblocks per chunk), i.e. min(nsb, (c + 1) k) items; items are numbered c-major,
// so a CTA's contiguous range of items mostly shares one chunk and its R sums stay in SMEM.
__device__ __forceinline__ int64_t items_before(int64_t c, int k, int nsb) {
  const int64_t cs = nsb / k;  // chunks c' < cs have (c' + 1) k <= nsb superblocks
  if (c <= cs) return (int64_t)k * c * (c + 1) / 2;
  return (int64_t)k * cs * (cs + 1) / 2 + (c - cs) * nsb;
}

// Dynamic SMEM: R-block ring [kSymStages][kSymT][32][14] | red [kSymRedBufs][kSymWarps][6][kBlk] |
// chunk accumulator [6][chunk * 64].
template <int MODE>
__global__ void __launch_bounds__(kSymThreads, SER_SYM_MINB) sym_kernel(const SymParams p) {
  extern __shared__ __align__(128) unsigned char smem[];
  double* ring = reinterpret_cast<double*>(smem);
  double* red = ring + kSymStages * kSymT * kTileDoubles;
  double* cacc = red + kSymRedBufs * kSymWarps * 6 * kBlk;
  __shared__ __align__(8) uint64_t bar[kSymStages];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int G = gridDim.x;
  const int k = p.chunk / kSymWarps;
  const int cw = p.chunk * kBlk;  // accumulator columns
  if (tid == 0) {
    for (int b = 0; b < kSymStages; ++b) mbar_init(&bar[b], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t phase_bits = 0;
  double* my_acc = p.pacc + (int64_t)blockIdx.x * 6 * p.Npad;
  // this CTA's contiguous range of the c-major item list (static: deterministic sums)
  const int64_t n_mine = p.item_end - p.item_begin;
  const int64_t item_lo = p.item_begin + (int64_t)blockIdx.x * n_mine / G;
  const int64_t item_hi = p.item_begin + ((int64_t)blockIdx.x + 1) * n_mine / G;
  int cur_c = -1;
  auto flush_chunk = [&](int c) {  // the chunk's R sums into this CTA's slice
    const int r0 = c * p.chunk, nr = min(p.chunk, p.nb - r0);
    for (int x = tid; x < 6 * nr * kBlk; x += kSymThreads) {
      const int comp = x / (nr * kBlk), col = x - comp * (nr * kBlk);
      my_acc[comp * p.Npad + (int64_t)r0 * kBlk + col] += cacc[comp * cw + col];
    }
  };

  for (int64_t item = item_lo; item < item_hi; ++item) {
    // item -> (c, s): binary search on the c-major prefix counts
    int64_t lo = 0, hi = p.nchunks - 1;
    while (lo < hi) {
      const int64_t mid = (lo + hi + 1) >> 1;
      if (items_before(mid, k, p.nsb) <= item) lo = mid; else hi = mid - 1;
    }
    const int c = static_cast<int>(lo);
    const int s = static_cast<int>(item - items_before(lo, k, p.nsb));
    if (c != cur_c) {  // a new chunk: flush the previous one's R sums, start from zero
      if (cur_c >= 0) flush_chunk(cur_c);
      __syncthreads();
      for (int x = tid; x < 6 * cw; x += kSymThreads) cacc[x] = 0.0;
      cur_c = c;
    }
    const int myblk = s * kSymWarps + warp;
    const int r0 = c * p.chunk;
    const int nr = min(p.chunk, p.nb - r0);
    // this item's R blocks that can pair with some warp's I block: n > s W
    const int n_first = max(r0, s * kSymWarps + 1);
    const int first = n_first - r0;  // index of the first R block processed
    const bool has_i = myblk < p.nb;

    // I block of this warp in registers (kSymT nodes per lane)
#if SER_SYM_T == 2
    SymNode I0, I1;
    Acc a0{0, 0, 0, 0, 0, 0}, a1{0, 0, 0, 0, 0, 0};
    if (has_i) {
      const double* t = p.nsoa + (int64_t)(kSymT * myblk) * kTileDoubles;
      I0 = load_node<MODE>(t, lane);
      I1 = load_node<MODE>(t + kTileDoubles, lane);
    }
#else
    SymNode I[kSymT];
    Acc a[kSymT];
#pragma unroll
    for (int t = 0; t < kSymT; ++t) {
      a[t] = Acc{0, 0, 0, 0, 0, 0};
      if (has_i) I[t] = load_node<MODE>(p.nsoa + (int64_t)(kSymT * myblk + t) * kTileDoubles, lane);
    }
#endif
    __syncthreads();  // cacc ready; the previous item's readers of the ring are done
    if (tid == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      for (int b = 0; b < kSymStages && first + b < nr; ++b) {
        mbar_expect_tx(&bar[b], kBlkTileBytes);
        bulk_g2s(ring + b * kSymT * kTileDoubles, p.nsoa + (int64_t)(kSymT * (r0 + first + b)) * kTileDoubles,
                 kBlkTileBytes, &bar[b]);
      }
    }
    for (int ri = first; ri < nr; ++ri) {
      const int st = (ri - first) % kSymStages;
      double* const rd = red + ((ri - first) % kSymRedBufs) * (kSymWarps * 6 * kBlk);
      mbar_wait(&bar[st], (phase_bits >> st) & 1u);
      phase_bits ^= 1u << st;
      const int n = r0 + ri;
      const bool active = has_i && n > myblk && blocks_far(p.blk_box, myblk, n, p.rc2_box);
      const double* R = ring + st * kSymT * kTileDoubles;
      if (active) {
#if SER_SYM_T != 2
       {
        // kSymT I nodes per lane share each R node read and each accumulator rotation
#pragma unroll 1
        for (int hf = 0; hf < kSymT; ++hf) {
          Acc ra{0, 0, 0, 0, 0, 0};
          const double* Rt = R + hf * kTileDoubles;
#pragma unroll kSymUnroll
          for (int kk = 0; kk < 32; ++kk) {
            const SymNode rn = load_node<MODE>(Rt, (lane + kk) & 31);
#pragma unroll
            for (int t = 0; t < kSymT; ++t) sym_pair<MODE>(I[t], rn, a[t], ra);
            shfl_acc(ra, (lane + 1) & 31);
          }
          double* rw = rd + warp * 6 * kBlk + hf * 32 + lane;
          rw[0 * kBlk] = ra.u0; rw[1 * kBlk] = ra.u1; rw[2 * kBlk] = ra.u2;
          rw[3 * kBlk] = ra.v0; rw[4 * kBlk] = ra.v1; rw[5 * kBlk] = ra.v2;
        }
       }
#elif SER_SYM_PIPE
       {
        // 64 steps over the R block's two 32-node halves; step kk pairs this lane's I nodes
        // with R node (lane + kk) & 31 of half kk >> 5 (lane-varying, conflict-free SoA reads);
        // the geometry of step kk + 1 is issued before the contractions of step kk (the last
        // step recomputes step 0's and discards it)
        auto rnode = [&](int kk) { return R + (kk >> 5) * kTileDoubles + nfield((lane + kk) & 31, 0); };
        Geo g0, g1;
        {
          const double* t = rnode(0);
          g0 = sym_geo(I0, t[nfield(0, NX)], t[nfield(0, NY)], t[nfield(0, NZ)]);
          g1 = sym_geo(I1, t[nfield(0, NX)], t[nfield(0, NY)], t[nfield(0, NZ)]);
        }
        Acc ra{0, 0, 0, 0, 0, 0};
#pragma unroll 2
        for (int kk = 0; kk < 2 * 32; ++kk) {
          const double* tn = rnode((kk + 1) & 63);
          const Geo n0 = sym_geo(I0, tn[nfield(0, NX)], tn[nfield(0, NY)], tn[nfield(0, NZ)]);
          const Geo n1 = sym_geo(I1, tn[nfield(0, NX)], tn[nfield(0, NY)], tn[nfield(0, NZ)]);
          const double* t = rnode(kk);
          SymNode rn;
          rn.mx = t[nfield(0, NMX)]; rn.my = t[nfield(0, NMY)]; rn.mz = t[nfield(0, NMZ)];
          if (MODE & 1) { rn.fx = t[nfield(0, NFX)]; rn.fy = t[nfield(0, NFY)]; rn.fz = t[nfield(0, NFZ)]; rn.alpha = t[nfield(0, NALPHA)]; }
          if (MODE & 2) { rn.qx = t[nfield(0, NQX)]; rn.qy = t[nfield(0, NQY)]; rn.qz = t[nfield(0, NQZ)]; }
          sym_acc<MODE>(I0, rn, g0, a0, ra);
          sym_acc<MODE>(I1, rn, g1, a1, ra);
          shfl_acc(ra, (lane + 1) & 31);  // lane l holds node (l + kk + 1) & 31 next
          if ((kk & 31) == 31) {          // a half done: lane l holds R node (kk >> 5) * 32 + l
            double* rw = rd + warp * 6 * kBlk + (kk >> 5) * 32 + lane;
            rw[0 * kBlk] = ra.u0; rw[1 * kBlk] = ra.u1; rw[2 * kBlk] = ra.u2;
            rw[3 * kBlk] = ra.v0; rw[4 * kBlk] = ra.v1; rw[5 * kBlk] = ra.v2;
            ra = Acc{0, 0, 0, 0, 0, 0};
          }
          g0 = n0;
          g1 = n1;
        }
       }
#elif SER_SYM_TR2
       {
        // both halves at once: step kk pairs the lane's two I nodes with R node (lane + kk) & 31 of
        // EACH half (4 independent pairs per step, two rotating accumulators)
        Acc ra{0, 0, 0, 0, 0, 0}, rb{0, 0, 0, 0, 0, 0};
        const double* Rb = R + kTileDoubles;
#pragma unroll kSymUnroll
        for (int kk = 0; kk < 32; ++kk) {
          const SymNode rn = load_node<MODE>(R, (lane + kk) & 31);
          const SymNode rm = load_node<MODE>(Rb, (lane + kk) & 31);
          sym_pair<MODE>(I0, rn, a0, ra);
          sym_pair<MODE>(I1, rn, a1, ra);
          sym_pair<MODE>(I0, rm, a0, rb);
          sym_pair<MODE>(I1, rm, a1, rb);
          shfl_acc(ra, (lane + 1) & 31);
          shfl_acc(rb, (lane + 1) & 31);
        }
        double* rw = rd + warp * 6 * kBlk + lane;  // lane l holds R nodes l (ra) and 32 + l (rb)
        rw[0 * kBlk] = ra.u0; rw[1 * kBlk] = ra.u1; rw[2 * kBlk] = ra.u2;
        rw[3 * kBlk] = ra.v0; rw[4 * kBlk] = ra.v1; rw[5 * kBlk] = ra.v2;
        rw += 32;
        rw[0 * kBlk] = rb.u0; rw[1 * kBlk] = rb.u1; rw[2 * kBlk] = rb.u2;
        rw[3 * kBlk] = rb.v0; rw[4 * kBlk] = rb.v1; rw[5 * kBlk] = rb.v2;
       }
#else
       {
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          Acc ra{0, 0, 0, 0, 0, 0};
          const double* Rt = R + hf * kTileDoubles;
#pragma unroll kSymUnroll
          for (int kk = 0; kk < 32; ++kk) {
            const SymNode rn = load_node<MODE>(Rt, (lane + kk) & 31);
            sym_pair<MODE>(I0, rn, a0, ra);
            sym_pair<MODE>(I1, rn, a1, ra);
            shfl_acc(ra, (lane + 1) & 31);  // lane l holds node (l + kk + 1) & 31 next
          }
          // lane l holds R node hf * 32 + l
          double* rw = rd + warp * 6 * kBlk + hf * 32 + lane;
          rw[0 * kBlk] = ra.u0; rw[1 * kBlk] = ra.u1; rw[2 * kBlk] = ra.u2;
          rw[3 * kBlk] = ra.v0; rw[4 * kBlk] = ra.v1; rw[5 * kBlk] = ra.v2;
        }
       }
#endif
      } else {  // inactive warp: its share of this R block is zero
        double* rw = rd + warp * 6 * kBlk + lane;
#pragma unroll
        for (int c = 0; c < 6; ++c)
#pragma unroll
          for (int t = 0; t < kSymT; ++t) rw[c * kBlk + 32 * t] = 0.0;
      }
      __syncthreads();  // red complete; every warp is done reading ring[st]
      if (tid == 0 && ri + kSymStages < nr) {  // refill the stage just released
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_expect_tx(&bar[st], kBlkTileBytes);
        bulk_g2s(ring + st * kSymT * kTileDoubles, p.nsoa + (int64_t)(kSymT * (n + kSymStages)) * kTileDoubles,
                 kBlkTileBytes, &bar[st]);
      }
      for (int x = tid; x < 6 * kBlk; x += kSymThreads) {  // fixed warp order: deterministic
        const int comp = x / kBlk, col = x - comp * kBlk;
        double sum = 0.0;
#pragma unroll 4
        for (int w = 0; w < kSymWarps; ++w) sum += rd[(w * 6 + comp) * kBlk + col];
        cacc[comp * cw + ri * kBlk + col] += sum;
      }
      if (kSymRedBufs == 1) __syncthreads();  // red may be overwritten (with two buffers: the next R block's barrier)
    }
    // flush: the I sums of every warp into this CTA's slice (the chunk's R sums when the chunk changes)
    if (has_i) {
#if SER_SYM_T == 2
      const int64_t i0 = (int64_t)myblk * kBlk + lane, i1 = i0 + 32;
      double* a = my_acc;
      a[0 * p.Npad + i0] += a0.u0; a[1 * p.Npad + i0] += a0.u1; a[2 * p.Npad + i0] += a0.u2;
      a[3 * p.Npad + i0] += a0.v0; a[4 * p.Npad + i0] += a0.v1; a[5 * p.Npad + i0] += a0.v2;
      a[0 * p.Npad + i1] += a1.u0; a[1 * p.Npad + i1] += a1.u1; a[2 * p.Npad + i1] += a1.u2;
      a[3 * p.Npad + i1] += a1.v0; a[4 * p.Npad + i1] += a1.v1; a[5 * p.Npad + i1] += a1.v2;
#else
#pragma unroll
      for (int t = 0; t < kSymT; ++t) {
        const int64_t i = (int64_t)myblk * kBlk + 32 * t + lane;
        my_acc[0 * p.Npad + i] += a[t].u0; my_acc[1 * p.Npad + i] += a[t].u1; my_acc[2 * p.Npad + i] += a[t].u2;
        my_acc[3 * p.Npad + i] += a[t].v0; my_acc[4 * p.Npad + i] += a[t].v1; my_acc[5 * p.Npad + i] += a[t].v2;
      }
#endif
    }
    __syncthreads();  // I flush before any R flush (a diagonal chunk holds the same nodes)
  }
  if (cur_c >= 0) flush_chunk(cur_c);
}

// ---------------------------------------------------------------- K6
// Neighbour unit: 32 Morton-consecutive node targets (lane = target) x every
// source sub-tile of their own kBlk-node block or of a block that is not AF with
// it (blocks_far false): exactly the directed pairs sym_kernel does not own.
// Far pairs of those sub-tiles (r^2 > rc2) are summed here with the near pairs
// masked (far_pair_masked); near pairs go through the near unit's per-lane queue
// and near_pair (3 deltas, weights folded).  One unit = (group, phase), phase p
// takes every phases-th selected sub-tile.
#ifndef SER_NBR_ILP2
#define SER_NBR_ILP2 0  // masked far loop of the neighbour units into two accumulator sets (tuning macro)
#endif
struct NbrSmem {
  double src[kSrcDoubles][32];
  int q[kQCap][32];
  double tf[kNearFields][32];
};

template <int MODE, bool SHARP>
__device__ __forceinline__ void nbr_unit(const NearParams& p, const double* __restrict__ blk_box, int unit,
                                         NbrSmem& sm) {
  const int lane = threadIdx.x & 31;
  int(*q)[32] = sm.q;
  double(*tf)[32] = sm.tf;
  const int n_sub = static_cast<int>(p.Npad / kSub);
  const int64_t g = unit / p.phases;
  const int phase = unit - static_cast<int>(g) * p.phases;
  const int tblk = static_cast<int>(g / kSymT);
  const int64_t ti = g * 32 + lane;
  Tgt tg;
  tg.y0 = p.tgt[F_Y0 * p.Mpad + ti];
  tg.y1 = p.tgt[F_Y1 * p.Mpad + ti];
  tg.y2 = p.tgt[F_Y2 * p.Mpad + ti];
  tg.alpha = (MODE & 1) ? p.tgt[F_ALPHA * p.Mpad + ti] : 0.0;
  tg.q0 = (MODE & 2) ? p.tgt[F_Q0 * p.Mpad + ti] : 0.0;
  tg.q1 = (MODE & 2) ? p.tgt[F_Q1 * p.Mpad + ti] : 0.0;
  tg.q2 = (MODE & 2) ? p.tgt[F_Q2 * p.Mpad + ti] : 0.0;
  __syncwarp();
  {
    const double* tq = p.tgt + ti;
    tf[NF_ALPHA][lane] = tg.alpha;
    tf[NF_Q0][lane] = tg.q0;
    tf[NF_Q1][lane] = tg.q1;
    tf[NF_Q2][lane] = tg.q2;
    tf[NF_N0][lane] = tq[F_N0 * p.Mpad];
    tf[NF_N1][lane] = tq[F_N1 * p.Mpad];
    tf[NF_N2][lane] = tq[F_N2 * p.Mpad];
    tf[NF_B][lane] = tq[F_B * p.Mpad];
    tf[NF_W0][lane] = tq[F_W0 * p.Mpad];
    tf[NF_W1][lane] = tq[F_W1 * p.Mpad];
    tf[NF_W2][lane] = tq[F_W2 * p.Mpad];
  }
  Acc fa{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  NearAcc acc{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int head = 0, tail = 0, ordinal = 0, base = 0;
  unsigned mm = 0;
  for (;;) {
    while (mm == 0 && base < n_sub) {
      const int sb = base + lane;
      const bool sel = sb < n_sub && (sb / kSymT == tblk || !blocks_far(blk_box, tblk, sb / kSymT, p.rc2_box));
      mm = __ballot_sync(0xffffffffu, sel);
      unsigned keep = 0, m = mm;
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        if (ordinal % p.phases == phase) keep |= 1u << bit;
        ++ordinal;
      }
      mm = keep;
      base += 32;
    }
    int rounds;
    const bool last = (mm == 0);
    if (!last) {
      const int sub = base - 32 + __ffs(mm) - 1;
      mm &= mm - 1;
      {
        const double* gs = p.src + ((int64_t)sub * kSub + lane) * kSrcDoubles;
#pragma unroll
        for (int f = 0; f < kSrcDoubles; ++f) sm.src[f][lane] = __ldg(gs + f);
      }
      __syncwarp();
      unsigned smask = 0;
#if SER_NBR_ILP2
      Acc fb{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};  // odd sources: a second, independent accumulation chain
#endif
#pragma unroll 2
      for (int kk = 0; kk < 32; ++kk) {
        Src s;
        s.x = sm.src[0][kk]; s.y = sm.src[1][kk]; s.z = sm.src[2][kk];
        s.mx = sm.src[3][kk]; s.my = sm.src[4][kk]; s.mz = sm.src[5][kk];
        s.fx = sm.src[6][kk]; s.fy = sm.src[7][kk]; s.fz = sm.src[8][kk];
        s.qx = sm.src[9][kk]; s.qy = sm.src[10][kk]; s.qz = sm.src[11][kk];
        const double dx = tg.y0 - s.x, dy = tg.y1 - s.y, dz = tg.y2 - s.z;
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        smask |= (r2 <= p.rc2 ? 1u : 0u) << kk;
#if SER_NBR_ILP2
        far_pair_masked<MODE>(s, tg, (kk & 1) ? fb : fa, p.rc2);
#else
        far_pair_masked<MODE>(s, tg, fa, p.rc2);
#endif
      }
#if SER_NBR_ILP2
      fa.u0 += fb.u0; fa.u1 += fb.u1; fa.u2 += fb.u2;
      fa.v0 += fb.v0; fa.v1 += fb.v1; fa.v2 += fb.v2;
#endif
      __syncwarp();
      while (smask) {
        const int bit = __ffs(smask) - 1;
        smask &= smask - 1;
        q[tail & (kQCap - 1)][lane] = sub * kSub + bit;
        ++tail;
      }
      const int minlen = __reduce_min_sync(0xffffffffu, tail - head);
      const int maxlen = __reduce_max_sync(0xffffffffu, tail - head);
      rounds = max(minlen >= 32 ? minlen : 0, maxlen - (kQCap - 32));
    } else {
      rounds = __reduce_max_sync(0xffffffffu, tail - head);
    }
    for (int r = 0; r < rounds; ++r) {
      if (head < tail) {
        const int sidx = q[head & (kQCap - 1)][lane];
        ++head;
        const Src s = load_src_global<MODE>(p.src + (int64_t)sidx * kSrcDoubles);
        near_pair<MODE, SHARP>(s, tg.y0, tg.y1, tg.y2, tf, lane, p, acc);
      }
    }
    if (last) break;
  }
  const double v0 = fma(-tf[NF_N0][lane], acc.kn, acc.v0), v1 = fma(-tf[NF_N1][lane], acc.kn, acc.v1),
               v2 = fma(-tf[NF_N2][lane], acc.kn, acc.v2);
  __syncwarp();
  double* out = p.near_out + (int64_t)phase * 6 * p.Mpad + ti;
  out[0 * p.Mpad] = fa.u0 + acc.u0; out[1 * p.Mpad] = fa.u1 + acc.u1; out[2 * p.Mpad] = fa.u2 + acc.u2;
  out[3 * p.Mpad] = fa.v0 + v0; out[4 * p.Mpad] = fa.v1 + v1; out[5 * p.Mpad] = fa.v2 + v2;
}

template <int MODE, bool SHARP>
__global__ void __launch_bounds__(64, 6) nbr_kernel(const NearParams p, const double* __restrict__ blk_box,
                                                    int unit_base) {
  __shared__ NbrSmem s_nb[2];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    int unit = 0;
    if (lane == 0) unit = atomicAdd(p.counter, 1);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= p.n_units) break;
    nbr_unit<MODE, SHARP>(p, blk_box, unit_base + unit, s_nb[warp]);  // this call's units: [base, base + n)
  }
}

// Statistics (not on the hot path): directed pairs of real nodes owned by sym_kernel,
// 2 n_m n_n over the all-far block pairs m < n (n_m = real nodes of block m).
__global__ void sym_pair_count(const double* __restrict__ blk_box, int nb, int64_t N, double rc2_box,
                               unsigned long long* __restrict__ out) {
  const int m = blockIdx.x * blockDim.x + threadIdx.x;
  if (m >= nb) return;
  const int64_t nm = min((int64_t)kBlk, max((int64_t)0, N - (int64_t)m * kBlk));
  unsigned long long c = 0;
  for (int n = m + 1; n < nb; ++n) {
    const int64_t nn = min((int64_t)kBlk, max((int64_t)0, N - (int64_t)n * kBlk));
    if (nn > 0 && blocks_far(blk_box, m, n, rc2_box)) c += 2ull * (unsigned long long)(nm * nn);
  }
  if (c) atomicAdd(out, c);
}

// ---------------------------------------------------------------- K7
template <int MODE>
__global__ void finalize_nodes(const double* __restrict__ pacc, int G, const double* __restrict__ near_out,
                               int phases, const double* __restrict__ tgt, const int32_t* __restrict__ orig,
                               int64_t N, int64_t Npad, double chi, double* __restrict__ out_u,
                               double* __restrict__ out_v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= N) return;
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (int c = 0; c < G; ++c)  // fixed CTA order: deterministic
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if ((k < 3 && (MODE & 1)) || (k >= 3 && (MODE & 2))) s[k] += pacc[((int64_t)c * 6 + k) * Npad + i];
  for (int ph = 0; ph < phases; ++ph)
#pragma unroll
    for (int k = 0; k < 6; ++k)
      if ((k < 3 && (MODE & 1)) || (k >= 3 && (MODE & 2))) s[k] += near_out[((int64_t)ph * 6 + k) * Npad + i];
  const int64_t o = orig[i];
  const double inv8pi = 1.0 / (8.0 * kPi);
  if (MODE & 1)
    for (int k = 0; k < 3; ++k) out_u[k * N + o] = s[k] * inv8pi;                            // eq. (10)
  if (MODE & 2)
    for (int k = 0; k < 3; ++k)                                                               // eq. (11), chi = 1/2
      out_v[k * N + o] = -6.0 * s[3 + k] * inv8pi + chi * tgt[(F_Q0 + k) * Npad + i];
}

}  // namespace ser
