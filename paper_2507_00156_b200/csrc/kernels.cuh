// kernels.cuh -- sm_100a kernels of the
// localized extrapolated-regularization Stokes SL/DL evaluation
// (PAPER.md = arXiv 2507.00156; design: DESIGN.md Sec. 4-5).
//
// Pipeline of one stokes_er_eval (all on the caller's stream):
//   K0a bbox_kernel        bounding box of sources and targets (Morton frame)
//   K0b morton_kernel      30-bit Morton keys of sources and targets
//   K0c CUB radix sort     (key, index) pairs for sources, then targets
//   K0d pack_sources       AoS records x | m w | f w | q (96 B) in Morton order,
//                          padded with zero-weight copies to a whole tile, and
//                          per-32-source bounding boxes
//   K0e pack_targets       SoA records y | alpha = f(x0).n0 | q(x0) | n0 | b |
//                          extrapolation weights w_k (the 3x3 solve, eq. (17))
//   K1  pair_kernel        the O(MN) sum: persistent CTAs pull (target block,
//                          source chunk) items; source tiles are staged to SMEM
//                          by TMA bulk copies (cp.async.bulk + mbarrier, double
//                          buffered); each thread keeps T targets in registers;
//                          warp-level box tests send all-far 32-source sub-tiles
//                          to the lean far loop and mixed ones
//                          to the per-pair near/far loop (3 deltas in one pass)
//   K2  finalize_kernel    sums the chunk partials in fixed order, applies
//                          1/(8pi), -6, chi q(x0) and un-permutes
#pragma once
#include "stokes_er.h"

#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cstdint>
#include <cstring>

#include "device_math.cuh"

namespace ser {

constexpr int kThreads = 128;        // threads per pair-kernel CTA (4 warps)
constexpr int kTile = 128;           // sources per SMEM tile
constexpr int kSub = 32;             // sources per classification sub-tile
constexpr int kSrcDoubles = 12;      // packed source record: x(3) mw(3) fw(3) q(3)
constexpr int kTgtFields = 14;       // y(3) alpha q0(3) n0(3) b w(3)
constexpr int kTileBytes = kTile * kSrcDoubles * 8;
constexpr int kNominalCtas = 148 * 3;  // plan assumption
constexpr double kPartialCapBytes = 256.0 * 1024 * 1024;

enum TgtField { F_Y0 = 0, F_Y1, F_Y2, F_ALPHA, F_Q0, F_Q1, F_Q2, F_N0, F_N1, F_N2, F_B, F_W0, F_W1, F_W2 };

struct PairParams {
  const double* src;      // [Npad][12]
  const double* src_box;  // [Npad/32][8]  lo xyz, pad, hi xyz, pad
  const double* tgt;      // [14][Mpad]
  double* partial;        // [items][6][TB]
  int* counter;           // work-queue head
  int64_t Mpad;
  int n_items, n_chunks, chunk_tiles, n_tiles;
  double rc2;             // (c delta_max)^2: near iff r^2 <= rc2
  double rc2_box;         // conservative bound for sub-tile tests
  double r2_tiny;         // (1e-8 delta_1)^2: r -> 0 limits below (R3)
  double inv_delta[3];
};

struct NearParams {
  const double* src;      // [Npad][12]
  const double* src_box;  // [Npad/32][8]
  const double* tgt;      // [14][Mpad]
  double* near_out;       // [6][Mpad]
  int64_t Mpad, Npad;
  double rc2, rc2_box, r2_tiny;
  double inv_delta[3];
};

// ---------------------------------------------------------------- PTX helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      " .reg .pred P1;\n"
      "WAIT_%=:\n"
      " mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      " @!P1 bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// TMA bulk copy global -> shared (1-D, 16-byte granules), completes on `bar`.
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// ------------------------------------------------------------ K0: pack & sort
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

// One CTA: min/max over sources and targets -> box[0..2] lo, box[3..5] hi.
__global__ void bbox_kernel(const double* __restrict__ sx, int64_t N, const double* __restrict__ tx, int64_t M,
                            double* __restrict__ box) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  for (int64_t i = threadIdx.x; i < N; i += blockDim.x)
    for (int d = 0; d < 3; ++d) {
      const double v = sx[d * N + i];
      lo[d] = fmin(lo[d], v);
      hi[d] = fmax(hi[d], v);
    }
  for (int64_t i = threadIdx.x; i < M; i += blockDim.x)
    for (int d = 0; d < 3; ++d) {
      const double v = tx[d * M + i];
      lo[d] = fmin(lo[d], v);
      hi[d] = fmax(hi[d], v);
    }
  __shared__ double red[32][6];
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  const int w = threadIdx.x >> 5, l = threadIdx.x & 31;
  if (l == 0)
    for (int d = 0; d < 3; ++d) { red[w][d] = lo[d]; red[w][3 + d] = hi[d]; }
  __syncthreads();
  if (threadIdx.x < 6) {
    const int nw = blockDim.x >> 5;
    double v = red[0][threadIdx.x];
    for (int i = 1; i < nw; ++i) v = threadIdx.x < 3 ? fmin(v, red[i][threadIdx.x]) : fmax(v, red[i][threadIdx.x]);
    box[threadIdx.x] = v;
  }
}

__global__ void morton_kernel(const double* __restrict__ x, int64_t n, const double* __restrict__ box,
                              uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint32_t key = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    const double ext = fmax(box[3 + d] - box[d], 1e-300);
    double s = (x[d * n + i] - box[d]) / ext * 1023.0;
    s = fmin(fmax(s, 0.0), 1023.0);
    key |= spread10(static_cast<uint32_t>(s)) << d;
  }
  keys[i] = key;
  vals[i] = static_cast<int32_t>(i);
}

// One warp per 32-source sub-tile: gather into AoS records and its bounding box.
template <int MODE>
__global__ void pack_sources(const double* __restrict__ xyz, const double* __restrict__ nrm,
                             const double* __restrict__ wgt, const double* __restrict__ f,
                             const double* __restrict__ q, int64_t N, int64_t Npad,
                             const int32_t* __restrict__ perm, double* __restrict__ src,
                             double* __restrict__ src_box) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Npad) return;  // Npad is a multiple of 32 and blockDim: whole warps exit together
  const bool pad = i >= N;
  const int64_t j = perm[pad ? N - 1 : i];
  const double w = pad ? 0.0 : wgt[j];
  double rec[kSrcDoubles];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    rec[d] = xyz[d * N + j];
    rec[3 + d] = nrm[d * N + j] * w;                          // m w
    rec[6 + d] = (MODE & 1) ? f[d * N + j] * w : 0.0;         // f w
    rec[9 + d] = (MODE & 2) ? q[d * N + j] : 0.0;             // q
  }
  double2* out = reinterpret_cast<double2*>(src + i * kSrcDoubles);
#pragma unroll
  for (int k = 0; k < kSrcDoubles / 2; ++k) out[k] = make_double2(rec[2 * k], rec[2 * k + 1]);
  double lo[3] = {rec[0], rec[1], rec[2]}, hi[3] = {rec[0], rec[1], rec[2]};
#pragma unroll
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  if ((threadIdx.x & 31) == 0) {
    double* b = src_box + (i >> 5) * 8;
    b[0] = lo[0]; b[1] = lo[1]; b[2] = lo[2]; b[3] = 0.0;
    b[4] = hi[0]; b[5] = hi[1]; b[6] = hi[2]; b[7] = 0.0;
  }
}

struct Delta3 {
  double rho[3];
};

template <int MODE>
__global__ void pack_targets(const double* __restrict__ xyz, const double* __restrict__ tb,
                             const double* __restrict__ x0d, int64_t M, int64_t Mpad,
                             const int32_t* __restrict__ perm, double h, Delta3 rho, double* __restrict__ tgt,
                             int32_t* __restrict__ orig) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= Mpad) return;
  const int64_t j = perm[i < M ? i : M - 1];
  const double b = tb[j];
  double n0[3], f0[3], q0[3];
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    n0[d] = x0d[d * M + j];
    f0[d] = (MODE & 1) ? x0d[(3 + d) * M + j] : 0.0;
    q0[d] = (MODE & 2) ? x0d[(6 + d) * M + j] : 0.0;
  }
  double w[3];
  extrap_weights(b, h, rho.rho, STOKES_ER_CUTOFF, w);
  tgt[F_Y0 * Mpad + i] = xyz[j];
  tgt[F_Y1 * Mpad + i] = xyz[M + j];
  tgt[F_Y2 * Mpad + i] = xyz[2 * M + j];
  tgt[F_ALPHA * Mpad + i] = fma(f0[0], n0[0], fma(f0[1], n0[1], f0[2] * n0[2]));  // f(x0).n0
  tgt[F_Q0 * Mpad + i] = q0[0];
  tgt[F_Q1 * Mpad + i] = q0[1];
  tgt[F_Q2 * Mpad + i] = q0[2];
  tgt[F_N0 * Mpad + i] = n0[0];
  tgt[F_N1 * Mpad + i] = n0[1];
  tgt[F_N2 * Mpad + i] = n0[2];
  tgt[F_B * Mpad + i] = b;
  tgt[F_W0 * Mpad + i] = w[0];
  tgt[F_W1 * Mpad + i] = w[1];
  tgt[F_W2 * Mpad + i] = w[2];
  orig[i] = static_cast<int32_t>(i < M ? j : -1);
}

// ------------------------------------------------------------ K1: pair sums
struct Src {
  double x, y, z, mx, my, mz, fx, fy, fz, qx, qy, qz;
};

template <int MODE>
__device__ __forceinline__ Src load_src(const double* s) {
  const double2* p = reinterpret_cast<const double2*>(s);
  Src r;
  double2 a = p[0], b = p[1], c = p[2];
  r.x = a.x; r.y = a.y; r.z = b.x; r.mx = b.y; r.my = c.x; r.mz = c.y;
  if (MODE & 1) {
    double2 d = p[3], e = p[4];
    r.fx = d.x; r.fy = d.y; r.fz = e.x;
    if (MODE & 2) { r.qx = e.y; double2 g = p[5]; r.qy = g.x; r.qz = g.y; }
  } else {
    double2 e = p[4], g = p[5];
    r.qx = e.y; r.qy = g.x; r.qz = g.y;
  }
  return r;
}

struct Tgt {
  double y0, y1, y2, alpha, q0, q1, q2;
};
struct Acc {
  double u0, u1, u2, v0, v1, v2;
};

// Far pair: unregularized Stokeslet (eq. 3) on g = f w - alpha m w and stresslet
// (eq. 4) on dq = q - q0 contracted with m w; the -6
// and 1/(8pi) are applied once in the finalize.  41 FP64 instructions (BOTH).
template <int MODE>
__device__ __forceinline__ void far_pair(const Src& s, const Tgt& t, Acc& a) {
  const double dx = t.y0 - s.x, dy = t.y1 - s.y, dz = t.y2 - s.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double ri = rsqrt_nr(r2);
  const double ri2 = ri * ri;
  if (MODE & 1) {
    const double gx = fma(-t.alpha, s.mx, s.fx), gy = fma(-t.alpha, s.my, s.fy), gz = fma(-t.alpha, s.mz, s.fz);
    const double a3 = fma(dx, gx, fma(dy, gy, dz * gz)) * ri2;
    a.u0 = fma(fma(dx, a3, gx), ri, a.u0);
    a.u1 = fma(fma(dy, a3, gy), ri, a.u1);
    a.u2 = fma(fma(dz, a3, gz), ri, a.u2);
  }
  if (MODE & 2) {
    const double qx = s.qx - t.q0, qy = s.qy - t.q1, qz = s.qz - t.q2;
    const double dq = fma(dx, qx, fma(dy, qy, dz * qz));
    const double dm = fma(dx, s.mx, fma(dy, s.my, dz * s.mz));
    const double c = (dq * dm) * (ri2 * ri2 * ri);
    a.v0 = fma(dx, c, a.v0);
    a.v1 = fma(dy, c, a.v1);
    a.v2 = fma(dz, c, a.v2);
  }
}

// Far pair with the near pairs of a mixed sub-tile masked out: ri := 0 zeroes
// every term of far_pair (u += (g + d a3) 0, c = .. ri^5 = 0) at the cost of
// one compare and a select; the near kernel owns those pairs.
template <int MODE>
__device__ __forceinline__ void far_pair_masked(const Src& s, const Tgt& t, Acc& a, double rc2) {
  const double dx = t.y0 - s.x, dy = t.y1 - s.y, dz = t.y2 - s.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double ri = r2 > rc2 ? rsqrt_nr(r2) : 0.0;
  const double ri2 = ri * ri;
  if (MODE & 1) {
    const double gx = fma(-t.alpha, s.mx, s.fx), gy = fma(-t.alpha, s.my, s.fy), gz = fma(-t.alpha, s.mz, s.fz);
    const double a3 = fma(dx, gx, fma(dy, gy, dz * gz)) * ri2;
    a.u0 = fma(fma(dx, a3, gx), ri, a.u0);
    a.u1 = fma(fma(dy, a3, gy), ri, a.u1);
    a.u2 = fma(fma(dz, a3, gz), ri, a.u2);
  }
  if (MODE & 2) {
    const double qx = s.qx - t.q0, qy = s.qy - t.q1, qz = s.qz - t.q2;
    const double dq = fma(dx, qx, fma(dy, qy, dz * qz));
    const double dm = fma(dx, s.mx, fma(dy, s.my, dz * s.mz));
    const double c = (dq * dm) * (ri2 * ri2 * ri);
    a.v0 = fma(dx, c, a.v0);
    a.v1 = fma(dy, c, a.v1);
    a.v2 = fma(dz, c, a.v2);
  }
}

// K1: far-field pair sums (the non-local part, computed once
// and shared by the three deltas).  Persistent CTAs pull (target block,
// source chunk) items from a queue; each item's partial sums go to their own
// slot, summed in fixed order by the finalize (deterministic).
template <int MODE, int T>
__global__ void __launch_bounds__(kThreads) far_kernel(const PairParams p) {
  __shared__ __align__(128) double tile[2][kTile * kSrcDoubles];
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_item;
  constexpr int TB = kThreads * T;  // targets per block
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t parity0 = 0, parity1 = 0;

  for (;;) {
    if (tid == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int item = s_item;
    if (item >= p.n_items) break;
    const int tb = item / p.n_chunks, ch = item - tb * p.n_chunks;
    const int tile0 = ch * p.chunk_tiles;
    const int ntiles = min(p.chunk_tiles, p.n_tiles - tile0);
    const double* src_base = p.src + (int64_t)tile0 * kTile * kSrcDoubles;
    if (tid == 0) {  // prefetch the first tile of this item
      mbar_expect_tx(&bar[0], kTileBytes);
      bulk_g2s(tile[0], src_base, kTileBytes, &bar[0]);
    }

    // targets of this thread: warp-contiguous (Morton order) -> tight warp boxes
    Tgt tg[T];
    Acc acc[T];
    double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
#pragma unroll
    for (int j = 0; j < T; ++j) {
      const int64_t i = (int64_t)tb * TB + warp * 32 * T + j * 32 + lane;
      const double* q = p.tgt + i;
      tg[j].y0 = q[F_Y0 * p.Mpad];
      tg[j].y1 = q[F_Y1 * p.Mpad];
      tg[j].y2 = q[F_Y2 * p.Mpad];
      tg[j].alpha = (MODE & 1) ? q[F_ALPHA * p.Mpad] : 0.0;
      tg[j].q0 = (MODE & 2) ? q[F_Q0 * p.Mpad] : 0.0;
      tg[j].q1 = (MODE & 2) ? q[F_Q1 * p.Mpad] : 0.0;
      tg[j].q2 = (MODE & 2) ? q[F_Q2 * p.Mpad] : 0.0;
      acc[j] = Acc{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
      lo[0] = fmin(lo[0], tg[j].y0); hi[0] = fmax(hi[0], tg[j].y0);
      lo[1] = fmin(lo[1], tg[j].y1); hi[1] = fmax(hi[1], tg[j].y1);
      lo[2] = fmin(lo[2], tg[j].y2); hi[2] = fmax(hi[2], tg[j].y2);
    }
#pragma unroll
    for (int d = 0; d < 3; ++d)
      for (int o = 16; o; o >>= 1) {
        lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
        hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
      }

    for (int t = 0; t < ntiles; ++t) {
      const int buf = t & 1;
      if (tid == 0 && t + 1 < ntiles) {  // the other buffer was released by the __syncthreads below
        mbar_expect_tx(&bar[buf ^ 1], kTileBytes);
        bulk_g2s(tile[buf ^ 1], src_base + (int64_t)(t + 1) * kTile * kSrcDoubles, kTileBytes, &bar[buf ^ 1]);
      }
      if (buf == 0) { mbar_wait(&bar[0], parity0); parity0 ^= 1; }
      else { mbar_wait(&bar[1], parity1); parity1 ^= 1; }
      const double* sm = tile[buf];
      const double* boxes = p.src_box + ((int64_t)(tile0 + t) * (kTile / kSub)) * 8;
#pragma unroll 1
      for (int sub = 0; sub < kTile / kSub; ++sub) {
        const double* bx = boxes + sub * 8;
        double g2 = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double gap = fmax(0.0, fmax(__ldg(bx + d) - hi[d], lo[d] - __ldg(bx + 4 + d)));
          g2 = fma(gap, gap, g2);
        }
        const double* ss = sm + sub * kSub * kSrcDoubles;
        if (g2 > p.rc2_box) {  // warp-uniform: every pair of this sub-tile is far
#pragma unroll 2
          for (int k = 0; k < kSub; ++k) {
            const Src s = load_src<MODE>(ss + k * kSrcDoubles);
#pragma unroll
            for (int j = 0; j < T; ++j) far_pair<MODE>(s, tg[j], acc[j]);
          }
        } else {  // mixed: far pairs only, near pairs belong to the near kernel
#pragma unroll 2
          for (int k = 0; k < kSub; ++k) {
            const Src s = load_src<MODE>(ss + k * kSrcDoubles);
#pragma unroll
            for (int j = 0; j < T; ++j) far_pair_masked<MODE>(s, tg[j], acc[j], p.rc2);
          }
        }
      }
      __syncthreads();  // all reads of `buf` done before it is refilled
    }

    // partial sums of this item: [item][6][TB]
    double* out = p.partial + (int64_t)item * 6 * TB;
#pragma unroll
    for (int j = 0; j < T; ++j) {
      const int loc = warp * 32 * T + j * 32 + lane;
      if (MODE & 1) { out[0 * TB + loc] = acc[j].u0; out[1 * TB + loc] = acc[j].u1; out[2 * TB + loc] = acc[j].u2; }
      if (MODE & 2) { out[3 * TB + loc] = acc[j].v0; out[4 * TB + loc] = acc[j].v1; out[5 * TB + loc] = acc[j].v2; }
    }
  }
}

// ------------------------------------------------------------ K3: near pairs
// Target record in SMEM for the near kernel (16 doubles).
struct NearTgt {
  double y0, y1, y2, alpha, q0, q1, q2, n0, n1, n2, b, w0, w1, w2, pad0, pad1;
};

// Near pair (r <= c delta_max): the three regularized kernels folded with the
// extrapolation weights w_k:
//   S_i = sum_k w_k s_i(r/delta_k),  C = sum_k w_k (s2 - s3)(r/delta_k)
//   u = g S1/r + d (d.g) S2/r^3                                   (eq. 12)
//   v = d (d.dq)(d.mw) S3/r^5 + P C/r^3,  P = t1 contracted        (eq. 13 with
//       eq. 7 rearranged: T1 s2 + T2 s3 = -6[yyy s3/r^5 + t1 (s2-s3)/r^3])
template <int MODE>
__device__ __forceinline__ Acc near_pair(const Src& s, const NearTgt& t, const NearParams& p) {
  Acc a{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const double dx = t.y0 - s.x, dy = t.y1 - s.y, dz = t.y2 - s.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double A1, A3, A5, AP;
  if (r2 < p.r2_tiny) {  // r -> 0 limits (R3)
    const double i0 = p.inv_delta[0], i1 = p.inv_delta[1], i2 = p.inv_delta[2];
    A1 = kTwoOverSqrtPi * (t.w0 * i0 + t.w1 * i1 + t.w2 * i2);
    A3 = (2.0 / 3.0) * kTwoOverSqrtPi * (t.w0 * i0 * i0 * i0 + t.w1 * i1 * i1 * i1 + t.w2 * i2 * i2 * i2);
    A5 = (4.0 / 15.0) * kTwoOverSqrtPi *
         (t.w0 * i0 * i0 * i0 * i0 * i0 + t.w1 * i1 * i1 * i1 * i1 * i1 + t.w2 * i2 * i2 * i2 * i2 * i2);
    AP = A3;
  } else {
    const double ri = rsqrt_nr(r2);
    const double r = r2 * ri;
    double S1 = 0.0, S2 = 0.0, S3 = 0.0, C = 0.0;
    const double wk[3] = {t.w0, t.w1, t.w2};
#pragma unroll
    for (int k = 0; k < 3; ++k) {
      double s1, s2, s3, c23;
      s_factors(r * p.inv_delta[k], s1, s2, s3, c23);
      S1 = fma(wk[k], s1, S1);
      S2 = fma(wk[k], s2, S2);
      S3 = fma(wk[k], s3, S3);
      C = fma(wk[k], c23, C);
    }
    const double ri3 = ri * ri * ri;
    A1 = S1 * ri;
    A3 = S2 * ri3;
    A5 = S3 * ri3 * ri * ri;
    AP = C * ri3;
  }
  if (MODE & 1) {
    const double gx = fma(-t.alpha, s.mx, s.fx), gy = fma(-t.alpha, s.my, s.fy), gz = fma(-t.alpha, s.mz, s.fz);
    const double dg = fma(dx, gx, fma(dy, gy, dz * gz)) * A3;
    a.u0 = fma(gx, A1, dx * dg);
    a.u1 = fma(gy, A1, dy * dg);
    a.u2 = fma(gz, A1, dz * dg);
  }
  if (MODE & 2) {
    const double n0 = t.n0, n1 = t.n1, n2 = t.n2, b = t.b;
    const double qx = s.qx - t.q0, qy = s.qy - t.q1, qz = s.qz - t.q2;
    const double dq = fma(dx, qx, fma(dy, qy, dz * qz));
    const double dm = fma(dx, s.mx, fma(dy, s.my, dz * s.mz));
    const double c = dq * dm * A5;
    // xh = x - x0 = b n0 - (y - x)   (y = x0 + b n0)
    const double hx = fma(b, n0, -dx), hy = fma(b, n1, -dy), hz = fma(b, n2, -dz);
    const double an = fma(n0, qx, fma(n1, qy, n2 * qz));          // n0.dq
    const double cn = fma(n0, s.mx, fma(n1, s.my, n2 * s.mz));    // n0.mw
    const double dd = fma(hx, qx, fma(hy, qy, hz * qz));          // xh.dq
    const double e = fma(hx, s.mx, fma(hy, s.my, hz * s.mz));     // xh.mw
    const double ac = an * cn;
    const double pn = (fma(b, ac, -dd * cn) - an * e) * AP;       // n0 coefficient of t1 contraction
    const double ph = ac * AP;                                    // xh coefficient (with minus)
    a.v0 = fma(dx, c, fma(n0, pn, -hx * ph));
    a.v1 = fma(dy, c, fma(n1, pn, -hy * ph));
    a.v2 = fma(dz, c, fma(n2, pn, -hz * ph));
  }
  return a;
}

// K3: near-field pairs.  One warp owns 32 Morton-consecutive targets (lane l
// accumulates target l).  It finds the 32-source sub-tiles whose box is
// within c delta_max of its target box, tests the 32 x 32 candidate pairs,
// compacts the near ones into a target-major list (ballot transpose + warp
// prefix sum) and evaluates the list 32 pairs at a time with all lanes busy.
// Each target's results are added in list order: deterministic.
constexpr int kNearWarps = 4;
template <int MODE>
__global__ void __launch_bounds__(kNearWarps * 32) near_kernel(const NearParams p) {
  __shared__ __align__(16) NearTgt s_tgt[kNearWarps][32];
  __shared__ __align__(16) double s_src[kNearWarps][32 * kSrcDoubles];
  __shared__ __align__(16) double s_res[kNearWarps][32][6];
  __shared__ uint16_t s_list[kNearWarps][32 * 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t g = (int64_t)blockIdx.x * kNearWarps + warp;  // target group
  if (g * 32 >= p.Mpad) return;
  const int64_t ti = g * 32 + lane;
  {
    NearTgt t;
    const double* q = p.tgt + ti;
    t.y0 = q[F_Y0 * p.Mpad]; t.y1 = q[F_Y1 * p.Mpad]; t.y2 = q[F_Y2 * p.Mpad];
    t.alpha = q[F_ALPHA * p.Mpad];
    t.q0 = q[F_Q0 * p.Mpad]; t.q1 = q[F_Q1 * p.Mpad]; t.q2 = q[F_Q2 * p.Mpad];
    t.n0 = q[F_N0 * p.Mpad]; t.n1 = q[F_N1 * p.Mpad]; t.n2 = q[F_N2 * p.Mpad];
    t.b = q[F_B * p.Mpad];
    t.w0 = q[F_W0 * p.Mpad]; t.w1 = q[F_W1 * p.Mpad]; t.w2 = q[F_W2 * p.Mpad];
    t.pad0 = t.pad1 = 0.0;
    s_tgt[warp][lane] = t;
  }
  double lo[3], hi[3];
  lo[0] = hi[0] = s_tgt[warp][lane].y0;
  lo[1] = hi[1] = s_tgt[warp][lane].y1;
  lo[2] = hi[2] = s_tgt[warp][lane].y2;
#pragma unroll
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  __syncwarp();
  Acc acc{0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  const int n_sub = static_cast<int>(p.Npad / kSub);
  for (int base = 0; base < n_sub; base += 32) {
    bool mixed = false;
    const int sb = base + lane;
    if (sb < n_sub) {
      const double* bx = p.src_box + (int64_t)sb * 8;
      double g2 = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double gap = fmax(0.0, fmax(bx[d] - hi[d], lo[d] - bx[4 + d]));
        g2 = fma(gap, gap, g2);
      }
      mixed = g2 <= p.rc2_box;
    }
    unsigned mm = __ballot_sync(0xffffffffu, mixed);
    while (mm) {
      const int sub = base + __ffs(mm) - 1;
      mm &= mm - 1;
      // stage the 32 sources of this sub-tile (lane l loads source l)
      {
        const double2* gs = reinterpret_cast<const double2*>(p.src + ((int64_t)sub * kSub + lane) * kSrcDoubles);
        double2* ds = reinterpret_cast<double2*>(&s_src[warp][lane * kSrcDoubles]);
#pragma unroll
        for (int k = 0; k < kSrcDoubles / 2; ++k) ds[k] = gs[k];
      }
      __syncwarp();
      // lane l (as source l): which targets are near?
      const double sx = s_src[warp][lane * kSrcDoubles + 0], sy = s_src[warp][lane * kSrcDoubles + 1],
                   sz = s_src[warp][lane * kSrcDoubles + 2];
      unsigned tmask = 0;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const double dx = s_tgt[warp][t].y0 - sx, dy = s_tgt[warp][t].y1 - sy, dz = s_tgt[warp][t].y2 - sz;
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        tmask |= (r2 <= p.rc2 ? 1u : 0u) << t;
      }
      // transpose: lane t gets the mask of its near sources
      unsigned smask = 0;
#pragma unroll 8
      for (int t = 0; t < 32; ++t) {
        const unsigned b = __ballot_sync(0xffffffffu, (tmask >> t) & 1u);
        if (lane == t) smask = b;
      }
      const int cnt = __popc(smask);
      int pre = cnt;  // inclusive warp scan
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, pre, o);
        if (lane >= o) pre += v;
      }
      const int total = __shfl_sync(0xffffffffu, pre, 31);
      const int start = pre - cnt;
      {  // target-major pair list: (target << 5) | source
        unsigned m = smask;
        int pos = start;
        while (m) {
          const int sidx = __ffs(m) - 1;
          m &= m - 1;
          s_list[warp][pos++] = static_cast<uint16_t>((lane << 5) | sidx);
        }
      }
      __syncwarp();
      for (int rb = 0; rb < total; rb += 32) {
        const int pidx = rb + lane;
        if (pidx < total) {
          const int code = s_list[warp][pidx];
          const Src s = load_src<MODE>(&s_src[warp][(code & 31) * kSrcDoubles]);
          const Acc d = near_pair<MODE>(s, s_tgt[warp][code >> 5], p);
          s_res[warp][lane][0] = d.u0; s_res[warp][lane][1] = d.u1; s_res[warp][lane][2] = d.u2;
          s_res[warp][lane][3] = d.v0; s_res[warp][lane][4] = d.v1; s_res[warp][lane][5] = d.v2;
        }
        __syncwarp();
        // lane t adds its own entries of this round, in list order
        const int lo_i = max(start, rb), hi_i = min(start + cnt, rb + 32);
        for (int k = lo_i; k < hi_i; ++k) {
          const double* r = s_res[warp][k - rb];
          acc.u0 += r[0]; acc.u1 += r[1]; acc.u2 += r[2];
          acc.v0 += r[3]; acc.v1 += r[4]; acc.v2 += r[5];
        }
        __syncwarp();
      }
    }
  }
  double* out = p.near_out + ti;
  out[0 * p.Mpad] = acc.u0; out[1 * p.Mpad] = acc.u1; out[2 * p.Mpad] = acc.u2;
  out[3 * p.Mpad] = acc.v0; out[4 * p.Mpad] = acc.v1; out[5 * p.Mpad] = acc.v2;
}

// ------------------------------------------------------------ K2: finalize
template <int MODE>
__global__ void finalize_kernel(const double* __restrict__ partial, const double* __restrict__ near_out,
                                const double* __restrict__ tgt, const int32_t* __restrict__ orig, int64_t M,
                                int64_t Mpad, int n_chunks, int TB, double* __restrict__ out_u,
                                double* __restrict__ out_v) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const int64_t tb = i / TB, loc = i - tb * TB;
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (int ch = 0; ch < n_chunks; ++ch) {  // fixed order: deterministic
    const double* pp = partial + ((tb * n_chunks + ch) * 6) * TB + loc;
#pragma unroll
    for (int c = 0; c < 6; ++c)
      if ((c < 3 && (MODE & 1)) || (c >= 3 && (MODE & 2))) s[c] += pp[c * TB];
  }
#pragma unroll
  for (int c = 0; c < 6; ++c)
    if ((c < 3 && (MODE & 1)) || (c >= 3 && (MODE & 2))) s[c] += near_out[c * Mpad + i];
  const int64_t o = orig[i];
  const double inv8pi = 1.0 / (8.0 * kPi);
  if (MODE & 1)
    for (int c = 0; c < 3; ++c) out_u[c * M + o] = s[c] * inv8pi;                 // eq. (10)
  if (MODE & 2) {
    const double b = tgt[(int64_t)F_B * Mpad + i];
    const double chi = b < 0.0 ? 1.0 : (b > 0.0 ? 0.0 : 0.5);
    for (int c = 0; c < 3; ++c)                                                  // eq. (11), T = -6...
      out_v[c * M + o] = -6.0 * s[3 + c] * inv8pi + chi * tgt[(F_Q0 + c) * Mpad + i];
  }
}

}  // namespace ser
