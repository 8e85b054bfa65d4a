// kernels.cuh -- sm_100a kernels of the
// localized extrapolated-regularization Stokes SL/DL evaluation
// (PAPER.md = arXiv 2507.00156; design: DESIGN.md Sec. 4-5).
//
// Pipeline of one stokes_er_eval (all on the caller's stream):
//   K0a bbox_kernel        grid-wide bounding box of sources and targets (Morton frame)
//   K0b morton_kernel      30-bit Morton keys of sources and targets
//   K0c CUB radix sort     (key, index) pairs for sources, then targets
//   K0d pack_sources       AoS records x | m w | f w | q (96 B) in Morton order,
//                          padded with zero-weight copies to a whole tile, and
//                          per-32-source bounding boxes
//   K0e pack_targets       SoA records y | alpha = f(x0).n0 | q(x0) | n0 | b |
//                          extrapolation weights w_k (the 3x3 solve, eq. (17))
//   K13 fused_kernel       (default schedule) one persistent kernel whose CTAs take
//                          from one interleaved queue
//                          - far items (K1 body, far_item): a target block x a source
//                            chunk; source tiles staged to SMEM by TMA bulk copies
//                            (cp.async.bulk + mbarrier, double buffered); T targets
//                            per thread in registers; warp-level box tests send
//                            all-far 32-source sub-tiles to the lean pipelined far
//                            loop, mixed ones to the loop with the
//                            near pairs masked, and all-near ones nowhere
//                          - near units (K3 body, near_unit): 32 targets x one phase of
//                            their mixed sub-tiles; the near pairs (r <= 6 delta_max)
//                            with the three regularized kernels folded with the
//                            extrapolation weights
//   K1  far_kernel / K3 near_kernel   the same bodies as two kernels (separate schedule)
//   K2  finalize_kernel    sums the partial slots in fixed order, applies
//                          1/(8pi), -6, chi q(x0) and un-permutes
// The treecode (NEXT-3) kernels are in treecode.cuh.
#pragma once
#include "stokes_er.h"

#include <cuda_runtime.h>

#include <cub/device/device_radix_sort.cuh>
#include <cstdint>
#include <cstring>

#include "device_math.cuh"

namespace ser {

#ifndef SER_FAR_THREADS
#define SER_FAR_THREADS 64
#endif
constexpr int kThreads = SER_FAR_THREADS;  // threads per far-kernel CTA (tuning macro)
#ifndef SER_HALF_BOXES
#define SER_HALF_BOXES 1  // mixed sub-tiles re-classified by 16-source halves (tuning macro)
#endif
#ifndef SER_FAR_UNROLL
#define SER_FAR_UNROLL 2
#endif
constexpr int kFarUnroll = SER_FAR_UNROLL;  // sources per all-far loop iteration (tuning macro)
#ifndef SER_TILE
#define SER_TILE 128
#endif
constexpr int kTile = SER_TILE;      // sources per SMEM tile (tuning macro)
constexpr int kSub = 32;             // sources per classification sub-tile
constexpr int kSrcDoubles = 12;      // packed source record: x(3) mw(3) fw(3) q(3)
constexpr int kTgtFields = 14;       // y(3) alpha q0(3) n0(3) b w(3)
constexpr int kTileBytes = kTile * kSrcDoubles * 8;
constexpr int kFarSmemBytes = 2 * kTileBytes;  // far-item TMA double buffer
constexpr double kPartialCapBytes = 1024.0 * 1024 * 1024;  // far partial sums (workspace)

enum TgtField { F_Y0 = 0, F_Y1, F_Y2, F_ALPHA, F_Q0, F_Q1, F_Q2, F_N0, F_N1, F_N2, F_B, F_W0, F_W1, F_W2 };

struct PairParams {
  const double* src;      // [Npad][12]
  const double* src_box;  // [Npad/32][8]  lo xyz, pad, hi xyz, pad; then [Npad/16][8] half boxes
  const double* tgt;      // [14][Mpad]
  double* partial;        // [items][6][TB]
  int* counter;           // work-queue head
  int64_t Mpad;
  int n_items, n_chunks, chunk_tiles, n_tiles;
  double rc2;             // (c delta_max)^2: near iff r^2 <= rc2
  double rc2_box;         // conservative bound for sub-tile tests
  double rc2_inner;       // sub-tiles whose farthest pair is within this are all-near (skipped)
  double inv_delta[3];
};

struct NearParams {
  const double* src;      // [Npad][12]
  const double* src_box;  // [Npad/32][8]
  const double* tgt;      // [14][Mpad]
  double* near_out;       // [phases][6][Mpad] partial near sums
  int* counter;           // warp work-queue head
  int64_t Mpad, Npad;
  int n_units, phases;    // unit = (32-target group, phase); phase p takes every phases-th mixed sub-tile
  double rc2, rc2_box;
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

// Barrier of the kThreads far-item threads (warps 0 .. kThreads/32 - 1): named
// barrier 1, so a warp-specialized CTA's near warps never take part.
__device__ __forceinline__ void far_bar_sync() { asm volatile("bar.sync 1, %0;" ::"n"(SER_FAR_THREADS) : "memory"); }

// ------------------------------------------------------------ K0: pack & sort
__device__ __forceinline__ uint32_t spread10(uint32_t v) {
  v &= 0x3ff;
  v = (v | (v << 16)) & 0x030000FF;
  v = (v | (v << 8)) & 0x0300F00F;
  v = (v | (v << 4)) & 0x030C30C3;
  v = (v | (v << 2)) & 0x09249249;
  return v;
}

// Bounding box of sources and targets as order-preserving int64 keys:
// key(v) = bits(v) ^ ((bits(v) >> 63) & 0x7fff...) orders like the doubles, so
// a grid-wide reduction is atomicMin/atomicMax on long long.  box[0..2] = lo
// keys (pre-set to 0x7f7f.. by a memset), box[3..5] = hi keys (0x8080..).
__device__ __forceinline__ long long dkey(double v) {
  const long long b = __double_as_longlong(v);
  return b ^ ((b >> 63) & 0x7fffffffffffffffLL);
}
__device__ __forceinline__ double dkey_inv(long long k) {
  return __longlong_as_double(k ^ ((k >> 63) & 0x7fffffffffffffffLL));
}
__global__ void bbox_kernel(const double* __restrict__ sx, int64_t N, const double* __restrict__ tx, int64_t M,
                            long long* __restrict__ box) {
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < N + M; i += stride) {
    const double* x = i < N ? sx + i : tx + (i - N);
    const int64_t n = i < N ? N : M;
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      const double v = x[d * n];
      lo[d] = fmin(lo[d], v);
      hi[d] = fmax(hi[d], v);
    }
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
    if (threadIdx.x < 3) atomicMin(box + threadIdx.x, dkey(v));
    else atomicMax(box + threadIdx.x, dkey(v));
  }
}

// 30-bit Morton key of point i of x [3][n] in the box with corner blo and per-axis scale
// 1023 / extent (morton_scale): 10 bits per axis.
__device__ __forceinline__ void morton_scale(const double (&blo)[3], const double (&bhi)[3], double (&sc)[3]) {
#pragma unroll
  for (int d = 0; d < 3; ++d) sc[d] = 1023.0 / fmax(bhi[d] - blo[d], 1e-300);
}
__device__ __forceinline__ uint32_t morton_key(const double* __restrict__ x, int64_t n, int64_t i,
                                               const double (&blo)[3], const double (&sc)[3]) {
  uint32_t key = 0;
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    double s = (x[d * n + i] - blo[d]) * sc[d];
    s = s > 0.0 ? s : 0.0;  // plain selects: no NaN-propagation sequence per bound
    s = s < 1023.0 ? s : 1023.0;
    key |= spread10(static_cast<uint32_t>(s)) << d;
  }
  return key;
}

__global__ void morton_kernel(const double* __restrict__ x, int64_t n, const long long* __restrict__ box,
                              uint32_t* __restrict__ keys, int32_t* __restrict__ vals) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= n) return;
  const double blo[3] = {dkey_inv(box[0]), dkey_inv(box[1]), dkey_inv(box[2])};
  const double bhi[3] = {dkey_inv(box[3]), dkey_inv(box[4]), dkey_inv(box[5])};
  double sc[3];
  morton_scale(blo, bhi, sc);
  keys[i] = morton_key(x, n, i, blo, sc);
  vals[i] = static_cast<int32_t>(i);
}

// Small problems (N, M <= kSmallSort): the Morton order by counting, in ONE launch of many CTAs
// (instead of bbox + 2 morton + the CUB device sorts, ~15 launches). The position of point i in
// the stable sort by key -- the order the large path's CUB sorts produce from the same keys -- is
//   rank(i) = #{j < i : key_j <= key_i} + #{j > i : key_j < key_i}.
// CTA c takes 32 points (lane = point) of the sources (c < ceil(N/32)) or of the targets; it
// recomputes the common bounding box (exact min/max: the same frame as bbox_kernel) and every key
// of that array into shared memory; its 16 warps count over 16 slices of j, four keys per 16-B
// broadcast read: slices below the CTA's points use <=, slices above use <, and the few keys among
// the CTA's own points take the exact (key, index) comparison. The slice counts are added in a
// fixed order and perm[rank(i)] = i is written: integer counts, so the permutation is exact and
// deterministic.
constexpr int64_t kSmallSort = 8192;
constexpr int kRankThreads = 512, kRankWarps = kRankThreads / 32, kRankPts = 32;
__global__ void __launch_bounds__(kRankThreads) small_rank_kernel(const double* __restrict__ sx, int64_t N,
                                                                 const double* __restrict__ tx, int64_t M,
                                                                 int32_t* __restrict__ svout,
                                                                 int32_t* __restrict__ tvout,
                                                                 int* __restrict__ counters) {
  __shared__ __align__(16) uint32_t skey[kSmallSort];
  __shared__ double red[kRankWarps][6];
  __shared__ double sbox[6];
  __shared__ int cnt[kRankWarps][kRankPts];
  if (blockIdx.x == 0 && threadIdx.x < 2) counters[threadIdx.x] = 0;  // the pair kernel's queues (no memset)
  const int tid = threadIdx.x, lane = tid & 31, w = tid >> 5;
  double lo[3] = {1e300, 1e300, 1e300}, hi[3] = {-1e300, -1e300, -1e300};
#pragma unroll 4
  for (int64_t i = tid; i < N + M; i += kRankThreads) {  // independent loads in flight (latency-bound)
    const double* x = i < N ? sx + i : tx + (i - N);
    const int64_t n = i < N ? N : M;
#pragma unroll
    for (int d = 0; d < 3; ++d) {  // min/max: exact and order-free (plain selects)
      const double v = x[d * n];
      lo[d] = v < lo[d] ? v : lo[d];
      hi[d] = v > hi[d] ? v : hi[d];
    }
  }
#pragma unroll
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      const double a = __shfl_xor_sync(0xffffffffu, lo[d], o), b = __shfl_xor_sync(0xffffffffu, hi[d], o);
      lo[d] = a < lo[d] ? a : lo[d];
      hi[d] = b > hi[d] ? b : hi[d];
    }
  if (lane == 0)
    for (int d = 0; d < 3; ++d) { red[w][d] = lo[d]; red[w][3 + d] = hi[d]; }
  __syncthreads();
  if (tid < 6) {  // one thread per box field reduces the warps' results
    double v = red[0][tid];
    for (int k = 1; k < kRankWarps; ++k)
      v = tid < 3 ? (red[k][tid] < v ? red[k][tid] : v) : (red[k][tid] > v ? red[k][tid] : v);
    sbox[tid] = v;
  }
  __syncthreads();
  const double blo[3] = {sbox[0], sbox[1], sbox[2]}, bhi[3] = {sbox[3], sbox[4], sbox[5]};
  double sc[3];
  morton_scale(blo, bhi, sc);
  const int64_t cs = (N + kRankPts - 1) / kRankPts;
  const bool is_src = blockIdx.x < cs;
  const double* x = is_src ? sx : tx;
  const int n = static_cast<int>(is_src ? N : M);
  int32_t* out = is_src ? svout : tvout;
  const int base = static_cast<int>((is_src ? blockIdx.x : blockIdx.x - cs) * kRankPts);
  const int nq = (n + 3) >> 2;  // keys padded to whole quads with 0xffffffff (never counted)
#pragma unroll 4
  for (int j = tid; j < 4 * nq; j += kRankThreads) skey[j] = j < n ? morton_key(x, n, j, blo, sc) : 0xffffffffu;
  __syncthreads();
  const int i = base + lane;
  const uint32_t ki = i < n ? skey[i] : 0u;
  const uint4* k4 = reinterpret_cast<const uint4*>(skey);
  const int q0 = w * nq / kRankWarps, q1 = (w + 1) * nq / kRankWarps;
  const int qa = base >> 2, qb = (base + kRankPts) >> 2;  // quads [qa, qb) hold the CTA's own points
  int c = 0;
#pragma unroll 4
  for (int q = q0; q < min(q1, qa); ++q) {  // every j < every i of the CTA: key_j <= key_i counts
    const uint4 k = k4[q];
    c += (k.x <= ki) + (k.y <= ki) + (k.z <= ki) + (k.w <= ki);
  }
  for (int q = max(q0, qa); q < min(q1, qb); ++q) {  // among the CTA's points: the exact comparison
    const uint4 k = k4[q];
    const uint32_t kk[4] = {k.x, k.y, k.z, k.w};
#pragma unroll
    for (int t = 0; t < 4; ++t) c += (kk[t] < ki || (kk[t] == ki && 4 * q + t < i)) ? 1 : 0;
  }
#pragma unroll 4
  for (int q = max(q0, qb); q < q1; ++q) {  // every j > every i: key_j < key_i counts
    const uint4 k = k4[q];
    c += (k.x < ki) + (k.y < ki) + (k.z < ki) + (k.w < ki);
  }
  cnt[w][lane] = c;
  __syncthreads();
  if (w == 0 && i < n) {
    int r = 0;
#pragma unroll
    for (int k = 0; k < kRankWarps; ++k) r += cnt[k][lane];
    out[r] = i;
  }
}

// One warp per 32-source sub-tile: gather into AoS records and its bounding box.
template <int MODE>
__device__ __forceinline__ void pack_source_at(int64_t i, const double* __restrict__ xyz,
                                               const double* __restrict__ nrm, const double* __restrict__ wgt,
                                               const double* __restrict__ f, const double* __restrict__ q,
                                               int64_t N, int64_t Npad, const int32_t* __restrict__ perm,
                                               double* __restrict__ src, double* __restrict__ src_box) {
  if (i >= Npad) return;  // Npad is a multiple of 32 and of the block size: whole warps exit together
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
    for (int o = 8; o; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  if ((threadIdx.x & 15) == 0) {  // the 16-source half box (after the Npad/32 full boxes)
    double* b = src_box + (Npad >> 5) * 8 + (i >> 4) * 8;
    b[0] = lo[0]; b[1] = lo[1]; b[2] = lo[2]; b[3] = 0.0;
    b[4] = hi[0]; b[5] = hi[1]; b[6] = hi[2]; b[7] = 0.0;
  }
#pragma unroll
  for (int d = 0; d < 3; ++d) {
    lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], 16));
    hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], 16));
  }
  if ((threadIdx.x & 31) == 0) {
    double* b = src_box + (i >> 5) * 8;
    b[0] = lo[0]; b[1] = lo[1]; b[2] = lo[2]; b[3] = 0.0;
    b[4] = hi[0]; b[5] = hi[1]; b[6] = hi[2]; b[7] = 0.0;
  }
}

template <int MODE>
__global__ void pack_sources(const double* __restrict__ xyz, const double* __restrict__ nrm,
                             const double* __restrict__ wgt, const double* __restrict__ f,
                             const double* __restrict__ q, int64_t N, int64_t Npad,
                             const int32_t* __restrict__ perm, double* __restrict__ src,
                             double* __restrict__ src_box) {
  pack_source_at<MODE>(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, xyz, nrm, wgt, f, q, N, Npad, perm, src,
                       src_box);
}

struct Delta3 {
  double rho[3];
};

template <int MODE>
__device__ __forceinline__ void pack_target_at(int64_t i, const double* __restrict__ xyz,
                                               const double* __restrict__ tb, const double* __restrict__ x0d,
                                               int64_t M, int64_t Mpad, const int32_t* __restrict__ perm, double h,
                                               const Delta3& rho, bool sharp, double* __restrict__ tgt,
                                               int32_t* __restrict__ orig) {
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
  double w[3] = {1.0, 0.0, 0.0};  // NEXT-1: a single delta, no extrapolation
  if (!sharp) extrap_weights(b, h, rho.rho, STOKES_ER_CUTOFF, w);
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

template <int MODE>
__global__ void pack_targets(const double* __restrict__ xyz, const double* __restrict__ tb,
                             const double* __restrict__ x0d, int64_t M, int64_t Mpad,
                             const int32_t* __restrict__ perm, double h, Delta3 rho, bool sharp,
                             double* __restrict__ tgt, int32_t* __restrict__ orig) {
  pack_target_at<MODE>(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, xyz, tb, x0d, M, Mpad, perm, h, rho, sharp,
                       tgt, orig);
}

// Small problems: both packs in one launch (128-thread blocks: the first Npad/128 pack sources).
template <int MODE>
__global__ void pack_both(const double* __restrict__ sxyz, const double* __restrict__ nrm,
                          const double* __restrict__ wgt, const double* __restrict__ f, const double* __restrict__ q,
                          int64_t N, int64_t Npad, const int32_t* __restrict__ sperm, double* __restrict__ src,
                          double* __restrict__ src_box, const double* __restrict__ txyz, const double* __restrict__ tb,
                          const double* __restrict__ x0d, int64_t M, int64_t Mpad, const int32_t* __restrict__ tperm,
                          double h, Delta3 rho, bool sharp, double* __restrict__ tgt, int32_t* __restrict__ orig) {
  const int64_t sblocks = Npad / blockDim.x;
  if (blockIdx.x < sblocks)
    pack_source_at<MODE>(blockIdx.x * (int64_t)blockDim.x + threadIdx.x, sxyz, nrm, wgt, f, q, N, Npad, sperm, src,
                         src_box);
  else
    pack_target_at<MODE>((blockIdx.x - sblocks) * (int64_t)blockDim.x + threadIdx.x, txyz, tb, x0d, M, Mpad, tperm,
                         h, rho, sharp, tgt, orig);
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
// The all-far loop runs it split in two halves (far_geo / far_acc below); the
// mixed sub-tiles run far_pair_masked.
// far_pair split in two halves for software pipelining (K1's all-far loop):
// far_geo (d, r^2 and the MUFU + Newton rsqrt: the long dependency chain) of
// source k+1 is issued before far_acc (the SL/DL contractions) of source k.
struct Geo {
  double dx, dy, dz, ri;
};
__device__ __forceinline__ Geo far_geo(const Src& s, const Tgt& t) {
  Geo g;
  g.dx = t.y0 - s.x;
  g.dy = t.y1 - s.y;
  g.dz = t.y2 - s.z;
  g.ri = rsqrt_nr(fma(g.dx, g.dx, fma(g.dy, g.dy, g.dz * g.dz)));
  return g;
}
template <int MODE>
__device__ __forceinline__ void far_acc(const Src& s, const Tgt& t, const Geo& g, Acc& a) {
  const double dx = g.dx, dy = g.dy, dz = g.dz, ri = g.ri;
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

// The all-far loop over NS sources at ss (software pipeline: geometry + rsqrt of
// source k+1 overlap the contractions of source k; the last step recomputes
// source 0 and discards it).
template <int MODE, int T, int NS>
__device__ __forceinline__ void far_run(const double* ss, const Tgt (&tg)[T], Acc (&acc)[T]) {
  Src s = load_src<MODE>(ss);
  Geo g[T];
#pragma unroll
  for (int j = 0; j < T; ++j) g[j] = far_geo(s, tg[j]);
#pragma unroll kFarUnroll
  for (int k = 0; k < NS; ++k) {
    const Src sn = load_src<MODE>(ss + ((k + 1) & (NS - 1)) * kSrcDoubles);
    Geo gn[T];
#pragma unroll
    for (int j = 0; j < T; ++j) gn[j] = far_geo(sn, tg[j]);
#pragma unroll
    for (int j = 0; j < T; ++j) far_acc<MODE>(s, tg[j], g[j], acc[j]);
    s = sn;
#pragma unroll
    for (int j = 0; j < T; ++j) g[j] = gn[j];
  }
}
// The mixed loop: far pairs only (near pairs masked, the near kernel owns them).
template <int MODE, int T, int NS>
__device__ __forceinline__ void far_run_masked(const double* ss, const Tgt (&tg)[T], Acc (&acc)[T], double rc2) {
#pragma unroll 2
  for (int k = 0; k < NS; ++k) {
    const Src s = load_src<MODE>(ss + k * kSrcDoubles);
#pragma unroll
    for (int j = 0; j < T; ++j) far_pair_masked<MODE>(s, tg[j], acc[j], rc2);
  }
}

// K1 body: one far work item = (target block of kThreads*T targets, source
// chunk) -- the far-field pair sums (the non-local part,
// computed once and shared by the three deltas).  Each item's partial sums go
// to their own slot, summed in fixed order by the finalize (deterministic).
// Source tiles are TMA bulk copies into the double buffer `tile` (completion on
// bar[0..1]; parities carried across items by the caller).
template <int MODE, int T>
__device__ __forceinline__ void far_item(const PairParams& p, int item, double (*tile)[kTile * kSrcDoubles],
                                         uint64_t* bar, uint32_t& parity0, uint32_t& parity1) {
  constexpr int TB = kThreads * T;  // targets per block
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int tb = item / p.n_chunks, ch = item - tb * p.n_chunks;
  const int tile0 = ch * p.chunk_tiles;
  const int ntiles = min(p.chunk_tiles, p.n_tiles - tile0);
  const double* src_base = p.src + (int64_t)tile0 * kTile * kSrcDoubles;
  if (tid == 0) {  // prefetch the first tile of this item
    // order the CTA's earlier generic-proxy SMEM accesses (the fused kernel's
    // near units alias this buffer; the caller's far-group barrier precedes) before
    // the async-proxy (TMA) writes
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
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
    if (tid == 0 && t + 1 < ntiles) {  // the other buffer was released by the far_bar_sync below
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
      double g2 = 0.0, f2 = 0.0;
#pragma unroll
      for (int d = 0; d < 3; ++d) {
        const double blo = __ldg(bx + d), bhi = __ldg(bx + 4 + d);
        const double gap = fmax(0.0, fmax(blo - hi[d], lo[d] - bhi));
        const double span = fmax(bhi - lo[d], hi[d] - blo);  // largest coordinate distance
        g2 = fma(gap, gap, g2);
        f2 = fma(span, span, f2);
      }
      const double* ss = sm + sub * kSub * kSrcDoubles;
      if (g2 > p.rc2_box) {  // warp-uniform: every pair of this sub-tile is far
        far_run<MODE, T, kSub>(ss, tg, acc);
      } else if (f2 > p.rc2_inner) {  // mixed: far pairs only, near pairs belong to the near kernel
#if SER_HALF_BOXES
        // the two 16-source halves are classified again: all-far halves take the
        // lean loop, all-near ones are skipped, only mixed halves mask pairs
        const double* hb = p.src_box + (p.n_tiles * (int64_t)kTile / kSub) * 8 +
                           ((int64_t)(tile0 + t) * (kTile / 16) + sub * 2) * 8;
#pragma unroll 1
        for (int hf = 0; hf < 2; ++hf) {
          double h2 = 0.0, s2 = 0.0;
#pragma unroll
          for (int d = 0; d < 3; ++d) {
            const double blo = __ldg(hb + hf * 8 + d), bhi = __ldg(hb + hf * 8 + 4 + d);
            const double gap = fmax(0.0, fmax(blo - hi[d], lo[d] - bhi));
            const double span = fmax(bhi - lo[d], hi[d] - blo);
            h2 = fma(gap, gap, h2);
            s2 = fma(span, span, s2);
          }
          const double* hs = ss + hf * 16 * kSrcDoubles;
          if (h2 > p.rc2_box) far_run<MODE, T, 16>(hs, tg, acc);
          else if (s2 > p.rc2_inner) far_run_masked<MODE, T, 16>(hs, tg, acc, p.rc2);
        }
#else
        far_run_masked<MODE, T, kSub>(ss, tg, acc, p.rc2);
#endif
      }  // else: every pair of the sub-tile is near (r^2 <= rc2): nothing far to add
    }
    far_bar_sync();  // all reads of `buf` done before it is refilled
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

// K1 (separate schedule): persistent CTAs pull far items from a queue.
template <int MODE, int T>
#ifndef SER_FAR_MINB
#define SER_FAR_MINB (512 / SER_FAR_THREADS)
#endif
__global__ void __launch_bounds__(kThreads, SER_FAR_MINB) far_kernel(const PairParams p) {
  extern __shared__ __align__(128) unsigned char far_smem[];  // kFarSmemBytes (dynamic)
  auto* tile = reinterpret_cast<double(*)[kTile * kSrcDoubles]>(far_smem);
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_item;
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t parity0 = 0, parity1 = 0;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int item = s_item;
    __syncthreads();  // every thread has read s_item before thread 0 may overwrite it
    if (item >= p.n_items) break;
    far_item<MODE, T>(p, item, tile, bar, parity0, parity1);
  }
}

// ------------------------------------------------------------ K3: near pairs

// Near pair (r <= c delta_max): the three regularized kernels folded with the
// extrapolation weights w_k:
//   A1 = sum_k w_k s1(r/d_k)/r, A3 = sum_k w_k s2/r^3, A5 = sum_k w_k s3/r^5,
//   AP = sum_k w_k (s2 - s3)/r^3
//   u = g A1 + d (d.g) A3                                         (eq. 12)
//   v = d (d.dq)(d.mw) A5 + P AP,  P = t1 contracted               (eq. 13 with
//       eq. 7 rearranged: T1 s2 + T2 s3 = -6[yyy s3/r^5 + t1 (s2-s3)/r^3])
// Target fields other than y live in SMEM, SoA [field][lane] (conflict-free).
enum NearField { NF_ALPHA = 0, NF_Q0, NF_Q1, NF_Q2, NF_N0, NF_N1, NF_N2, NF_B, NF_W0, NF_W1, NF_W2, kNearFields };
// The near accumulators of one target: u, the d-part of v, and kn, the sum of
// the n0 coefficients (n0 is the target's, so sum_pairs n0 kn = n0 sum kn:
// v = (v0, v1, v2) - n0 kn at the end).  Each pair adds with fused FMAs.
struct NearAcc {
  double u0, u1, u2, v0, v1, v2, kn;
};
template <int MODE, bool SHARP>
__device__ __forceinline__ void near_pair(const Src& s, double y0, double y1, double y2,
                                          const double (*__restrict__ tf)[32], int lane, const NearParams& p,
                                          NearAcc& a) {
  const double dx = y0 - s.x, dy = y1 - s.y, dz = y2 - s.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  const double ri = r2 > 0.0 ? rsqrt_nr(r2) : 0.0;
  const double r = r2 * ri;  // 0 for a coincident node
  if (SHARP) {  // NEXT-1: one delta, s# factors, unsplit stresslet (R16)
    double A1, A3, A5;
    sharp_weights(r, ri, p.inv_delta[0], A1, A3, A5);
    if (MODE & 1) {
      const double alpha = tf[NF_ALPHA][lane];
      const double gx = fma(-alpha, s.mx, s.fx), gy = fma(-alpha, s.my, s.fy), gz = fma(-alpha, s.mz, s.fz);
      const double dg = fma(dx, gx, fma(dy, gy, dz * gz)) * A3;
      a.u0 = fma(gx, A1, fma(dx, dg, a.u0));
      a.u1 = fma(gy, A1, fma(dy, dg, a.u1));
      a.u2 = fma(gz, A1, fma(dz, dg, a.u2));
    }
    if (MODE & 2) {
      const double qx = s.qx - tf[NF_Q0][lane], qy = s.qy - tf[NF_Q1][lane], qz = s.qz - tf[NF_Q2][lane];
      const double c = fma(dx, qx, fma(dy, qy, dz * qz)) * fma(dx, s.mx, fma(dy, s.my, dz * s.mz)) * A5;
      a.v0 = fma(dx, c, a.v0);
      a.v1 = fma(dy, c, a.v1);
      a.v2 = fma(dz, c, a.v2);
    }
    return;
  }
  // all three deltas through the branch-free table path (independent chains)
  const double t0 = r * p.inv_delta[0], t1 = r * p.inv_delta[1], t2 = r * p.inv_delta[2];
  double e0, e1, e2, P0, P1, P2, u0, u1, u2;
  sfactor_eP(t0, e0, P0, u0);
  sfactor_eP(t1, e1, P1, u1);
  sfactor_eP(t2, e2, P2, u2);
  const double tw0 = tf[NF_W0][lane], tw1 = tf[NF_W1][lane], tw2 = tf[NF_W2][lane];
  const double w0 = t0 >= 0.5 ? tw0 : 0.0, w1 = t1 >= 0.5 ? tw1 : 0.0, w2 = t2 >= 0.5 ? tw2 : 0.0;
  // the weighted sums over k of w_k s_i(t_k) (eqs. (14)-(16)) with a_k = w_k e_k, b_k = a_k t_k:
  //   S1 = sum w_k erf t_k = W - sum a_k P_k,  S2 = sum w_k s2 = S1 - (2/sqrt pi) sum b_k,
  //   C = sum w_k (s2 - s3) = (2/sqrt pi)(2/3) sum b_k t_k^2,  W = sum w_k
  const double a0 = w0 * e0, a1 = w1 * e1, a2 = w2 * e2;
  const double S1 = fma(-a2, P2, fma(-a1, P1, fma(-a0, P0, (w0 + w1) + w2)));
  const double b0 = a0 * t0, b1 = a1 * t1, b2 = a2 * t2;
  const double S2 = fma(-kTwoOverSqrtPi, (b0 + b1) + b2, S1);
  const double C = ((2.0 / 3.0) * kTwoOverSqrtPi) * fma(b2, u2, fma(b1, u1, b0 * u0));
  const double S3 = S2 - C;
  const double ri3 = ri * ri * ri;
  double A1 = S1 * ri, A3 = S2 * ri3, A5 = S3 * (ri3 * ri * ri), AP = C * ri3;
  if (t2 < 0.5) {  // rare: r < delta_3 / 2 (t2 is the smallest t)
    if (t0 < 0.5) sfactor_series_add(t0, p.inv_delta[0], tw0, A1, A3, A5, AP);
    if (t1 < 0.5) sfactor_series_add(t1, p.inv_delta[1], tw1, A1, A3, A5, AP);
    sfactor_series_add(t2, p.inv_delta[2], tw2, A1, A3, A5, AP);
  }
  if (MODE & 1) {
    const double alpha = tf[NF_ALPHA][lane];
    const double gx = fma(-alpha, s.mx, s.fx), gy = fma(-alpha, s.my, s.fy), gz = fma(-alpha, s.mz, s.fz);
    const double dg = fma(dx, gx, fma(dy, gy, dz * gz)) * A3;
    a.u0 = fma(gx, A1, fma(dx, dg, a.u0));
    a.u1 = fma(gy, A1, fma(dy, dg, a.u1));
    a.u2 = fma(gz, A1, fma(dz, dg, a.u2));
  }
  if (MODE & 2) {
    const double n0 = tf[NF_N0][lane], n1 = tf[NF_N1][lane], n2 = tf[NF_N2][lane], b = tf[NF_B][lane];
    const double qx = s.qx - tf[NF_Q0][lane], qy = s.qy - tf[NF_Q1][lane], qz = s.qz - tf[NF_Q2][lane];
    const double dq = fma(dx, qx, fma(dy, qy, dz * qz));
    const double dm = fma(dx, s.mx, fma(dy, s.my, dz * s.mz));
    // t1 contracted with dq and mw (eq. (8)) is
    //   P = n0 (b a c' - (xh.dq) c' - a (xh.mw)) - xh (a c'),   a = n0.dq, c' = n0.mw,
    // and with xh = x - x0 = b n0 - (y - x) (y = x0 + b n0) it needs no xh:
    //   P = (y - x) a c' - n0 (2 b a c' - (d.dq) c' - a (d.mw)),
    // so v = d ((d.dq)(d.mw) A5 + a c' AP) - n0 (2 b a c' - (d.dq) c' - a (d.mw)) AP; the n0 term is
    // summed as a scalar (NearAcc::kn) and applied once per target.
    const double an = fma(n0, qx, fma(n1, qy, n2 * qz));          // n0.dq
    const double cn = fma(n0, s.mx, fma(n1, s.my, n2 * s.mz));    // n0.mw
    const double ac = an * cn;
    const double cd = fma(dq * dm, A5, ac * AP);                    // coefficient of d = y - x
    a.kn = fma(fma(-an, dm, fma(-dq, cn, (2.0 * b) * ac)), AP, a.kn);  // minus the coefficient of n0
    a.v0 = fma(dx, cd, a.v0);
    a.v1 = fma(dy, cd, a.v1);
    a.v2 = fma(dz, cd, a.v2);
  }
}

template <int MODE>
__device__ __forceinline__ Src load_src_global(const double* __restrict__ g) {
  const double2* q = reinterpret_cast<const double2*>(g);
  Src r;
  double2 a = __ldg(q), b = __ldg(q + 1), c = __ldg(q + 2);
  r.x = a.x; r.y = a.y; r.z = b.x; r.mx = b.y; r.my = c.x; r.mz = c.y;
  double2 d = (MODE & 1) ? __ldg(q + 3) : make_double2(0.0, 0.0);
  double2 e = __ldg(q + 4), f = (MODE & 2) ? __ldg(q + 5) : make_double2(0.0, 0.0);
  r.fx = d.x; r.fy = d.y; r.fz = e.x;
  r.qx = e.y; r.qy = f.x; r.qz = f.y;
  return r;
}

// K3: near-field pairs.  One warp owns 32 Morton-consecutive targets; lane l
// owns target l and accumulates it in registers.  The warp walks the 32-source
// sub-tiles whose box lies within c delta_max of its target box; for each,
// every lane tests the 32 sources against its target (the same FP64 r^2 as
// K1's mask, so every pair is counted by exactly one kernel) and appends its
// near sources to a per-lane ring queue in SMEM.  Whenever every lane holds
// work, all lanes evaluate one queued pair each per round (no divergence); a
// lane's pairs are added in discovery order: deterministic.
constexpr int kNearWarps = SER_FAR_THREADS / 32;  // one near unit per warp of the fused CTA
constexpr int kQCap = 64;  // per-lane ring capacity (power of two)
#ifndef SER_NEAR_MINB
#define SER_NEAR_MINB (512 / SER_FAR_THREADS)  // 16 resident warps per SM
#endif
// Per-warp SMEM of the near unit: source xyz of the sub-tile being classified,
// the per-lane ring queues and the lane targets' fields (SoA [field][lane]).
struct NearSmem {
  double sx[3][32];
  int q[kQCap][32];
  double tf[kNearFields][32];
};

template <int MODE, bool SHARP>
__device__ __forceinline__ void near_unit(const NearParams& p, int unit, NearSmem& sm) {
  const int lane = threadIdx.x & 31;
  int(*q)[32] = sm.q;
  double(*tf)[32] = sm.tf;
  const int n_sub = static_cast<int>(p.Npad / kSub);
  const int64_t g = unit / p.phases;
  const int phase = unit - static_cast<int>(g) * p.phases;
  const int64_t ti = g * 32 + lane;
  const double y0 = p.tgt[F_Y0 * p.Mpad + ti], y1 = p.tgt[F_Y1 * p.Mpad + ti], y2 = p.tgt[F_Y2 * p.Mpad + ti];
  __syncwarp();
  {
    const double* tq = p.tgt + ti;
    tf[NF_ALPHA][lane] = (MODE & 1) ? tq[F_ALPHA * p.Mpad] : 0.0;
    tf[NF_Q0][lane] = (MODE & 2) ? tq[F_Q0 * p.Mpad] : 0.0;
    tf[NF_Q1][lane] = (MODE & 2) ? tq[F_Q1 * p.Mpad] : 0.0;
    tf[NF_Q2][lane] = (MODE & 2) ? tq[F_Q2 * p.Mpad] : 0.0;
    tf[NF_N0][lane] = tq[F_N0 * p.Mpad];
    tf[NF_N1][lane] = tq[F_N1 * p.Mpad];
    tf[NF_N2][lane] = tq[F_N2 * p.Mpad];
    tf[NF_B][lane] = tq[F_B * p.Mpad];
    tf[NF_W0][lane] = tq[F_W0 * p.Mpad];
    tf[NF_W1][lane] = tq[F_W1 * p.Mpad];
    tf[NF_W2][lane] = tq[F_W2 * p.Mpad];
  }
  double lo[3] = {y0, y1, y2}, hi[3] = {y0, y1, y2};
#pragma unroll
  for (int d = 0; d < 3; ++d)
    for (int o = 16; o; o >>= 1) {
      lo[d] = fmin(lo[d], __shfl_xor_sync(0xffffffffu, lo[d], o));
      hi[d] = fmax(hi[d], __shfl_xor_sync(0xffffffffu, hi[d], o));
    }
  NearAcc acc{0.0, 0.0, 0.0, 0.0, 0.0, 0.0, 0.0};
  int head = 0, tail = 0;
  int ordinal = 0;  // index of the mixed sub-tile among this group's mixed sub-tiles

  // Invariant: every lane's queue holds <= kQCap - 32 entries before a sub-tile
  // appends its (<= 32) near sources.  One call site of the pair code.
  int base = 0;
  unsigned mm = 0;
  for (;;) {
    while (mm == 0 && base < n_sub) {
      bool mixed = false;
      const int sb = base + lane;
      if (sb < n_sub) {
        const double* bx = p.src_box + (int64_t)sb * 8;
        double g2 = 0.0;
#pragma unroll
        for (int d = 0; d < 3; ++d) {
          const double gap = fmax(0.0, fmax(__ldg(bx + d) - hi[d], lo[d] - __ldg(bx + 4 + d)));
          g2 = fma(gap, gap, g2);
        }
        mixed = g2 <= p.rc2_box;
      }
      mm = __ballot_sync(0xffffffffu, mixed);
      // keep only this phase's share of the mixed sub-tiles (round robin by ordinal)
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
        sm.sx[0][lane] = __ldg(gs);
        sm.sx[1][lane] = __ldg(gs + 1);
        sm.sx[2][lane] = __ldg(gs + 2);
      }
      __syncwarp();
      unsigned smask = 0;
#pragma unroll 8
      for (int k = 0; k < 32; ++k) {
        const double dx = y0 - sm.sx[0][k], dy = y1 - sm.sx[1][k], dz = y2 - sm.sx[2][k];
        const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
        smask |= (r2 <= p.rc2 ? 1u : 0u) << k;
      }
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
      rounds = __reduce_max_sync(0xffffffffu, tail - head);  // drain
    }
    for (int r = 0; r < rounds; ++r) {
      if (head < tail) {
        const int sidx = q[head & (kQCap - 1)][lane];
        ++head;
        const Src s = load_src_global<MODE>(p.src + (int64_t)sidx * kSrcDoubles);
        near_pair<MODE, SHARP>(s, y0, y1, y2, tf, lane, p, acc);
      }
    }
    if (last) break;
  }
  const double v0 = fma(-tf[NF_N0][lane], acc.kn, acc.v0), v1 = fma(-tf[NF_N1][lane], acc.kn, acc.v1),
               v2 = fma(-tf[NF_N2][lane], acc.kn, acc.v2);
  __syncwarp();  // all lanes done with sm before the warp's next unit overwrites it
  double* out = p.near_out + (int64_t)phase * 6 * p.Mpad + ti;
  out[0 * p.Mpad] = acc.u0; out[1 * p.Mpad] = acc.u1; out[2 * p.Mpad] = acc.u2;
  out[3 * p.Mpad] = v0; out[4 * p.Mpad] = v1; out[5 * p.Mpad] = v2;
}

// K3 (separate schedule): persistent warps pull units (group, phase) from a
// queue: balanced tails.
template <int MODE, bool SHARP>
__global__ void __launch_bounds__(kNearWarps * 32, SER_NEAR_MINB) near_kernel(const NearParams p) {
  __shared__ NearSmem s_near[kNearWarps];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (;;) {
    int unit = 0;
    if (lane == 0) unit = atomicAdd(p.counter, 1);
    unit = __shfl_sync(0xffffffffu, unit, 0);
    if (unit >= p.n_units) break;
    near_unit<MODE, SHARP>(p, unit, s_near[warp]);
  }
}

// K13 (fused schedule, the default): one persistent kernel runs both the far
// items (K1 body) and the near units (K3 body).  A near item is kNearWarps
// units, one per warp.  The queue interleaves the two kinds: the first
// (100 - SER_NEAR_TAIL_PCT)% of the near items are spread uniformly among the
// far items, so an SM's resident CTAs mix the FP64-issue-bound far loop with the
// latency-bound near pairs and the far warps fill the near warps' stalls; the
// rest follow the last far item and fill the tail.  The
// SMEM of the two bodies is a union; the item counter is PairParams::counter.
constexpr int kNearSmemBytes = kNearWarps * (int)sizeof(NearSmem);
constexpr int kFusedSmemBytes = kFarSmemBytes > kNearSmemBytes ? kFarSmemBytes : kNearSmemBytes;
#ifndef SER_NEAR_TAIL_PCT
#define SER_NEAR_TAIL_PCT 0
#endif

// Queue position -> work: returns true for a near item (index *idx), false for
// a far item.  Near items 0 .. n_mix-1 sit uniformly among the n_far far items,
// the remaining near items follow the last far item.
__device__ __forceinline__ bool fused_slot(int64_t qi, int64_t n_far, int64_t n_mix, int64_t* idx) {
  const int64_t head = n_far + n_mix;
  if (qi >= head) { *idx = n_mix + (qi - head); return true; }
  const int64_t na = qi * n_mix / head, nb = (qi + 1) * n_mix / head;
  if (nb > na) { *idx = na; return true; }
  *idx = qi - na;
  return false;
}

template <int MODE, int T, bool SHARP>
__global__ void __launch_bounds__(kThreads, SER_FAR_MINB) fused_kernel(const PairParams p, const NearParams np,
                                                                       int n_near_items) {
  static_assert(kThreads == kNearWarps * 32, "fused kernel: one near unit per warp");
  extern __shared__ __align__(128) unsigned char smem[];  // kFusedSmemBytes (dynamic: may exceed 48 KB)
  __shared__ __align__(8) uint64_t bar[2];
  __shared__ int s_item;
  auto* tile = reinterpret_cast<double(*)[kTile * kSrcDoubles]>(smem);
  auto* near_sm = reinterpret_cast<NearSmem*>(smem);
  if (threadIdx.x == 0) {
    mbar_init(&bar[0], 1);
    mbar_init(&bar[1], 1);
    fence_mbar_init();
  }
  __syncthreads();
  uint32_t parity0 = 0, parity1 = 0;
  const int64_t n_far = p.n_items;
  const int64_t n_mix = n_near_items - (int64_t)n_near_items * SER_NEAR_TAIL_PCT / 100;
  const int64_t total = n_far + n_near_items;
  for (;;) {
    if (threadIdx.x == 0) s_item = atomicAdd(p.counter, 1);
    __syncthreads();
    const int64_t qi = s_item;
    __syncthreads();  // every thread has read s_item (and left the previous item's SMEM)
    if (qi >= total) break;
    int64_t idx;
    if (fused_slot(qi, n_far, n_mix, &idx)) {
      const int64_t unit = idx * kNearWarps + (threadIdx.x >> 5);
      if (unit < np.n_units) near_unit<MODE, SHARP>(np, static_cast<int>(unit), near_sm[threadIdx.x >> 5]);
    } else {
      far_item<MODE, T>(p, static_cast<int>(idx), tile, bar, parity0, parity1);
    }
  }
}

// ------------------------------------------------------------ K2: finalize
// Small M (many partial slots per target: fine far chunks, up to 64 near phases): one warp per
// target, lanes stride over the slots, a fixed butterfly combines them (deterministic).
template <int MODE>
__global__ void finalize_small_kernel(const double* __restrict__ partial, const double* __restrict__ near_out,
                                      const double* __restrict__ tgt, const int32_t* __restrict__ orig, int64_t M,
                                      int64_t Mpad, int n_chunks, int TB, int phases, double* __restrict__ out_u,
                                      double* __restrict__ out_v) {
  const int64_t i = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (i >= M) return;  // whole warps
  const int64_t tb = i / TB, loc = i - tb * TB;
  double s[6] = {0, 0, 0, 0, 0, 0};
  for (int ch = lane; ch < n_chunks; ch += 32) {
    const double* pp = partial + ((tb * n_chunks + ch) * 6) * TB + loc;
#pragma unroll
    for (int c = 0; c < 6; ++c)
      if ((c < 3 && (MODE & 1)) || (c >= 3 && (MODE & 2))) s[c] += pp[c * TB];
  }
  for (int ph = lane; ph < phases; ph += 32)
#pragma unroll
    for (int c = 0; c < 6; ++c)
      if ((c < 3 && (MODE & 1)) || (c >= 3 && (MODE & 2))) s[c] += near_out[((int64_t)ph * 6 + c) * Mpad + i];
#pragma unroll
  for (int c = 0; c < 6; ++c)
    for (int o = 16; o; o >>= 1) s[c] += __shfl_xor_sync(0xffffffffu, s[c], o);
  if (lane != 0) return;
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

template <int MODE>
__global__ void finalize_kernel(const double* __restrict__ partial, const double* __restrict__ near_out,
                                const double* __restrict__ tgt, const int32_t* __restrict__ orig, int64_t M,
                                int64_t Mpad, int n_chunks, int TB, int phases, double* __restrict__ out_u,
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
  for (int ph = 0; ph < phases; ++ph)
#pragma unroll
    for (int c = 0; c < 6; ++c)
      if ((c < 3 && (MODE & 1)) || (c >= 3 && (MODE & 2))) s[c] += near_out[((int64_t)ph * 6 + c) * Mpad + i];
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
