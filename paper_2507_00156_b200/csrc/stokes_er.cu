// stokes_er.cu -- the C ABI of include/stokes_er.h: argument validation,
// workspace planning, launches on the caller's stream; plus the two small
// test entry points (per-delta sums, the extrapolation solve alone).
#include <algorithm>
#include <climits>
#include <cmath>

#include "kernels.cuh"
#include "treecode.cuh"
#include "sym.cuh"

namespace ser {

// ------------------------------------------- debug: per-delta sums (simple)
// One target per thread over the raw (unsorted) inputs; same near/far rule
// and the same pair algebra as K1 but one accumulator set per delta_k.
template <int MODE>
__global__ void deltas_kernel(const double* __restrict__ sx, const double* __restrict__ sn,
                              const double* __restrict__ sw, const double* __restrict__ f,
                              const double* __restrict__ q, const double* __restrict__ ty,
                              const double* __restrict__ tb, const double* __restrict__ x0d, int64_t M,
                              int64_t N, double h, Delta3 rho, double rc2, double r2_tiny,
                              double* __restrict__ out_ud, double* __restrict__ out_vd) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  const double y[3] = {ty[i], ty[M + i], ty[2 * M + i]};
  const double b = tb[i];
  double n0[3], f0[3], q0[3];
  for (int d = 0; d < 3; ++d) {
    n0[d] = x0d[d * M + i];
    f0[d] = (MODE & 1) ? x0d[(3 + d) * M + i] : 0.0;
    q0[d] = (MODE & 2) ? x0d[(6 + d) * M + i] : 0.0;
  }
  const double alpha = f0[0] * n0[0] + f0[1] * n0[1] + f0[2] * n0[2];
  double inv_delta[3];
  for (int k = 0; k < 3; ++k) inv_delta[k] = 1.0 / (rho.rho[k] * h);
  double Uf[3] = {0, 0, 0}, Vf[3] = {0, 0, 0}, U[3][3] = {}, V[3][3] = {};
  for (int64_t s = 0; s < N; ++s) {
    const double w = sw[s];
    double d[3], m[3], g[3], dq[3];
    for (int c = 0; c < 3; ++c) {
      d[c] = y[c] - sx[c * N + s];
      m[c] = sn[c * N + s] * w;
      g[c] = (MODE & 1) ? f[c * N + s] * w - alpha * m[c] : 0.0;
      dq[c] = (MODE & 2) ? q[c * N + s] - q0[c] : 0.0;
    }
    const double r2 = d[0] * d[0] + d[1] * d[1] + d[2] * d[2];
    const double dg = d[0] * g[0] + d[1] * g[1] + d[2] * g[2];
    const double dqq = d[0] * dq[0] + d[1] * dq[1] + d[2] * dq[2];
    const double dm = d[0] * m[0] + d[1] * m[1] + d[2] * m[2];
    if (r2 > rc2) {
      const double ri = 1.0 / sqrt(r2);
      const double ri3 = ri * ri * ri, ri5 = ri3 * ri * ri;
      for (int c = 0; c < 3; ++c) {
        Uf[c] += g[c] * ri + d[c] * dg * ri3;
        Vf[c] += d[c] * dqq * dm * ri5;
      }
      continue;
    }
    double xh[3];
    for (int c = 0; c < 3; ++c) xh[c] = b * n0[c] - d[c];
    const double an = n0[0] * dq[0] + n0[1] * dq[1] + n0[2] * dq[2];
    const double cn = n0[0] * m[0] + n0[1] * m[1] + n0[2] * m[2];
    const double dd = xh[0] * dq[0] + xh[1] * dq[1] + xh[2] * dq[2];
    const double e = xh[0] * m[0] + xh[1] * m[1] + xh[2] * m[2];
    double P[3];
    for (int c = 0; c < 3; ++c) P[c] = n0[c] * (b * an * cn - dd * cn - an * e) - xh[c] * an * cn;
    for (int k = 0; k < 3; ++k) {
      double A1, A3, A5, AP;
      if (r2 < r2_tiny) {
        const double id = inv_delta[k];
        A1 = kTwoOverSqrtPi * id;
        A3 = (2.0 / 3.0) * kTwoOverSqrtPi * id * id * id;
        A5 = (4.0 / 15.0) * kTwoOverSqrtPi * id * id * id * id * id;
        AP = A3;
      } else {
        const double r = sqrt(r2);
        double s1, s2, s3, c23;
        s_factors(r * inv_delta[k], s1, s2, s3, c23);
        A1 = s1 / r;
        A3 = s2 / (r2 * r);
        A5 = s3 / (r2 * r2 * r);
        AP = c23 / (r2 * r);
      }
      for (int c = 0; c < 3; ++c) {
        U[k][c] += g[c] * A1 + d[c] * dg * A3;
        V[k][c] += d[c] * dqq * dm * A5 + P[c] * AP;
      }
    }
  }
  const double inv8pi = 1.0 / (8.0 * kPi);
  const double chi = b < 0.0 ? 1.0 : (b > 0.0 ? 0.0 : 0.5);
  for (int k = 0; k < 3; ++k)
    for (int c = 0; c < 3; ++c) {
      if (MODE & 1) out_ud[(k * 3 + c) * M + i] = (Uf[c] + U[k][c]) * inv8pi;
      if (MODE & 2) out_vd[(k * 3 + c) * M + i] = -6.0 * (Vf[c] + V[k][c]) * inv8pi + chi * q0[c];
    }
}

// ------------------------------------------- the extrapolation solve alone
__global__ void extrapolate_kernel(const double* __restrict__ tb, int64_t M, double h, Delta3 rho,
                                   const double* __restrict__ in, int C, double* __restrict__ out) {
  const int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x;
  if (i >= M) return;
  double w[3];
  extrap_weights(tb[i], h, rho.rho, STOKES_ER_CUTOFF, w);
  for (int c = 0; c < C; ++c) {
    const double a0 = in[((int64_t)0 * C + c) * M + i], a1 = in[((int64_t)1 * C + c) * M + i],
                 a2 = in[((int64_t)2 * C + c) * M + i];
    out[(int64_t)c * M + i] = (w[1] == 0.0 && w[2] == 0.0) ? a0 : fma(w[0], a0, fma(w[1], a1, w[2] * a2));
  }
}

}  // namespace ser

// =================================================================== host side
namespace {

using namespace ser;

constexpr size_t kAlign = 256;
size_t align_up(size_t x) { return (x + kAlign - 1) / kAlign * kAlign; }
int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

struct Plan {
  int mode = 3, T = 2;
  int64_t M = 0, N = 0, Mpad = 0, Npad = 0;
  int n_tiles = 0, n_tblocks = 0, chunk_tiles = 0, n_chunks = 0, n_items = 0, near_phases = 1;
  size_t cub_bytes = 0;
  size_t off_box, off_skin, off_skout, off_svin, off_svout, off_tkin, off_tkout, off_tvin, off_tvout;
  size_t off_cub, off_src, off_srcbox, off_tgt, off_orig, off_partial, off_near, off_counter, total;
};

size_t cub_sort_bytes(int64_t n) {
  size_t bytes = 0;
  cub::DeviceRadixSort::SortPairs(nullptr, bytes, static_cast<const uint32_t*>(nullptr),
                                  static_cast<uint32_t*>(nullptr), static_cast<const int32_t*>(nullptr),
                                  static_cast<int32_t*>(nullptr), static_cast<int>(n), 0, 30);
  return bytes;
}

#ifndef SER_MAX_PHASES
#define SER_MAX_PHASES 64  // near phases per 32-target group at most (small M)
#endif
Plan make_plan(int64_t M, int64_t N, int mode, int T, int chunk_override, int phases_override = 0) {
  Plan p;
  p.mode = mode;
  p.T = (T >= 1 && T <= 4) ? T : 2;
  p.M = M;
  p.N = N;
  p.Npad = ceil_div(N, kTile) * kTile;
  p.n_tiles = static_cast<int>(p.Npad / kTile);
  const int TB = kThreads * p.T;
  p.n_tblocks = static_cast<int>(ceil_div(M > 0 ? M : 1, TB));
  p.Mpad = (int64_t)p.n_tblocks * TB;
  // work items (target block, source chunk): >= 24 per nominal CTA slot so the
  // dynamic queue's tail is small (measured: 16 -> 24 per slot, -0.5%), each
  // >= 4 tiles, partials <= kPartialCapBytes.
  const int64_t nominal_ctas = 148 * (16 * 32 / kThreads);  // 16 resident warps per SM
  int64_t want = ceil_div(24 * nominal_ctas, p.n_tblocks);
  const int64_t mem_cap = std::max<int64_t>(1, (int64_t)(kPartialCapBytes / (48.0 * (double)p.Mpad)));
  // >= 512 sources per item, unless that leaves fewer than two waves of items (small problems,
  // e.g. config 1: the critical path is then one item's loop): 128-source items
  int64_t min_tiles = std::max(1, 512 / kTile);
  if ((int64_t)p.n_tblocks * ceil_div(p.n_tiles, min_tiles) < 2 * nominal_ctas) min_tiles = 1;
  const int64_t max_chunks = std::max<int64_t>(1, std::min<int64_t>(ceil_div(p.n_tiles, min_tiles), mem_cap));
  want = std::min<int64_t>(std::max<int64_t>(want, 1), max_chunks);
  p.chunk_tiles = static_cast<int>(ceil_div(p.n_tiles, want));
  if (chunk_override > 0) p.chunk_tiles = std::min(chunk_override, p.n_tiles);
  p.n_chunks = static_cast<int>(ceil_div(p.n_tiles, p.chunk_tiles));
  p.n_items = p.n_tblocks * p.n_chunks;
  p.cub_bytes = std::max(cub_sort_bytes(N), cub_sort_bytes(std::max<int64_t>(M, 1)));
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  p.off_box = take(8 * sizeof(double));
  p.off_skin = take(N * 4);
  p.off_skout = take(N * 4);
  p.off_svin = take(N * 4);
  p.off_svout = take(N * 4);
  p.off_tkin = take(M * 4);
  p.off_tkout = take(M * 4);
  p.off_tvin = take(M * 4);
  p.off_tvout = take(M * 4);
  p.off_cub = take(p.cub_bytes);
  p.off_src = take(p.Npad * kSrcDoubles * sizeof(double));
  p.off_srcbox = take((p.Npad / kSub + p.Npad / 16) * 8 * sizeof(double));  // 32-source boxes, then halves
  p.off_tgt = take(p.Mpad * kTgtFields * sizeof(double));
  p.off_orig = take(p.Mpad * sizeof(int32_t));
  p.off_partial = take((size_t)p.n_items * 6 * TB * sizeof(double));
  // near units (32-target group, phase): >= ~4 per resident warp (148 SMs x 12 warps)
  const int64_t groups = p.Mpad / 32;
  // (up to 64 phases when there are few groups: small M; up to 128 below 32 groups, e.g. config 1's
  // 16: measured -8% per step there, +5-10% at 125-200 groups)
  const int64_t cap = groups >= 512 ? 16 : (groups < 32 ? 2 * SER_MAX_PHASES : SER_MAX_PHASES);
  p.near_phases = static_cast<int>(std::min<int64_t>(cap, std::max<int64_t>(1, ceil_div(10 * 148 * 16, groups))));
  if (phases_override > 0) p.near_phases = std::min(phases_override, 2 * SER_MAX_PHASES);
  p.off_near = take((size_t)p.near_phases * p.Mpad * 6 * sizeof(double));
  p.off_counter = take(sizeof(int) * 4);
  p.total = off;
  return p;
}

// N, M small enough for the counting-rank prologue (small_rank_kernel, kernels.cuh)
bool small_problem(int64_t M, int64_t N) { return N <= kSmallSort && M <= kSmallSort; }

bool rho_ok(const double* rho) {
  return rho && std::isfinite(rho[0]) && std::isfinite(rho[2]) && rho[0] > 0.0 && rho[1] > rho[0] &&
         rho[2] > rho[1];
}

int validate(const double* sx, const double* sn, const double* sw, const double* f, const double* q,
             const double* ty, const double* tb, const double* x0d, int64_t M, int64_t N, double h,
             const double* rho, int mode, bool check_rho = true) {
  if (mode < 1 || mode > 3) return STOKES_ER_EINVAL;
  if (M < 0 || N < 1 || M > INT32_MAX || N > INT32_MAX) return STOKES_ER_EINVAL;
  if (!(h > 0.0) || !std::isfinite(h) || (check_rho && !rho_ok(rho))) return STOKES_ER_EINVAL;
  if (!sx || !sn || !sw) return STOKES_ER_EINVAL;
  if (M > 0 && (!ty || !tb || !x0d)) return STOKES_ER_EINVAL;  // M == 0: no target arrays needed
  if ((mode & 1) && !f) return STOKES_ER_EINVAL;
  if ((mode & 2) && !q) return STOKES_ER_EINVAL;
  return STOKES_ER_OK;
}

int check_arch() {
  int dev = 0, major = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return STOKES_ER_ECUDA;
  if (cudaDeviceGetAttribute(&major, cudaDevAttrComputeCapabilityMajor, dev) != cudaSuccess)
    return STOKES_ER_ECUDA;
  return major == 10 ? STOKES_ER_OK : STOKES_ER_EARCH;
}

int opt_T(const stokes_er_options* o, int64_t M = -1) {
  if (o && o->targets_per_thread >= 1 && o->targets_per_thread <= 4) return o->targets_per_thread;
  // default 2 targets per thread; 1 for tiny M (fewer than 37 blocks of 128 targets, e.g. config 1's 504):
  // twice the target blocks for the critical path of a problem far smaller than the GPU
  return (M >= 0 && ceil_div(M, (int64_t)kThreads * 2) < 37) ? 1 : 2;
}
int opt_chunk(const stokes_er_options* o) { return o ? o->source_chunk_tiles : 0; }
int opt_phases(const stokes_er_options* o) { return o ? o->near_phases : 0; }
int opt_schedule(const stokes_er_options* o) { return o ? o->schedule : STOKES_ER_SCHEDULE_FUSED; }

// The caller's timing events (stokes_er_options): a plain record on the stream, or, while the stream
// is being captured into a CUDA graph, an external event-record node (a plain cudaEventRecord would
// only become a capture dependency, not a timestamp of each replay).
void record_event(void* ev, cudaStream_t s) {
  if (!ev) return;
  cudaStreamCaptureStatus st = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(s, &st) == cudaSuccess && st == cudaStreamCaptureStatusActive)
    cudaEventRecordWithFlags(static_cast<cudaEvent_t>(ev), s, cudaEventRecordExternal);
  else
    cudaEventRecord(static_cast<cudaEvent_t>(ev), s);
}

// Launch facts computed once per device (and per kernel): the SM count and a kernel's resident
// CTAs per SM after raising its dynamic-SMEM limit. Host-side only; it keeps the driver queries
// (~µs each) off the enqueue path of small evaluations, whose kernels take ~0.1 ms.
constexpr int kMaxDevices = 64;
int current_device() {
  int dev = 0;
  cudaGetDevice(&dev);
  return dev;
}
int device_sms() {
  static int cache[kMaxDevices];
  const int dev = current_device();
  int sms = (dev >= 0 && dev < kMaxDevices) ? cache[dev] : 0;
  if (sms == 0) {
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (dev >= 0 && dev < kMaxDevices) cache[dev] = sms;
  }
  return sms;
}
template <auto Kernel>
int resident_ctas(int threads, int dyn_smem) {
  static int cache[kMaxDevices][3];  // occupancy, threads, dyn_smem + 1
  const int dev = current_device();
  const bool ok = dev >= 0 && dev < kMaxDevices;
  if (ok && cache[dev][1] == threads && cache[dev][2] == dyn_smem + 1) return cache[dev][0];
  if (dyn_smem > 0) cudaFuncSetAttribute(Kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, dyn_smem);
  int occ = 0;
  cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, Kernel, threads, dyn_smem);
  if (ok) {
    cache[dev][0] = occ;
    cache[dev][1] = threads;
    cache[dev][2] = dyn_smem + 1;
  }
  return occ;
}

template <int MODE, int T>
void launch_pairs(const PairParams& pp, cudaStream_t s, int* grid_out) {
  const int sms = device_sms();
  const int occ = resident_ctas<far_kernel<MODE, T>>(kThreads, kFarSmemBytes);
  const int grid = std::max(1, std::min(pp.n_items, sms * std::max(occ, 1)));
  *grid_out = grid;
  far_kernel<MODE, T><<<grid, kThreads, kFarSmemBytes, s>>>(pp);
}

template <int MODE, int T, bool SHARP>
int launch_fused(const PairParams& pp, const NearParams& np, int n_near_items, int sms, cudaStream_t s) {
  const int occ = resident_ctas<fused_kernel<MODE, T, SHARP>>(kThreads, kFusedSmemBytes);
  const int64_t work = (int64_t)pp.n_items + n_near_items;
  const int grid = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(work, (int64_t)sms * std::max(occ, 1))));
  fused_kernel<MODE, T, SHARP><<<grid, kThreads, kFusedSmemBytes, s>>>(pp, np, n_near_items);
  return grid;
}

// SHARP = NEXT-1 on-surface variant: h = delta, rho = (1,1,1), weights (1,0,0),
// cutoff STOKES_ER_CUTOFF_SURFACE; otherwise the 3-delta extrapolated method.
template <int MODE, bool SHARP>
int run_eval(const double* sx, const double* sn, const double* sw, const double* f, const double* q,
             const double* ty, const double* tb, const double* x0d, int64_t M, int64_t N, double h,
             const double* rho, double* out_u, double* out_v, char* ws, const Plan& P, cudaStream_t s,
             stokes_er_options* opt) {
  long long* box = reinterpret_cast<long long*>(ws + P.off_box);
  uint32_t* skin = reinterpret_cast<uint32_t*>(ws + P.off_skin);
  uint32_t* skout = reinterpret_cast<uint32_t*>(ws + P.off_skout);
  int32_t* svin = reinterpret_cast<int32_t*>(ws + P.off_svin);
  int32_t* svout = reinterpret_cast<int32_t*>(ws + P.off_svout);
  uint32_t* tkin = reinterpret_cast<uint32_t*>(ws + P.off_tkin);
  uint32_t* tkout = reinterpret_cast<uint32_t*>(ws + P.off_tkout);
  int32_t* tvin = reinterpret_cast<int32_t*>(ws + P.off_tvin);
  int32_t* tvout = reinterpret_cast<int32_t*>(ws + P.off_tvout);
  double* src = reinterpret_cast<double*>(ws + P.off_src);
  double* srcbox = reinterpret_cast<double*>(ws + P.off_srcbox);
  double* tgt = reinterpret_cast<double*>(ws + P.off_tgt);
  int32_t* orig = reinterpret_cast<int32_t*>(ws + P.off_orig);
  double* partial = reinterpret_cast<double*>(ws + P.off_partial);
  double* near_out = reinterpret_cast<double*>(ws + P.off_near);
  int* counter = reinterpret_cast<int*>(ws + P.off_counter);

  Delta3 r3{{rho[0], rho[1], rho[2]}};
  if (small_problem(M, N)) {
    // small problems: box, keys and both Morton orders in one launch (ranks by counting), both packs
    // in one launch (the same order and records as below, 2 launches instead of ~15)
    small_rank_kernel<<<static_cast<int>(ceil_div(N, kRankPts) + ceil_div(M, kRankPts)), kRankThreads, 0, s>>>(
        sx, N, ty, M, svout, tvout, counter);
    pack_both<MODE><<<static_cast<int>(P.Npad / kTile + ceil_div(P.Mpad, kTile)), kTile, 0, s>>>(
        sx, sn, sw, f, q, N, P.Npad, svout, src, srcbox, ty, tb, x0d, M, P.Mpad, tvout, h, r3, SHARP, tgt, orig);
  } else {
    if (cudaMemsetAsync(box, 0x7f, 3 * sizeof(long long), s) != cudaSuccess ||
        cudaMemsetAsync(box + 3, 0x80, 3 * sizeof(long long), s) != cudaSuccess)
      return STOKES_ER_ECUDA;
    bbox_kernel<<<static_cast<int>(std::min<int64_t>(2 * 148, ceil_div(N + M, 256))), 256, 0, s>>>(sx, N, ty, M,
                                                                                                    box);
    morton_kernel<<<ceil_div(N, 256), 256, 0, s>>>(sx, N, box, skin, svin);
    morton_kernel<<<ceil_div(M, 256), 256, 0, s>>>(ty, M, box, tkin, tvin);
    size_t cb = P.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(ws + P.off_cub, cb, skin, skout, svin, svout, (int)N, 0, 30, s) !=
        cudaSuccess)
      return STOKES_ER_ECUDA;
    cb = P.cub_bytes;
    if (cub::DeviceRadixSort::SortPairs(ws + P.off_cub, cb, tkin, tkout, tvin, tvout, (int)M, 0, 30, s) !=
        cudaSuccess)
      return STOKES_ER_ECUDA;
    pack_sources<MODE><<<P.Npad / kTile, kTile, 0, s>>>(sx, sn, sw, f, q, N, P.Npad, svout, src, srcbox);
    pack_targets<MODE><<<ceil_div(P.Mpad, 256), 256, 0, s>>>(ty, tb, x0d, M, P.Mpad, tvout, h, r3, SHARP, tgt,
                                                              orig);
  }
  if (!small_problem(M, N) && cudaMemsetAsync(counter, 0, 2 * sizeof(int), s) != cudaSuccess)
    return STOKES_ER_ECUDA;

  PairParams pp;
  pp.src = src;
  pp.src_box = srcbox;
  pp.tgt = tgt;
  pp.partial = partial;
  pp.counter = counter;
  pp.Mpad = P.Mpad;
  pp.n_items = P.n_items;
  pp.n_chunks = P.n_chunks;
  pp.chunk_tiles = P.chunk_tiles;
  pp.n_tiles = P.n_tiles;
  const double dmax = rho[2] * h;
  const double cutoff = SHARP ? STOKES_ER_CUTOFF_SURFACE : STOKES_ER_CUTOFF;
  pp.rc2 = (cutoff * dmax) * (cutoff * dmax);
  pp.rc2_box = pp.rc2 * (1.0 + 1e-9);
  pp.rc2_inner = pp.rc2 * (1.0 - 1e-9);
  for (int k = 0; k < 3; ++k) pp.inv_delta[k] = 1.0 / (rho[k] * h);

  NearParams np;
  np.src = src;
  np.src_box = srcbox;
  np.tgt = tgt;
  np.near_out = near_out;
  np.counter = counter + 1;
  np.phases = P.near_phases;
  np.n_units = static_cast<int>((P.Mpad / 32) * P.near_phases);
  np.Mpad = P.Mpad;
  np.Npad = P.Npad;
  np.rc2 = pp.rc2;
  np.rc2_box = pp.rc2_box;
  for (int k = 0; k < 3; ++k) np.inv_delta[k] = pp.inv_delta[k];

  const int sms = device_sms();
  int grid = 0;
  if (opt_schedule(opt) == STOKES_ER_SCHEDULE_FUSED) {
    // one persistent kernel: far items and near items (kNearWarps units each) interleaved
    const int n_near_items = static_cast<int>(ceil_div(np.n_units, kNearWarps));
    if (opt) record_event(opt->pair_kernel_start_event, s);
    if (P.T == 4) grid = launch_fused<MODE, 4, SHARP>(pp, np, n_near_items, sms, s);
    else if (P.T == 3) grid = launch_fused<MODE, 3, SHARP>(pp, np, n_near_items, sms, s);
    else if (P.T == 1) grid = launch_fused<MODE, 1, SHARP>(pp, np, n_near_items, sms, s);
    else grid = launch_fused<MODE, 2, SHARP>(pp, np, n_near_items, sms, s);
    if (opt) record_event(opt->pair_kernel_end_event, s);
  } else {
    if (opt) record_event(opt->pair_kernel_start_event, s);
    if (P.T == 4) launch_pairs<MODE, 4>(pp, s, &grid);
    else if (P.T == 3) launch_pairs<MODE, 3>(pp, s, &grid);
    else if (P.T == 1) launch_pairs<MODE, 1>(pp, s, &grid);
    else launch_pairs<MODE, 2>(pp, s, &grid);
    if (opt) record_event(opt->pair_kernel_end_event, s);
    if (opt) record_event(opt->near_kernel_start_event, s);
    const int occ = resident_ctas<near_kernel<MODE, SHARP>>(kNearWarps * 32, 0);
    const int ngrid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(np.n_units, kNearWarps), (int64_t)sms * std::max(occ, 1))));
    near_kernel<MODE, SHARP><<<ngrid, kNearWarps * 32, 0, s>>>(np);
    if (opt) record_event(opt->near_kernel_end_event, s);
  }
  if (opt) {
    opt->stats[0] = P.n_items;
    opt->stats[1] = grid;
    opt->stats[2] = P.chunk_tiles;
    opt->stats[3] = P.T;
  }
  if (small_problem(M, N))  // many slots per target, few targets: a warp per target
    finalize_small_kernel<MODE><<<ceil_div(M * 32, 256), 256, 0, s>>>(partial, near_out, tgt, orig, M, P.Mpad,
                                                                      P.n_chunks, kThreads * P.T, P.near_phases,
                                                                      out_u, out_v);
  else
    finalize_kernel<MODE><<<ceil_div(M, 256), 256, 0, s>>>(partial, near_out, tgt, orig, M, P.Mpad, P.n_chunks,
                                                            kThreads * P.T, P.near_phases, out_u, out_v);
  return cudaGetLastError() == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}


// NEXT-3: the treecode evaluation (treecode.cuh).  Same pipeline as run_eval
// with the sources in tree order (the plan's permutation), the far part from
// tree_far_kernel and the near pairs from the near units.
struct TreeWs {
  size_t off_nodes, off_perm, off_G, off_sched, total;
};
TreeWs tree_ws_layout(const Plan& P, int nnodes, int64_t N, int p) {
  TreeWs w;
  size_t off = align_up(P.total);
  w.off_nodes = off;
  off = align_up(off + (size_t)nnodes * sizeof(TreeNode));
  w.off_perm = off;
  off = align_up(off + (size_t)N * sizeof(int32_t));
  w.off_G = off;
  off = align_up(off + (size_t)nnodes * (p + 1) * (p + 1) * (p + 1) * kTreeCh * sizeof(double));
  w.off_sched = off;
  off = align_up(off + (size_t)nnodes * sizeof(int));
  w.total = off;
  return w;
}

template <int MODE, bool SHARP>
int run_eval_tree(const double* sx, const double* sn, const double* sw, const double* f, const double* q,
                  const double* ty, const double* tb, const double* x0d, int64_t M, int64_t N, double h,
                  const double* rho, const stokes_er_tree_params* tp, const TreePlanHeader* hdr,
                  const char* plan, double* out_u, double* out_v, char* ws, const Plan& P, const TreeWs& W,
                  cudaStream_t s) {
  long long* box = reinterpret_cast<long long*>(ws + P.off_box);
  uint32_t* tkin = reinterpret_cast<uint32_t*>(ws + P.off_tkin);
  uint32_t* tkout = reinterpret_cast<uint32_t*>(ws + P.off_tkout);
  int32_t* tvin = reinterpret_cast<int32_t*>(ws + P.off_tvin);
  int32_t* tvout = reinterpret_cast<int32_t*>(ws + P.off_tvout);
  double* src = reinterpret_cast<double*>(ws + P.off_src);
  double* srcbox = reinterpret_cast<double*>(ws + P.off_srcbox);
  double* tgt = reinterpret_cast<double*>(ws + P.off_tgt);
  int32_t* orig = reinterpret_cast<int32_t*>(ws + P.off_orig);
  double* partial = reinterpret_cast<double*>(ws + P.off_partial);
  double* near_out = reinterpret_cast<double*>(ws + P.off_near);
  int* counter = reinterpret_cast<int*>(ws + P.off_counter);
  TreeNode* nodes = reinterpret_cast<TreeNode*>(ws + W.off_nodes);
  int32_t* perm = reinterpret_cast<int32_t*>(ws + W.off_perm);
  double* G = reinterpret_cast<double*>(ws + W.off_G);
  const int nn = hdr->nnodes, p = tp->degree;

  if (cudaMemcpyAsync(nodes, plan + hdr->off_nodes, (size_t)nn * sizeof(TreeNode), cudaMemcpyHostToDevice, s) !=
          cudaSuccess ||
      cudaMemcpyAsync(perm, plan + hdr->off_perm, (size_t)N * sizeof(int32_t), cudaMemcpyHostToDevice, s) !=
          cudaSuccess)
    return STOKES_ER_ECUDA;
  if (cudaMemsetAsync(box, 0x7f, 3 * sizeof(long long), s) != cudaSuccess ||
      cudaMemsetAsync(box + 3, 0x80, 3 * sizeof(long long), s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  bbox_kernel<<<static_cast<int>(std::min<int64_t>(2 * 148, ceil_div(N + M, 256))), 256, 0, s>>>(sx, N, ty, M, box);
  morton_kernel<<<ceil_div(M, 256), 256, 0, s>>>(ty, M, box, tkin, tvin);
  size_t cb = P.cub_bytes;
  if (cub::DeviceRadixSort::SortPairs(ws + P.off_cub, cb, tkin, tkout, tvin, tvout, (int)M, 0, 30, s) !=
      cudaSuccess)
    return STOKES_ER_ECUDA;
  pack_sources<MODE><<<P.Npad / kTile, kTile, 0, s>>>(sx, sn, sw, f, q, N, P.Npad, perm, src, srcbox);
  Delta3 r3{{rho[0], rho[1], rho[2]}};
  pack_targets<MODE><<<ceil_div(P.Mpad, 256), 256, 0, s>>>(ty, tb, x0d, M, P.Mpad, tvout, h, r3, SHARP, tgt, orig);
  {  // modified weights: leaves from their sources, then internal nodes level by level (M2M)
    const TreeNode* hn = reinterpret_cast<const TreeNode*>(plan + hdr->off_nodes);
    std::vector<int> sched;
    std::vector<int> level_start;
    for (int i = 0; i < nn; ++i)
      if (hn[i].nchild == 0) sched.push_back(i);
    const int n_leaves = static_cast<int>(sched.size());
    for (int lv = hdr->depth; lv >= 0; --lv) {
      level_start.push_back(static_cast<int>(sched.size()));
      for (int i = 0; i < nn; ++i)
        if (hn[i].nchild > 0 && hn[i].level == lv) sched.push_back(i);
    }
    level_start.push_back(static_cast<int>(sched.size()));
    int* ids = reinterpret_cast<int*>(ws + W.off_sched);
    if (cudaMemcpyAsync(ids, sched.data(), sched.size() * sizeof(int), cudaMemcpyHostToDevice, s) != cudaSuccess)
      return STOKES_ER_ECUDA;
    tree_p2m_kernel<MODE><<<n_leaves, 256, 0, s>>>(nodes, ids, src, p, G);
    const int m2m_smem = 2 * (p + 1) * (p + 1) * (p + 1) * static_cast<int>(sizeof(double));
    if (cudaFuncSetAttribute(tree_m2m_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, m2m_smem) !=
        cudaSuccess)
      return STOKES_ER_ECUDA;
    for (size_t l = 0; l + 1 < level_start.size(); ++l) {
      const int a = level_start[l], b = level_start[l + 1];
      if (b > a) tree_m2m_kernel<MODE><<<b - a, 256, m2m_smem, s>>>(nodes, ids + a, p, G);
    }
  }
  if (cudaMemsetAsync(counter, 0, 2 * sizeof(int), s) != cudaSuccess) return STOKES_ER_ECUDA;
  const double dmax = rho[2] * h;
  const double cutoff = SHARP ? STOKES_ER_CUTOFF_SURFACE : STOKES_ER_CUTOFF;
  const double rc2 = (cutoff * dmax) * (cutoff * dmax);
  const int sms = device_sms();
  TreeFarParams tfp;
  tfp.nodes = nodes;
  tfp.G = G;
  tfp.src = src;
  tfp.tgt = tgt;
  tfp.partial = partial;
  tfp.counter = counter;
  tfp.Mpad = P.Mpad;
  tfp.n_groups = static_cast<int>(P.Mpad / 32);
  tfp.p = p;
  tfp.theta = tp->theta;
  tfp.rc2 = rc2;
  tfp.rc2_guard = rc2 * (1.0 + 1e-9);  // R23 guard with the rc2_box margin: no pair the near units own is approximated
  NearParams np;
  np.src = src;
  np.src_box = srcbox;
  np.tgt = tgt;
  np.near_out = near_out;
  np.counter = counter + 1;
  np.phases = P.near_phases;
  np.n_units = static_cast<int>((P.Mpad / 32) * P.near_phases);
  np.Mpad = P.Mpad;
  np.Npad = P.Npad;
  np.rc2 = rc2;
  np.rc2_box = rc2 * (1.0 + 1e-9);
  for (int k = 0; k < 3; ++k) np.inv_delta[k] = 1.0 / (rho[k] * h);
  {  // one persistent kernel: tree walks of the target groups + the near units
    const int n_near = SER_TREE_FUSED_NEAR ? np.n_units : 0;
    const int occ = resident_ctas<tree_far_kernel<MODE, SHARP>>(kTreeWarps * 32, 0);
    const int64_t work = (int64_t)tfp.n_groups + n_near;
    const int grid = static_cast<int>(std::max<int64_t>(
        1, std::min<int64_t>(ceil_div(work, kTreeWarps), (int64_t)sms * std::max(occ, 1))));
    tree_far_kernel<MODE, SHARP><<<grid, kTreeWarps * 32, 0, s>>>(tfp, np, n_near);
    if (!SER_TREE_FUSED_NEAR) {
      const int nocc = resident_ctas<near_kernel<MODE, SHARP>>(kNearWarps * 32, 0);
      const int ngrid = static_cast<int>(std::max<int64_t>(
          1, std::min<int64_t>(ceil_div(np.n_units, kNearWarps), (int64_t)sms * std::max(nocc, 1))));
      near_kernel<MODE, SHARP><<<ngrid, kNearWarps * 32, 0, s>>>(np);
    }
  }
  finalize_kernel<MODE><<<ceil_div(M, 256), 256, 0, s>>>(partial, near_out, tgt, orig, M, P.Mpad, 1, 32,
                                                          P.near_phases, out_u, out_v);
  return cudaGetLastError() == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}


// ------------------------------------------------------------- node targets
// stokes_er_eval_nodes (sym.cuh): the symmetric far kernel over kBlk-node (96-node) block
// pairs + the neighbour units + finalize.  The plan depends on N only.
struct NodePlan {
  int mode = 3;
  int64_t N = 0, Npad = 0, n_items = 0;
  int nb = 0, nsb = 0, chunk = 0, nchunks = 0, G = 0, near_phases = 1;
  size_t cub_bytes = 0, sym_smem = 0;
  size_t off_box, off_skin, off_skout, off_svin, off_svout, off_cub, off_src, off_srcbox, off_blkbox, off_nsoa;
  size_t off_tgt, off_orig, off_pacc, off_near, off_counter, total;
};

#ifndef SER_SYM_GRID
#define SER_SYM_GRID 148
#endif
constexpr int kSymGrid = SER_SYM_GRID;  // persistent CTAs (one per B200 SM): fixed, so results do not depend on the device

int64_t sym_items(int nsb, int k, int nchunks) {  // sum over chunks c of min(nsb, (c + 1) k)
  int64_t n = 0;
  for (int c = 0; c < nchunks; ++c) n += std::min<int64_t>(nsb, (int64_t)(c + 1) * k);
  return n;
}

NodePlan make_node_plan(int64_t N, int mode, int phases_override = 0) {
  NodePlan p;
  p.mode = mode;
  p.N = N;
  constexpr int64_t kPadUnit = kBlk % kTile == 0 ? kBlk : (kTile % kBlk == 0 ? kTile : (int64_t)kTile * kBlk / 32);
  p.Npad = ceil_div(N, kPadUnit) * kPadUnit;  // whole symmetric blocks and 128-target blocks (384 = lcm(96, 128) for 96-node blocks)
  p.nb = static_cast<int>(p.Npad / kBlk);
  p.nsb = static_cast<int>(ceil_div(p.nb, kSymWarps));
  // R blocks per item: the largest multiple of the warp count (<= 4 of them, SMEM) that still
  // gives every CTA >= 16 items (balance of the static assignment)
  auto smem_of = [](int kk) {
    return (size_t)kSymStages * kBlkTileBytes + (size_t)kSymRedBufs * kSymWarps * 6 * kBlk * 8 +
           (size_t)6 * kk * kSymWarps * kBlk * 8;
  };
  int k = SER_SYM_MAXK;
  while (k > 1 && smem_of(k) > 227 * 1024) --k;  // the opt-in SMEM limit per CTA (tuning macros can exceed it)
  for (; k > 1; --k) {
    const int nch = static_cast<int>(ceil_div(p.nb, k * kSymWarps));
    if (sym_items(p.nsb, k, nch) >= 16 * kSymGrid) break;
  }
  p.chunk = k * kSymWarps;
  p.nchunks = static_cast<int>(ceil_div(p.nb, p.chunk));
  p.n_items = sym_items(p.nsb, k, p.nchunks);
  p.G = static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(kSymGrid, p.n_items)));
  p.sym_smem = smem_of(k);
  p.cub_bytes = cub_sort_bytes(N);
  const int64_t groups = p.Npad / 32;
  p.near_phases = static_cast<int>(std::min<int64_t>(16, std::max<int64_t>(1, ceil_div(10 * 148 * 16, groups))));
  if (phases_override > 0) p.near_phases = std::min(phases_override, 64);
  size_t off = 0;
  auto take = [&](size_t bytes) {
    const size_t o = off;
    off = align_up(off + bytes);
    return o;
  };
  p.off_box = take(8 * sizeof(double));
  p.off_skin = take(N * 4);
  p.off_skout = take(N * 4);
  p.off_svin = take(N * 4);
  p.off_svout = take(N * 4);
  p.off_cub = take(p.cub_bytes);
  p.off_src = take(p.Npad * kSrcDoubles * sizeof(double));
  p.off_srcbox = take((p.Npad / kSub + p.Npad / 16) * 8 * sizeof(double));
  p.off_blkbox = take((size_t)p.nb * 8 * sizeof(double));
  p.off_nsoa = take(p.Npad * kNodeStride * sizeof(double));
  p.off_tgt = take(p.Npad * kTgtFields * sizeof(double));
  p.off_orig = take(p.Npad * sizeof(int32_t));
  p.off_pacc = take((size_t)p.G * 6 * p.Npad * sizeof(double));
  p.off_near = take((size_t)p.near_phases * p.Npad * 6 * sizeof(double));
  p.off_counter = take(sizeof(int) * 8);
  p.total = off;
  return p;
}

// SHARP: NEXT-1's on-surface s# evaluation (h = delta, rho = (1,1,1), cutoff STOKES_ER_CUTOFF_SURFACE,
// weights (1,0,0)); otherwise the 3-delta extrapolated method.  The far pairs are the same either way.
template <int MODE, bool SHARP>
int run_nodes(const double* sx, const double* sn, const double* sw, const double* f, const double* q, int64_t N,
              double h, const double* rho, double* out_u, double* out_v, char* ws, const NodePlan& P, cudaStream_t s,
              stokes_er_options* opt) {
  long long* box = reinterpret_cast<long long*>(ws + P.off_box);
  uint32_t* skin = reinterpret_cast<uint32_t*>(ws + P.off_skin);
  uint32_t* skout = reinterpret_cast<uint32_t*>(ws + P.off_skout);
  int32_t* svin = reinterpret_cast<int32_t*>(ws + P.off_svin);
  int32_t* svout = reinterpret_cast<int32_t*>(ws + P.off_svout);
  double* src = reinterpret_cast<double*>(ws + P.off_src);
  double* srcbox = reinterpret_cast<double*>(ws + P.off_srcbox);
  double* blkbox = reinterpret_cast<double*>(ws + P.off_blkbox);
  double* nsoa = reinterpret_cast<double*>(ws + P.off_nsoa);
  double* tgt = reinterpret_cast<double*>(ws + P.off_tgt);
  int32_t* orig = reinterpret_cast<int32_t*>(ws + P.off_orig);
  double* pacc = reinterpret_cast<double*>(ws + P.off_pacc);
  double* near_out = reinterpret_cast<double*>(ws + P.off_near);
  int* counter = reinterpret_cast<int*>(ws + P.off_counter);

  if (cudaMemsetAsync(box, 0x7f, 3 * sizeof(long long), s) != cudaSuccess ||
      cudaMemsetAsync(box + 3, 0x80, 3 * sizeof(long long), s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  bbox_kernel<<<static_cast<int>(std::min<int64_t>(2 * 148, ceil_div(N, 256))), 256, 0, s>>>(sx, N, sx, 0, box);
  morton_kernel<<<ceil_div(N, 256), 256, 0, s>>>(sx, N, box, skin, svin);
  size_t cb = P.cub_bytes;
  if (cub::DeviceRadixSort::SortPairs(ws + P.off_cub, cb, skin, skout, svin, svout, (int)N, 0, 30, s) !=
      cudaSuccess)
    return STOKES_ER_ECUDA;
  pack_sources<MODE><<<P.Npad / kTile, kTile, 0, s>>>(sx, sn, sw, f, q, N, P.Npad, svout, src, srcbox);
  Delta3 r3{{rho[0], rho[1], rho[2]}};
  pack_node_soa<MODE><<<ceil_div(P.Npad, 256), 256, 0, s>>>(sx, sn, sw, f, q, N, P.Npad, svout, h, r3, SHARP, nsoa,
                                                             tgt, orig);
  block_boxes<<<ceil_div(P.nb, 256), 256, 0, s>>>(srcbox, P.nb, blkbox);
  if (cudaMemsetAsync(pacc, 0, (size_t)P.G * 6 * P.Npad * sizeof(double), s) != cudaSuccess ||
      cudaMemsetAsync(counter, 0, 2 * sizeof(int), s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  if (opt && opt->shard_count > 1 &&  // a shard writes only its groups' neighbour partials: zero the rest
      cudaMemsetAsync(near_out, 0, (size_t)P.near_phases * P.Npad * 6 * sizeof(double), s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  const double dmax = rho[2] * h;
  const double cutoff = SHARP ? STOKES_ER_CUTOFF_SURFACE : STOKES_ER_CUTOFF;
  const double rc2 = (cutoff * dmax) * (cutoff * dmax);
  SymParams sp;
  sp.nsoa = nsoa;
  sp.blk_box = blkbox;
  sp.pacc = pacc;
  sp.Npad = P.Npad;
  sp.nb = P.nb;
  sp.nsb = P.nsb;
  sp.chunk = P.chunk;
  sp.nchunks = P.nchunks;
  sp.n_items = P.n_items;
  // a shard (options.shard_index / shard_count) takes a contiguous share of the items and of the
  // neighbour units' target groups, and returns partial sums
  const int nshard = (opt && opt->shard_count > 1) ? opt->shard_count : 1;
  const int ishard = nshard > 1 ? opt->shard_index : 0;
  sp.item_begin = P.n_items * ishard / nshard;
  sp.item_end = P.n_items * (ishard + 1) / nshard;
  sp.rc2_box = rc2 * (1.0 + 1e-9);
  NearParams np;
  np.src = src;
  np.src_box = srcbox;
  np.tgt = tgt;
  np.near_out = near_out;
  np.counter = counter + 1;
  np.phases = P.near_phases;
  const int64_t n_groups = P.Npad / 32;
  const int64_t g0 = n_groups * ishard / nshard, g1 = n_groups * (ishard + 1) / nshard;
  const int unit_base = static_cast<int>(g0 * P.near_phases);
  np.n_units = static_cast<int>((g1 - g0) * P.near_phases);
  np.Mpad = P.Npad;
  np.Npad = P.Npad;
  np.rc2 = rc2;
  np.rc2_box = sp.rc2_box;
  for (int k = 0; k < 3; ++k) np.inv_delta[k] = 1.0 / (rho[k] * h);
  if (cudaFuncSetAttribute(sym_kernel<MODE>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)P.sym_smem) !=
      cudaSuccess)
    return STOKES_ER_ECUDA;
  if (opt) record_event(opt->pair_kernel_start_event, s);
  sym_kernel<MODE><<<P.G, kSymThreads, P.sym_smem, s>>>(sp);
  if (opt) record_event(opt->pair_kernel_end_event, s);
  if (opt) record_event(opt->near_kernel_start_event, s);
  {
    const int sms = device_sms();
    const int occ = resident_ctas<nbr_kernel<MODE, SHARP>>(64, 0);
    const int ngrid = static_cast<int>(
        std::max<int64_t>(1, std::min<int64_t>(ceil_div(np.n_units, 2), (int64_t)sms * std::max(occ, 1))));
    nbr_kernel<MODE, SHARP><<<ngrid, 64, 0, s>>>(np, blkbox, unit_base);
  }
  if (opt) record_event(opt->near_kernel_end_event, s);
  if (opt) {
    opt->stats[0] = P.n_items;
    opt->stats[1] = P.G;
    opt->stats[2] = P.chunk;
    opt->stats[3] = kSymT;  // I nodes per lane of the symmetric kernel
  }
  finalize_nodes<MODE><<<ceil_div(N, 256), 256, 0, s>>>(pacc, P.G, near_out, P.near_phases, tgt, orig, N, P.Npad,
                                                         ishard == 0 ? 0.5 : 0.0, out_u, out_v);
  return cudaGetLastError() == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}

size_t node_host_stage_bytes(int64_t N) { return align_up(13 * N * sizeof(double)) + align_up(6 * N * sizeof(double)) + 2 * kAlign; }

bool tree_params_ok(const stokes_er_tree_params* tp) {
  return tp && tp->leaf_size >= 1 && tp->degree >= 1 && tp->degree <= kTreeMaxDegree && std::isfinite(tp->theta) &&
         tp->theta >= 0.0;
}

const TreePlanHeader* tree_header(const void* plan, int64_t N) {
  if (!plan) return nullptr;
  const TreePlanHeader* h = static_cast<const TreePlanHeader*>(plan);
  if (h->magic != kTreeMagic || h->N != N || h->nnodes < 1) return nullptr;
  return h;
}

size_t host_stage_bytes(int64_t M, int64_t N) {
  return align_up(13 * N * sizeof(double)) + align_up(13 * M * sizeof(double)) + align_up(6 * M * sizeof(double)) +
         4 * kAlign;
}

}  // namespace

extern "C" {

size_t stokes_er_workspace_bytes(int64_t M, int64_t N, int mode) {
  if (M < 0 || N < 1 || mode < 1 || mode > 3) return 0;
  // the larger of the two tunings, so one workspace serves every option
  return std::max({make_plan(M, N, mode, 1, 0).total, make_plan(M, N, mode, 2, 0).total,
                   make_plan(M, N, mode, 3, 0).total, make_plan(M, N, mode, 4, 0).total});
}

size_t stokes_er_workspace_bytes_ex(int64_t M, int64_t N, int mode, const stokes_er_options* options) {
  if (M < 0 || N < 1 || mode < 1 || mode > 3) return 0;
  return std::max(stokes_er_workspace_bytes(M, N, mode),
                  make_plan(M, N, mode, opt_T(options, M), opt_chunk(options), opt_phases(options)).total);
}

static int eval_common(const double* src_xyz, const double* src_normal, const double* src_weight, const double* f,
                       const double* q, const double* tgt_xyz, const double* tgt_b, const double* tgt_x0_density,
                       int64_t M, int64_t N, double h, const double rho[3], int mode, double* out_u,
                       double* out_v, void* workspace, size_t workspace_bytes, void* stream,
                       stokes_er_options* options, bool sharp) {
  int st = validate(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, mode,
                    !sharp);
  if (st) return st;
  if (M == 0) return STOKES_ER_OK;
  if (((mode & 1) && !out_u) || ((mode & 2) && !out_v)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  const Plan P = make_plan(M, N, mode, opt_T(options, M), opt_chunk(options), opt_phases(options));
  if (!workspace || workspace_bytes < P.total) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
#define SER_RUN(M_, S_)                                                                                          \
  run_eval<M_, S_>(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, out_u, \
                   out_v, ws, P, s, options)
  if (sharp) {
    switch (mode) {
      case 1: return SER_RUN(1, true);
      case 2: return SER_RUN(2, true);
      default: return SER_RUN(3, true);
    }
  }
  switch (mode) {
    case 1: return SER_RUN(1, false);
    case 2: return SER_RUN(2, false);
    default: return SER_RUN(3, false);
  }
#undef SER_RUN
}

int stokes_er_eval_ex(const double* src_xyz, const double* src_normal, const double* src_weight,
                      const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                      const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho[3],
                      int mode, double* out_u, double* out_v, void* workspace, size_t workspace_bytes,
                      void* stream, stokes_er_options* options) {
  return eval_common(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, mode,
                     out_u, out_v, workspace, workspace_bytes, stream, options, false);
}

int stokes_er_eval_onsurface(const double* src_xyz, const double* src_normal, const double* src_weight,
                             const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                             const double* tgt_x0_density, int64_t M, int64_t N, double delta, int mode,
                             double* out_u, double* out_v, void* workspace, size_t workspace_bytes,
                             void* stream) {
  const double one[3] = {1.0, 1.0, 1.0};  // delta_1 = delta_2 = delta_3 = delta; weights (1, 0, 0)
  return eval_common(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, delta, one, mode,
                     out_u, out_v, workspace, workspace_bytes, stream, nullptr, true);
}

int stokes_er_eval(const double* src_xyz, const double* src_normal, const double* src_weight, const double* f,
                   const double* q, const double* tgt_xyz, const double* tgt_b, const double* tgt_x0_density,
                   int64_t M, int64_t N, double h, const double rho[3], int mode, double* out_u, double* out_v,
                   void* workspace, size_t workspace_bytes, void* stream) {
  return stokes_er_eval_ex(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho,
                           mode, out_u, out_v, workspace, workspace_bytes, stream, nullptr);
}

size_t stokes_er_host_workspace_bytes(int64_t M, int64_t N, int mode) {
  const size_t w = stokes_er_workspace_bytes(M, N, mode);
  return w ? align_up(w) + host_stage_bytes(M, N) : 0;
}

int stokes_er_eval_host(const double* sx, const double* sn, const double* sw, const double* f, const double* q,
                        const double* ty, const double* tb, const double* x0d, int64_t M, int64_t N, double h,
                        const double rho[3], int mode, double* out_u, double* out_v, void* workspace,
                        size_t workspace_bytes, void* stream) {
  int st = validate(sx, sn, sw, f, q, ty, tb, x0d, M, N, h, rho, mode);
  if (st) return st;
  if (M == 0) return STOKES_ER_OK;
  if (((mode & 1) && !out_u) || ((mode & 2) && !out_v)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  const size_t wbytes = align_up(stokes_er_workspace_bytes(M, N, mode));
  if (!workspace || workspace_bytes < wbytes + host_stage_bytes(M, N)) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* stage = static_cast<char*>(workspace) + wbytes;
  double* dsx = reinterpret_cast<double*>(stage);
  double *dsn = dsx + 3 * N, *dsw = dsn + 3 * N, *df = dsw + N, *dq = df + 3 * N;
  double* dty = reinterpret_cast<double*>(stage + align_up(13 * N * sizeof(double)));
  double *dtb = dty + 3 * M, *dx0 = dtb + M;
  double* du =
      reinterpret_cast<double*>(stage + align_up(13 * N * sizeof(double)) + align_up(13 * M * sizeof(double)));
  double* dv = du + 3 * M;
  auto h2d = [&](double* dst, const double* src, int64_t n) {
    return src ? cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  if (h2d(dsx, sx, 3 * N) || h2d(dsn, sn, 3 * N) || h2d(dsw, sw, N) || h2d(df, (mode & 1) ? f : nullptr, 3 * N) ||
      h2d(dq, (mode & 2) ? q : nullptr, 3 * N) || h2d(dty, ty, 3 * M) || h2d(dtb, tb, M) || h2d(dx0, x0d, 9 * M))
    return STOKES_ER_ECUDA;
  st = stokes_er_eval_ex(dsx, dsn, dsw, (mode & 1) ? df : nullptr, (mode & 2) ? dq : nullptr, dty, dtb, dx0, M, N,
                         h, rho, mode, (mode & 1) ? du : nullptr, (mode & 2) ? dv : nullptr, workspace, wbytes,
                         stream, nullptr);
  if (st) return st;
  if ((mode & 1) && cudaMemcpyAsync(out_u, du, 3 * M * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  if ((mode & 2) && cudaMemcpyAsync(out_v, dv, 3 * M * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}

int stokes_er_eval_deltas(const double* sx, const double* sn, const double* sw, const double* f, const double* q,
                          const double* ty, const double* tb, const double* x0d, int64_t M, int64_t N, double h,
                          const double rho[3], int mode, double* out_ud, double* out_vd, void* workspace,
                          size_t workspace_bytes, void* stream) {
  (void)workspace;
  (void)workspace_bytes;
  int st = validate(sx, sn, sw, f, q, ty, tb, x0d, M, N, h, rho, mode);
  if (st) return st;
  if (M == 0) return STOKES_ER_OK;
  if (((mode & 1) && !out_ud) || ((mode & 2) && !out_vd)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  Delta3 r3{{rho[0], rho[1], rho[2]}};
  const double dmax = rho[2] * h;
  const double rc2 = (STOKES_ER_CUTOFF * dmax) * (STOKES_ER_CUTOFF * dmax);
  const double r2_tiny = (1e-8 * rho[0] * h) * (1e-8 * rho[0] * h);
  const int grid = static_cast<int>(ceil_div(M, 128));
  switch (mode) {
    case 1:
      deltas_kernel<1><<<grid, 128, 0, s>>>(sx, sn, sw, f, q, ty, tb, x0d, M, N, h, r3, rc2, r2_tiny, out_ud, out_vd);
      break;
    case 2:
      deltas_kernel<2><<<grid, 128, 0, s>>>(sx, sn, sw, f, q, ty, tb, x0d, M, N, h, r3, rc2, r2_tiny, out_ud, out_vd);
      break;
    default:
      deltas_kernel<3><<<grid, 128, 0, s>>>(sx, sn, sw, f, q, ty, tb, x0d, M, N, h, r3, rc2, r2_tiny, out_ud, out_vd);
  }
  return cudaGetLastError() == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}

int stokes_er_extrapolate(const double* tgt_b, int64_t M, double h, const double rho[3], const double* in_delta,
                          int C, double* out, void* stream) {
  if (M < 0 || M > INT32_MAX || !(h > 0.0) || !std::isfinite(h) || !rho_ok(rho) || C < 1 || C > 64)
    return STOKES_ER_EINVAL;
  if (!tgt_b || !in_delta || !out) return STOKES_ER_EINVAL;
  if (M == 0) return STOKES_ER_OK;
  const int st = check_arch();
  if (st) return st;
  Delta3 r3{{rho[0], rho[1], rho[2]}};
  extrapolate_kernel<<<ceil_div(M, 256), 256, 0, static_cast<cudaStream_t>(stream)>>>(tgt_b, M, h, r3, in_delta,
                                                                                       C, out);
  return cudaGetLastError() == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}

size_t stokes_er_nodes_workspace_bytes(int64_t N, int mode) {
  if (N < 1 || N > INT32_MAX || mode < 1 || mode > 3) return 0;
  return make_node_plan(N, mode).total;
}

size_t stokes_er_nodes_workspace_bytes_ex(int64_t N, int mode, const stokes_er_options* options) {
  if (N < 1 || N > INT32_MAX || mode < 1 || mode > 3) return 0;
  return make_node_plan(N, mode, opt_phases(options)).total;
}

int stokes_er_eval_nodes_ex(const double* src_xyz, const double* src_normal, const double* src_weight,
                            const double* f, const double* q, int64_t N, double h, const double rho[3], int mode,
                            double* out_u, double* out_v, void* workspace, size_t workspace_bytes, void* stream,
                            stokes_er_options* options) {
  int st = validate(src_xyz, src_normal, src_weight, f, q, src_xyz, src_xyz, src_xyz, N, N, h, rho, mode);
  if (st) return st;
  if (((mode & 1) && !out_u) || ((mode & 2) && !out_v)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  if (options && options->shard_count > 1 &&
      (options->shard_index < 0 || options->shard_index >= options->shard_count))
    return STOKES_ER_EINVAL;
  const NodePlan P = make_node_plan(N, mode, opt_phases(options));
  if (!workspace || workspace_bytes < P.total) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  switch (mode) {
    case 1: return run_nodes<1, false>(src_xyz, src_normal, src_weight, f, q, N, h, rho, out_u, out_v, ws, P, s, options);
    case 2: return run_nodes<2, false>(src_xyz, src_normal, src_weight, f, q, N, h, rho, out_u, out_v, ws, P, s, options);
    default: return run_nodes<3, false>(src_xyz, src_normal, src_weight, f, q, N, h, rho, out_u, out_v, ws, P, s, options);
  }
}

int stokes_er_eval_nodes_onsurface(const double* src_xyz, const double* src_normal, const double* src_weight,
                                   const double* f, const double* q, int64_t N, double delta, int mode, double* out_u,
                                   double* out_v, void* workspace, size_t workspace_bytes, void* stream) {
  const double one[3] = {1.0, 1.0, 1.0};  // delta_1 = delta_2 = delta_3 = delta; weights (1, 0, 0)
  int st = validate(src_xyz, src_normal, src_weight, f, q, src_xyz, src_xyz, src_xyz, N, N, delta, one, mode, false);
  if (st) return st;
  if (((mode & 1) && !out_u) || ((mode & 2) && !out_v)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  const NodePlan P = make_node_plan(N, mode);
  if (!workspace || workspace_bytes < P.total) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  switch (mode) {
    case 1: return run_nodes<1, true>(src_xyz, src_normal, src_weight, f, q, N, delta, one, out_u, out_v, ws, P, s, nullptr);
    case 2: return run_nodes<2, true>(src_xyz, src_normal, src_weight, f, q, N, delta, one, out_u, out_v, ws, P, s, nullptr);
    default: return run_nodes<3, true>(src_xyz, src_normal, src_weight, f, q, N, delta, one, out_u, out_v, ws, P, s, nullptr);
  }
}

int stokes_er_eval_nodes(const double* src_xyz, const double* src_normal, const double* src_weight, const double* f,
                         const double* q, int64_t N, double h, const double rho[3], int mode, double* out_u,
                         double* out_v, void* workspace, size_t workspace_bytes, void* stream) {
  return stokes_er_eval_nodes_ex(src_xyz, src_normal, src_weight, f, q, N, h, rho, mode, out_u, out_v, workspace,
                                 workspace_bytes, stream, nullptr);
}

size_t stokes_er_nodes_host_workspace_bytes(int64_t N, int mode) {
  const size_t w = stokes_er_nodes_workspace_bytes(N, mode);
  return w ? align_up(w) + node_host_stage_bytes(N) : 0;
}

int stokes_er_eval_nodes_host(const double* sx, const double* sn, const double* sw, const double* f, const double* q,
                              int64_t N, double h, const double rho[3], int mode, double* out_u, double* out_v,
                              void* workspace, size_t workspace_bytes, void* stream) {
  int st = validate(sx, sn, sw, f, q, sx, sx, sx, N, N, h, rho, mode);
  if (st) return st;
  if (((mode & 1) && !out_u) || ((mode & 2) && !out_v)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  const size_t wbytes = align_up(stokes_er_nodes_workspace_bytes(N, mode));
  if (!workspace || workspace_bytes < wbytes + node_host_stage_bytes(N)) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* stage = static_cast<char*>(workspace) + wbytes;
  double* dsx = reinterpret_cast<double*>(stage);
  double *dsn = dsx + 3 * N, *dsw = dsn + 3 * N, *df = dsw + N, *dq = df + 3 * N;
  double* du = reinterpret_cast<double*>(stage + align_up(13 * N * sizeof(double)));
  double* dv = du + 3 * N;
  auto h2d = [&](double* dst, const double* src, int64_t n) {
    return src ? cudaMemcpyAsync(dst, src, n * sizeof(double), cudaMemcpyHostToDevice, s) : cudaSuccess;
  };
  if (h2d(dsx, sx, 3 * N) || h2d(dsn, sn, 3 * N) || h2d(dsw, sw, N) || h2d(df, (mode & 1) ? f : nullptr, 3 * N) ||
      h2d(dq, (mode & 2) ? q : nullptr, 3 * N))
    return STOKES_ER_ECUDA;
  st = stokes_er_eval_nodes_ex(dsx, dsn, dsw, (mode & 1) ? df : nullptr, (mode & 2) ? dq : nullptr, N, h, rho, mode,
                               (mode & 1) ? du : nullptr, (mode & 2) ? dv : nullptr, workspace, wbytes, stream,
                               nullptr);
  if (st) return st;
  if ((mode & 1) && cudaMemcpyAsync(out_u, du, 3 * N * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  if ((mode & 2) && cudaMemcpyAsync(out_v, dv, 3 * N * sizeof(double), cudaMemcpyDeviceToHost, s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  return cudaStreamSynchronize(s) == cudaSuccess ? STOKES_ER_OK : STOKES_ER_ECUDA;
}

int stokes_er_nodes_pair_counts(int64_t N, int mode, double h, const double rho[3], void* workspace,
                                size_t workspace_bytes, int64_t* counts_host, void* stream) {
  if (N < 1 || N > INT32_MAX || mode < 1 || mode > 3 || !(h > 0.0) || !std::isfinite(h) || !rho_ok(rho) ||
      !counts_host)
    return STOKES_ER_EINVAL;
  int st = check_arch();
  if (st) return st;
  const NodePlan P = make_node_plan(N, mode);
  if (!workspace || workspace_bytes < P.total) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  unsigned long long* d = reinterpret_cast<unsigned long long*>(ws + P.off_counter + 2 * sizeof(int) + 8);
  const double dmax = rho[2] * h;
  const double rc2 = (STOKES_ER_CUTOFF * dmax) * (STOKES_ER_CUTOFF * dmax);
  if (cudaMemsetAsync(d, 0, sizeof(unsigned long long), s) != cudaSuccess) return STOKES_ER_ECUDA;
  sym_pair_count<<<ceil_div(P.nb, 128), 128, 0, s>>>(reinterpret_cast<const double*>(ws + P.off_blkbox), P.nb, N,
                                                     rc2 * (1.0 + 1e-9), d);
  unsigned long long c = 0;
  if (cudaMemcpyAsync(&c, d, sizeof(c), cudaMemcpyDeviceToHost, s) != cudaSuccess ||
      cudaStreamSynchronize(s) != cudaSuccess)
    return STOKES_ER_ECUDA;
  counts_host[0] = static_cast<int64_t>(c);
  counts_host[1] = N * N - static_cast<int64_t>(c);
  return STOKES_ER_OK;
}

int stokes_er_nodes_launch_count(int64_t N, int mode) {
  (void)mode;
  // bbox, morton, pack_sources, pack_node_soa, block_boxes, sym_kernel, nbr_kernel, finalize_nodes
  // (+ the CUB radix sort's own launches, library code)
  return N > 0 ? 8 : 0;
}

int stokes_er_launch_count(int64_t M, int64_t N, int mode) {
  (void)mode;
  // bbox, 2x morton, pack sources, pack targets, fused far+near, finalize: our
  // kernels (default schedule; STOKES_ER_SCHEDULE_SEPARATE adds one).  The two
  // CUB radix sorts add their own launches (library code).  Small problems (N, M <=
  // 8192): small_rank, pack_both, fused far+near, finalize (no CUB launches).
  if (M <= 0) return 0;
  return small_problem(M, N) ? 4 : 7;
}

const char* stokes_er_status_string(int status) {
  switch (status) {
    case STOKES_ER_OK: return "ok";
    case STOKES_ER_EINVAL: return "invalid argument";
    case STOKES_ER_ECUDA: return "CUDA error";
    case STOKES_ER_EWORKSPACE: return "workspace too small";
    case STOKES_ER_EARCH: return "device is not sm_100 (B200)";
    case STOKES_ER_ENOCONV: return "GMRES reached max_iter above the tolerance";
    default: return "unknown status";
  }
}

int stokes_er_abi_version(void) { return STOKES_ER_ABI_VERSION; }


size_t stokes_er_tree_plan_bytes(int64_t N, const stokes_er_tree_params* params) {
  if (N < 1 || N > INT32_MAX || !tree_params_ok(params)) return 0;
  return tree_plan_bytes(N, params->leaf_size);
}

int stokes_er_tree_build(const double* src_xyz_host, int64_t N, const stokes_er_tree_params* params, void* plan,
                         size_t plan_bytes) {
  if (!src_xyz_host || N < 1 || N > INT32_MAX || !tree_params_ok(params) || !plan) return STOKES_ER_EINVAL;
  if (plan_bytes < tree_plan_bytes(N, params->leaf_size)) return STOKES_ER_EWORKSPACE;
  for (int64_t j = 0; j < 3 * N; ++j)
    if (!std::isfinite(src_xyz_host[j])) return STOKES_ER_EINVAL;  // the midpoint splits need finite nodes
  TreeBuilder b;
  b.x = src_xyz_host;
  b.N = N;
  b.N0 = params->leaf_size;
  b.max_nodes = tree_max_nodes(N, params->leaf_size);
  b.idx.resize(N);
  b.tmp.resize(N);
  for (int64_t j = 0; j < N; ++j) b.idx[j] = static_cast<int32_t>(j);
  TreeNode root{};
  root.begin = 0;
  root.end = static_cast<int32_t>(N);
  b.tight_box(root);
  for (int d = 0; d < 3; ++d)
    if (!std::isfinite(root.lo[d]) || !std::isfinite(root.hi[d])) return STOKES_ER_EINVAL;
  b.nodes.reserve(1024);
  b.nodes.push_back(root);
  if (!b.split(0, 0)) return STOKES_ER_EINVAL;  // too many nodes or too deep
  char* out = static_cast<char*>(plan);
  TreePlanHeader hdr{};
  hdr.magic = kTreeMagic;
  hdr.N = N;
  hdr.nnodes = static_cast<int32_t>(b.nodes.size());
  hdr.max_nodes = static_cast<int32_t>(b.max_nodes);
  hdr.leaf_size = params->leaf_size;
  hdr.depth = b.depth;
  hdr.off_nodes = 64;
  hdr.off_perm = 64 + (int64_t)b.nodes.size() * (int64_t)sizeof(TreeNode);
  std::memcpy(out, &hdr, sizeof(hdr));
  std::memcpy(out + hdr.off_nodes, b.nodes.data(), b.nodes.size() * sizeof(TreeNode));
  std::memcpy(out + hdr.off_perm, b.idx.data(), (size_t)N * sizeof(int32_t));
  return STOKES_ER_OK;
}

int stokes_er_tree_info(const void* plan, int64_t N, int64_t* out_nodes, int64_t* out_depth) {
  const TreePlanHeader* h = tree_header(plan, N);
  if (!h) return STOKES_ER_EINVAL;
  if (out_nodes) *out_nodes = h->nnodes;
  if (out_depth) *out_depth = h->depth;
  return STOKES_ER_OK;
}

size_t stokes_er_tree_workspace_bytes(int64_t M, int64_t N, int mode, const stokes_er_tree_params* params,
                                      const void* plan) {
  if (M < 0 || N < 1 || mode < 1 || mode > 3 || !tree_params_ok(params)) return 0;
  const TreePlanHeader* h = tree_header(plan, N);
  if (!h) return 0;
  const Plan P = make_plan(M, N, mode, 1, 0);
  return tree_ws_layout(P, h->nnodes, N, params->degree).total;
}

static int eval_tree_common(const double* src_xyz, const double* src_normal, const double* src_weight,
                            const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                            const double* tgt_x0_density, int64_t M, int64_t N, double h, const double rho[3],
                            int mode, const stokes_er_tree_params* params, const void* plan, double* out_u,
                            double* out_v, void* workspace, size_t workspace_bytes, void* stream, bool sharp) {
  int st = validate(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, mode,
                    !sharp);
  if (st) return st;
  if (!tree_params_ok(params)) return STOKES_ER_EINVAL;
  const TreePlanHeader* hdr = tree_header(plan, N);
  if (!hdr) return STOKES_ER_EINVAL;
  if (M == 0) return STOKES_ER_OK;
  if (((mode & 1) && !out_u) || ((mode & 2) && !out_v)) return STOKES_ER_EINVAL;
  if ((st = check_arch())) return st;
  const Plan P = make_plan(M, N, mode, 1, 0);
  const TreeWs W = tree_ws_layout(P, hdr->nnodes, N, params->degree);
  if (!workspace || workspace_bytes < W.total) return STOKES_ER_EWORKSPACE;
  cudaStream_t s = static_cast<cudaStream_t>(stream);
  char* ws = static_cast<char*>(workspace);
  const char* pl = static_cast<const char*>(plan);
#define SER_TREE_RUN(M_, S_)                                                                                    \
  run_eval_tree<M_, S_>(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, params, \
                        hdr, pl, out_u, out_v, ws, P, W, s)
  if (sharp) {
    switch (mode) {
      case 1: return SER_TREE_RUN(1, true);
      case 2: return SER_TREE_RUN(2, true);
      default: return SER_TREE_RUN(3, true);
    }
  }
  switch (mode) {
    case 1: return SER_TREE_RUN(1, false);
    case 2: return SER_TREE_RUN(2, false);
    default: return SER_TREE_RUN(3, false);
  }
#undef SER_TREE_RUN
}

int stokes_er_eval_tree(const double* src_xyz, const double* src_normal, const double* src_weight, const double* f,
                        const double* q, const double* tgt_xyz, const double* tgt_b, const double* tgt_x0_density,
                        int64_t M, int64_t N, double h, const double rho[3], int mode,
                        const stokes_er_tree_params* params, const void* plan, double* out_u, double* out_v,
                        void* workspace, size_t workspace_bytes, void* stream) {
  return eval_tree_common(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, h, rho, mode,
                          params, plan, out_u, out_v, workspace, workspace_bytes, stream, false);
}

int stokes_er_eval_tree_onsurface(const double* src_xyz, const double* src_normal, const double* src_weight,
                                  const double* f, const double* q, const double* tgt_xyz, const double* tgt_b,
                                  const double* tgt_x0_density, int64_t M, int64_t N, double delta, int mode,
                                  const stokes_er_tree_params* params, const void* plan, double* out_u,
                                  double* out_v, void* workspace, size_t workspace_bytes, void* stream) {
  const double one[3] = {1.0, 1.0, 1.0};  // delta_1 = delta_2 = delta_3 = delta; weights (1, 0, 0)
  return eval_tree_common(src_xyz, src_normal, src_weight, f, q, tgt_xyz, tgt_b, tgt_x0_density, M, N, delta, one,
                          mode, params, plan, out_u, out_v, workspace, workspace_bytes, stream, true);
}

}  // extern "C"
