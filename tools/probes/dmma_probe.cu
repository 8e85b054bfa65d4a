// Microbenchmark probe: FP64 tensor-core (DMMA, mma.sync .f64) throughput on
// sm_100a, alone and concurrently with DFMA, to decide whether the far-field
// pair sum's bilinear parts (dot products, accumulations) can move to the
// tensor pipe while the vector FP64 pipe does the rsqrt / per-pair scalars.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o dmma_probe dmma_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

// m8n8k4 f64: A 8x4 (1 double / lane), B 4x8 (1 / lane), C/D 8x8 (2 / lane)
__device__ __forceinline__ void mma884(double& c0, double& c1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c0), "+d"(c1) : "d"(a), "d"(b));
}
#ifdef WITH_M16
// m16n8k4 f64 (sm_90+): A 16x4 (2 / lane), B 4x8 (1), C 16x8 (4)
__device__ __forceinline__ void mma1684(double* c, double a0, double a1, double b) {
  asm volatile("mma.sync.aligned.m16n8k4.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5}, {%6}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3]) : "d"(a0), "d"(a1), "d"(b));
}
// m16n8k16 f64: A 16x16 (8 / lane), B 16x8 (4), C 16x8 (4)
__device__ __forceinline__ void mma16816(double* c, const double* a, const double* b) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f64.f64.f64.f64 {%0,%1,%2,%3}, {%4,%5,%6,%7,%8,%9,%10,%11}, "
               "{%12,%13,%14,%15}, {%0,%1,%2,%3};"
               : "+d"(c[0]), "+d"(c[1]), "+d"(c[2]), "+d"(c[3])
               : "d"(a[0]), "d"(a[1]), "d"(a[2]), "d"(a[3]), "d"(a[4]), "d"(a[5]), "d"(a[6]), "d"(a[7]),
                 "d"(b[0]), "d"(b[1]), "d"(b[2]), "d"(b[3]));
}
#endif

// DMMA-only: NA independent accumulators per warp
template <int NA>
__global__ void dmma_loop(double* out, int iters, double a, double b) {
  double c[NA][2];
#pragma unroll
  for (int k = 0; k < NA; ++k) { c[k][0] = threadIdx.x + k; c[k][1] = 1.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NA; ++k) mma884(c[k][0], c[k][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NA; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

#ifdef WITH_M16
template <int NA>
__global__ void dmma16816_loop(double* out, int iters, double a, double b) {
  double c[NA][4], av[8], bv[4];
#pragma unroll
  for (int k = 0; k < 8; ++k) av[k] = a + k * 1e-3;
#pragma unroll
  for (int k = 0; k < 4; ++k) bv[k] = b + k * 1e-3;
#pragma unroll
  for (int k = 0; k < NA; ++k) for (int j = 0; j < 4; ++j) c[k][j] = threadIdx.x + k + j;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < NA; ++k) mma16816(c[k], av, bv);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < NA; ++k) s += c[k][0] + c[k][1] + c[k][2] + c[k][3];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
#endif

// DFMA-only: 8 independent chains x 16 per iteration
__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x[8];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 16; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Same warp: per iteration ND x 8 DFMA and NM DMMA (independent)
template <int ND, int NM>
__global__ void mixed_loop(double* out, int iters, double a, double b) {
  double x[8], c[4][2];
#pragma unroll
  for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
#pragma unroll
  for (int k = 0; k < 4; ++k) { c[k][0] = k; c[k][1] = 1.0; }
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < ND; ++r)
#pragma unroll
      for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
#pragma unroll
    for (int m = 0; m < NM; ++m) mma884(c[m & 3][0], c[m & 3][1], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < 8; ++k) s += x[k];
#pragma unroll
  for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

// Warp-specialized: even warps DFMA, odd warps DMMA
__global__ void split_loop(double* out, int iters_d, int iters_m, double a, double b) {
  const int warp = threadIdx.x >> 5;
  double s = 0;
  if (warp & 1) {
    double c[4][2];
#pragma unroll
    for (int k = 0; k < 4; ++k) { c[k][0] = k; c[k][1] = 1.0; }
    for (int i = 0; i < iters_m; ++i) {
#pragma unroll
      for (int k = 0; k < 4; ++k) mma884(c[k][0], c[k][1], a, b);
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) s += c[k][0] + c[k][1];
  } else {
    double x[8];
#pragma unroll
    for (int k = 0; k < 8; ++k) x[k] = threadIdx.x * 1e-3 + k;
    for (int i = 0; i < iters_d; ++i) {
#pragma unroll
      for (int r = 0; r < 16; ++r)
#pragma unroll
        for (int k = 0; k < 8; ++k) x[k] = fma(x[k], a, b);
    }
#pragma unroll
    for (int k = 0; k < 8; ++k) s += x[k];
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

static int g_sms, g_clk;
static cudaEvent_t e0, e1;

template <typename F>
static float timeit(F launch) {
  launch();
  cudaDeviceSynchronize();
  float best = 1e30f;
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  return best;
}

static void report(const char* name, float ms, double dfma_lane, double dmma_fma) {
  const double clk = g_clk * 1e3 * 1e-3 * ms;  // cycles during the run
  printf("%-28s %8.3f ms  DFMA %6.2f TF (%5.1f lane-FMA/SM/clk)  DMMA %6.2f TF (%6.1f FMA/SM/clk)  sum %6.2f TF\n",
         name, ms, 2 * dfma_lane / ms / 1e9, dfma_lane / g_sms / clk, 2 * dmma_fma / ms / 1e9,
         dmma_fma / g_sms / clk, 2 * (dfma_lane + dmma_fma) / ms / 1e9);
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  g_sms = p.multiProcessorCount;
  cudaDeviceGetAttribute(&g_clk, cudaDevAttrClockRate, 0);
  printf("name=%s sms=%d cc=%d.%d clock_khz=%d\n", p.name, g_sms, p.major, p.minor, g_clk);
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  double* out;
  cudaMalloc(&out, 1 << 26);
  const int threads = 256;
  for (int bps : {4, 8}) {
    const int blocks = g_sms * bps;
    const double nthr = (double)blocks * threads, nwarp = nthr / 32;
    int it = 2048;
    float ms = timeit([&] { dfma_loop<<<blocks, threads>>>(out, it, 0.999999, 1e-7); });
    printf("-- %d blocks/SM x %d threads\n", bps, threads);
    report("dfma", ms, nthr * 128.0 * it, 0);
    int itm = 2048 * 8;
    ms = timeit([&] { dmma_loop<1><<<blocks, threads>>>(out, itm, 0.999999, 1e-7); });
    report("dmma884 x1 acc", ms, 0, nwarp * 256.0 * itm);
    ms = timeit([&] { dmma_loop<4><<<blocks, threads>>>(out, itm / 4, 0.999999, 1e-7); });
    report("dmma884 x4 acc", ms, 0, nwarp * 256.0 * itm);
    ms = timeit([&] { dmma_loop<8><<<blocks, threads>>>(out, itm / 8, 0.999999, 1e-7); });
    report("dmma884 x8 acc", ms, 0, nwarp * 256.0 * itm);
#ifdef WITH_M16
    ms = timeit([&] { dmma16816_loop<2><<<blocks, threads>>>(out, itm / 16, 0.999999, 1e-7); });
    report("dmma16816 x2 acc", ms, 0, nwarp * 2048.0 * 2 * (itm / 16));
#endif
    ms = timeit([&] { mixed_loop<2, 1><<<blocks, threads>>>(out, it * 4, 0.999999, 1e-7); });
    report("mixed 16 dfma : 1 dmma", ms, nthr * 16.0 * it * 4, nwarp * 256.0 * 1 * it * 4);
    ms = timeit([&] { mixed_loop<2, 2><<<blocks, threads>>>(out, it * 4, 0.999999, 1e-7); });
    report("mixed 16 dfma : 2 dmma", ms, nthr * 16.0 * it * 4, nwarp * 256.0 * 2 * it * 4);
    ms = timeit([&] { mixed_loop<2, 4><<<blocks, threads>>>(out, it * 4, 0.999999, 1e-7); });
    report("mixed 16 dfma : 4 dmma", ms, nthr * 16.0 * it * 4, nwarp * 256.0 * 4 * it * 4);
    ms = timeit([&] { mixed_loop<1, 4><<<blocks, threads>>>(out, it * 4, 0.999999, 1e-7); });
    report("mixed 8 dfma : 4 dmma", ms, nthr * 8.0 * it * 4, nwarp * 256.0 * 4 * it * 4);
    ms = timeit([&] { split_loop<<<blocks, threads>>>(out, it, itm / 4, 0.999999, 1e-7); });
    report("split warps dfma | dmma", ms, nthr / 2 * 128.0 * it, nwarp / 2 * 256.0 * itm);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
