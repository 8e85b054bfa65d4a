// Probe: throughput of DMUL / DADD / MUFU.RSQ64H mixes vs DFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double rsq(double x) { double y; asm volatile("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x)); return y; }
template <int KIND>
__global__ void k(double* out, int iters, double s) {
  double a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = 1.0 + threadIdx.x * 1e-3 + i; b[i] = 0.999 + i * 1e-6 + s; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (KIND == 0) a[i] = a[i] * b[i];                 // DMUL
        if (KIND == 1) a[i] = a[i] + b[i];                 // DADD
        if (KIND == 2) a[i] = fma(a[i], b[i], s);          // DFMA
        if (KIND == 3) { a[i] = fma(a[i], b[i], s); if ((r & 7) == 0) a[i] = rsq(a[i]); }  // DFMA + 1/8 MUFU.RSQ64H
        if (KIND == 4) { a[i] = fma(a[i], b[i], s); if ((r & 3) == 0) a[i] = rsq(a[i]); }  // 1/4 MUFU
      }
    }
  }
  double t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int KIND> void run(double* out, int sms, const char* name) {
  int blocks = sms * 4, threads = 256, iters = 2000;
  k<KIND><<<blocks, threads>>>(out, 10, 0.5);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<KIND><<<blocks, threads>>>(out, iters, 0.5); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)iters * 64 * blocks * threads;  // FP64 instructions (lane)
  printf("%-22s %.1f FP64 lane-instr/clk/SM at 1965 MHz\n", name, n / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  run<0>(out, p.multiProcessorCount, "DMUL");
  run<1>(out, p.multiProcessorCount, "DADD");
  run<2>(out, p.multiProcessorCount, "DFMA");
  run<3>(out, p.multiProcessorCount, "DFMA+1/8 RSQ64H");
  run<4>(out, p.multiProcessorCount, "DFMA+1/4 RSQ64H");
  return 0;
}
