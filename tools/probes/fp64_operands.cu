// Probe: FP64 issue rate vs number of distinct register operands per DFMA on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(double* out, int iters, double s) {
  double a[8], b[8], c[8];
  for (int i = 0; i < 8; ++i) { a[i] = threadIdx.x * 1e-3 + i; b[i] = 0.999 + i * 1e-6; c[i] = 1e-7 * i + s; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (KIND == 0) a[i] = fma(a[i], b[0], c[0]);            // 2 operands shared (reuse)
        if (KIND == 1) a[i] = fma(a[i], b[i], c[0]);            // 1 shared
        if (KIND == 2) a[i] = fma(a[i], b[i], c[i]);            // 3 distinct
        if (KIND == 3) { a[i] = fma(a[i], b[i], c[i]); c[i] = fma(c[i], b[i], a[i]); }  // 3 distinct, mixed
      }
    }
  }
  double t = 0; for (int i = 0; i < 8; ++i) t += a[i] + c[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int KIND> void run(double* out, int sms) {
  int blocks = sms * 4, threads = 256, iters = 2000;
  k<KIND><<<blocks, threads>>>(out, 10, 0.5);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<KIND><<<blocks, threads>>>(out, iters, 0.5); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double n = (double)iters * 64 * (KIND == 3 ? 2 : 1) * blocks * threads;
  printf("kind %d: %.2f TFLOP/s (%.1f DFMA/clk/SM at 1965 MHz)\n", KIND, 2 * n / ms / 1e9, n / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double* out; cudaMalloc(&out, 1 << 24);
  run<0>(out, p.multiProcessorCount); run<1>(out, p.multiProcessorCount); run<2>(out, p.multiProcessorCount); run<3>(out, p.multiProcessorCount);
  return 0;
}
