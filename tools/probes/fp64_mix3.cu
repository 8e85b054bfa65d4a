// Probe: which FP64 op classes overlap (independent ops, 8 chains/thread, 8 warps/SMSP).
#include <cstdio>
#include <cuda_runtime.h>
// pattern bits over r = 0..7: 0 = DFMA, 1 = DMUL, 2 = DADD
template <int P0, int P1, int P2, int P3, int P4, int P5, int P6, int P7>
__global__ void k(double* out, int iters, double s) {
  double a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = 1.0 + threadIdx.x * 1e-3 + i; b[i] = 0.999 + i * 1e-6 + s; }
  constexpr int P[8] = {P0, P1, P2, P3, P4, P5, P6, P7};
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (P[r] == 0) a[i] = fma(a[i], b[i], s);
        if (P[r] == 1) a[i] = a[i] * b[i];
        if (P[r] == 2) a[i] = a[i] + b[i];
      }
    }
  }
  double t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <typename F> void timeit(F f, int sms, double n_per_thread, const char* name) {
  int blocks = sms * 4, threads = 256;
  f(10, blocks, threads);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); f(2000, blocks, threads); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-34s %.1f FP64 lane-instr/clk/SM at 1965 MHz\n", name, 2000 * n_per_thread * blocks * threads / (ms * 1e-3) / sms / 1.965e9);
}
#define RUN(name, ...) timeit([&](int it, int b, int t) { k<__VA_ARGS__><<<b, t>>>(out, it, 0.5); }, sms, 64, name)
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 1 << 24);
  RUN("DFMA only", 0, 0, 0, 0, 0, 0, 0, 0);
  RUN("DMUL only", 1, 1, 1, 1, 1, 1, 1, 1);
  RUN("DADD only", 2, 2, 2, 2, 2, 2, 2, 2);
  RUN("DFMA:DADD 1:1", 0, 2, 0, 2, 0, 2, 0, 2);
  RUN("DFMA:DMUL 1:1", 0, 1, 0, 1, 0, 1, 0, 1);
  RUN("DMUL:DADD 1:1", 1, 2, 1, 2, 1, 2, 1, 2);
  RUN("DFMA:DMUL:DADD 4:2:2", 0, 0, 0, 0, 1, 1, 2, 2);
  RUN("DFMA:DMUL:DADD 5:2:1", 0, 0, 0, 0, 0, 1, 1, 2);
  return 0;
}
