// Probe: independent FP64 instruction mixes (DFMA:DMUL:DADD) and dependent chains.
#include <cstdio>
#include <cuda_runtime.h>
template <int KIND>
__global__ void k(double* out, int iters, double s) {
  double a[8], b[8];
  for (int i = 0; i < 8; ++i) { a[i] = 1.0 + threadIdx.x * 1e-3 + i; b[i] = 0.999 + i * 1e-6 + s; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int r = 0; r < 8; ++r) {
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        if (KIND == 0) { if (r < 4) a[i] = fma(a[i], b[i], s); else if (r < 6) a[i] = a[i] * b[i]; else a[i] = a[i] + b[i]; }
        if (KIND == 1) { if (r < 4) a[i] = fma(a[i], b[i], s); else if (r < 6) a[i] = a[i] * b[(i+1)&7]; else a[i] = a[i] - b[(i+3)&7]; }
      }
    }
  }
  double t = 0; for (int i = 0; i < 8; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
// dependent chains: only C independent chains per thread
template <int C>
__global__ void kd(double* out, int iters, double s) {
  double a[C];
  for (int i = 0; i < C; ++i) a[i] = 1.0 + threadIdx.x * 1e-3 + i;
  for (int it = 0; it < iters; ++it)
#pragma unroll
    for (int r = 0; r < 64 / C; ++r)
#pragma unroll
      for (int i = 0; i < C; ++i) a[i] = fma(a[i], 0.9999999, s);
  double t = 0; for (int i = 0; i < C; ++i) t += a[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <typename F> void timeit(F f, int sms, int blocks, int threads, double n_per_thread, const char* name) {
  f(10);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); f(2000); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  printf("%-28s %.1f FP64 lane-instr/clk/SM at 1965 MHz\n", name, 2000 * n_per_thread * blocks * threads / (ms * 1e-3) / sms / 1.965e9);
}
int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  int sms = p.multiProcessorCount;
  double* out; cudaMalloc(&out, 1 << 24);
  timeit([&](int it) { k<0><<<sms * 4, 256>>>(out, it, 0.5); }, sms, sms * 4, 256, 64, "mix 4:2:2 self-operand");
  timeit([&](int it) { k<1><<<sms * 4, 256>>>(out, it, 0.5); }, sms, sms * 4, 256, 64, "mix 4:2:2 3-distinct");
  for (int w : {4, 8, 16}) {
    char name[64];
    snprintf(name, 64, "chain C=1 warps/SMSP=%d", w);
    timeit([&](int it) { kd<1><<<sms, 128 * w / 4 * 4>>>(out, it, 0.5); }, sms, sms, 128 * w / 4 * 4, 64, name);
    snprintf(name, 64, "chain C=2 warps/SMSP=%d", w);
    timeit([&](int it) { kd<2><<<sms, 128 * w / 4 * 4>>>(out, it, 0.5); }, sms, sms, 128 * w / 4 * 4, 64, name);
    snprintf(name, 64, "chain C=4 warps/SMSP=%d", w);
    timeit([&](int it) { kd<4><<<sms, 128 * w / 4 * 4>>>(out, it, 0.5); }, sms, sms, 128 * w / 4 * 4, 64, name);
  }
  return 0;
}
