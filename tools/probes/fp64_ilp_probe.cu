// Probe: FP64 DFMA issue rate vs independent chains per warp (K) and warps per SM (W) on sm_100a,
// to size the instruction-level parallelism the FP64-bound kernels need.
#include <cstdio>
#include <cuda_runtime.h>

template <int K>
__global__ void chains(double* out, int iters, double a, double b) {
  double x[K];
#pragma unroll
  for (int k = 0; k < K; ++k) x[k] = threadIdx.x * 1e-3 + k;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int r = 0; r < 32; ++r)
#pragma unroll
      for (int k = 0; k < K; ++k) x[k] = fma(x[k], a, b);
  }
  double s = 0;
#pragma unroll
  for (int k = 0; k < K; ++k) s += x[k];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

template <int K>
void run(double* out, int sms, int clk_khz) {
  for (int W : {4, 8, 12, 16}) {
    const int iters = 2048 / K;
    chains<K><<<sms, 32 * W>>>(out, 16, 0.999999, 1e-7);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    cudaEventRecord(e0);
    chains<K><<<sms, 32 * W>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    const double fmas = 32.0 * K * (double)iters * sms * 32 * W;
    const double per_clk = fmas / (ms * 1e-3) / sms / (clk_khz * 1e3);
    const double cyc_per_dep = (ms * 1e-3) * clk_khz * 1e3 / (32.0 * iters);  // cycles per dependent step
    printf("K=%d W=%2d warps/SM: %.1f FMA/clk/SM (%.0f%% of 64)  %.1f cycles per dependent DFMA step\n", K, W,
           per_clk, 100.0 * per_clk / 64.0, cyc_per_dep);
  }
}

int main() {
  cudaDeviceProp p;
  cudaGetDeviceProperties(&p, 0);
  int clk = 0;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("%s sms=%d clock_khz=%d\n", p.name, p.multiProcessorCount, clk);
  double* out;
  cudaMalloc(&out, 1 << 24);
  run<1>(out, p.multiProcessorCount, clk);
  run<2>(out, p.multiProcessorCount, clk);
  run<4>(out, p.multiProcessorCount, clk);
  run<8>(out, p.multiProcessorCount, clk);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
