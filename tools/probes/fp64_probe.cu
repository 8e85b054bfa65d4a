// Microbenchmark probe: FP64 DFMA throughput per SM and rsqrt.approx.f64 accuracy on sm_100a.
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void dfma_loop(double* out, int iters, double a, double b) {
  double x0 = threadIdx.x * 1e-3, x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
  double x4 = x0 + 4, x5 = x0 + 5, x6 = x0 + 6, x7 = x0 + 7;
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int k = 0; k < 16; ++k) {
      x0 = fma(x0, a, b); x1 = fma(x1, a, b); x2 = fma(x2, a, b); x3 = fma(x3, a, b);
      x4 = fma(x4, a, b); x5 = fma(x5, a, b); x6 = fma(x6, a, b); x7 = fma(x7, a, b);
    }
  }
  out[blockIdx.x * blockDim.x + threadIdx.x] = x0 + x1 + x2 + x3 + x4 + x5 + x6 + x7;
}

__global__ void rsq_probe(const double* in, double* out_approx, double* out_full, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  double x = in[i], y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  out_approx[i] = y;
  out_full[i] = rsqrt(x);
}

int main() {
  int dev = 0; cudaDeviceProp p; cudaGetDeviceProperties(&p, dev);
  int clk = 0; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, dev);
  printf("name=%s sms=%d cc=%d.%d clock_khz=%d\n", p.name, p.multiProcessorCount, p.major, p.minor, clk);
  double* out; cudaMalloc(&out, 1 << 24);
  int blocks = p.multiProcessorCount * 8, threads = 256, iters = 4096;
  dfma_loop<<<blocks, threads>>>(out, 64, 0.999999, 1e-7);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(e0);
    dfma_loop<<<blocks, threads>>>(out, iters, 0.999999, 1e-7);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double flops = 2.0 * 8 * 16 * (double)iters * blocks * threads;
    printf("dfma: %.3f ms  %.2f TFLOP/s  per-SM-per-clk(at %d MHz)=%.1f FMA\n", ms, flops / ms / 1e9,
           clk / 1000, flops / 2 / (ms * 1e-3) / p.multiProcessorCount / (clk * 1e3));
  }
  // rsqrt.approx.f64 accuracy
  int n = 1 << 20; double *h = new double[n], *ha = new double[n], *hf = new double[n];
  for (int i = 0; i < n; ++i) h[i] = std::ldexp(1.0 + (double)i / n, (i % 41) - 20);
  double *din, *da, *df; cudaMalloc(&din, n * 8); cudaMalloc(&da, n * 8); cudaMalloc(&df, n * 8);
  cudaMemcpy(din, h, n * 8, cudaMemcpyHostToDevice);
  rsq_probe<<<(n + 255) / 256, 256>>>(din, da, df, n);
  cudaMemcpy(ha, da, n * 8, cudaMemcpyDeviceToHost); cudaMemcpy(hf, df, n * 8, cudaMemcpyDeviceToHost);
  double ea = 0, ef = 0;
  for (int i = 0; i < n; ++i) {
    long double ref = 1.0L / sqrtl((long double)h[i]);
    double ra = fabs((double)((ha[i] - ref) / ref)), rf = fabs((double)((hf[i] - ref) / ref));
    if (ra > ea) ea = ra; if (rf > ef) ef = rf;
  }
  printf("rsqrt.approx.f64 max rel err = %.3e (log2 %.2f); rsqrt() max rel err = %.3e\n", ea, log2(ea), ef);
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
