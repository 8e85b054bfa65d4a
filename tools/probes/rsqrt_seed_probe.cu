// Accuracy of the MUFU.RSQ64H seed (rsqrt.approx.ftz.f64) and of one quadratic / cubic Newton step
// from it, over r^2 in [1e-8, 16] (log-uniform): max |y sqrt(x) - 1| and the mean signed error.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o rsqrt_seed_probe rsqrt_seed_probe.cu
#include <cstdio>
#include <cmath>
#include <cuda_runtime.h>

__global__ void probe(int n, double* out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  // log-uniform x from a counter hash
  unsigned long long h = (unsigned long long)i * 0x9E3779B97F4A7C15ull;
  h ^= h >> 31; h *= 0xBF58476D1CE4E5B9ull; h ^= h >> 27;
  const double u = (double)(h >> 11) * (1.0 / 9007199254740992.0);
  const double x = exp(log(1e-8) + u * (log(16.0) - log(1e-8)));
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  const double e = fma(-x, y * y, 1.0);
  const double yq = fma(y * e, 0.5, y);
  const double yc = fma(y * e, fma(e, 0.375, 0.5), y);
  const double ref = 1.0 / sqrt(x);  // IEEE sqrt and division: within 1 ulp
  out[4 * i + 0] = (y - ref) / ref;
  out[4 * i + 1] = (yq - ref) / ref;
  out[4 * i + 2] = (yc - ref) / ref;
  out[4 * i + 3] = x;
}

int main() {
  const int n = 1 << 24;
  double* d;
  cudaMalloc(&d, sizeof(double) * 4 * n);
  probe<<<(n + 255) / 256, 256>>>(n, d);
  double* hst = new double[4 * (size_t)n];
  cudaMemcpy(hst, d, sizeof(double) * 4 * n, cudaMemcpyDeviceToHost);
  const char* name[3] = {"seed", "quadratic", "cubic"};
  for (int k = 0; k < 3; ++k) {
    double mx = 0, mean = 0;
    for (int i = 0; i < n; ++i) {
      const double v = hst[4 * i + k];
      mx = fmax(mx, fabs(v));
      mean += v;
    }
    printf("%-9s max |rel err| %.3e  (2^%.1f)  mean signed %.3e\n", name[k], mx, log2(mx), mean / n);
  }
  return 0;
}
