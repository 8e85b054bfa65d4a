// Probe: the far-pair instruction mix alone (sources from registers/SMEM broadcast, no TMA,
// no barriers, no box tests) to find the achievable FP64 pipe rate of far_pair<3>.
#include <cstdio>
#include <cuda_runtime.h>
#include "../../paper_2507_00156_b200/csrc/device_math.cuh"
struct Src { double x, y, z, mx, my, mz, fx, fy, fz, qx, qy, qz; };
struct Tgt { double y0, y1, y2, alpha, q0, q1, q2; };
struct Acc { double u0, u1, u2, v0, v1, v2; };
template <int V>
__device__ __forceinline__ void far_pair(const Src& s, const Tgt& t, Acc& a) {
  const double dx = t.y0 - s.x, dy = t.y1 - s.y, dz = t.y2 - s.z;
  const double r2 = fma(dx, dx, fma(dy, dy, dz * dz));
  double ri;
  if (V == 0) ri = ser::rsqrt_nr(r2);
  else if (V == 1) { const double y = r2 * 0.999; const double e = fma(-r2, y * y, 1.0); const double p = fma(e, 0.375, 0.5); ri = fma(y * e, p, y); }  // same FP64 ops, no MUFU
  else if (V == 2) ri = rsqrt(r2);
  else ri = r2;  // V >= 3: no rsqrt / Newton block
  const double ri2 = ri * ri;
  if (V != 5) {
  const double gx = fma(-t.alpha, s.mx, s.fx), gy = fma(-t.alpha, s.my, s.fy), gz = fma(-t.alpha, s.mz, s.fz);
  const double a3 = fma(dx, gx, fma(dy, gy, dz * gz)) * ri2;
  a.u0 = fma(fma(dx, a3, gx), ri, a.u0);
  a.u1 = fma(fma(dy, a3, gy), ri, a.u1);
  a.u2 = fma(fma(dz, a3, gz), ri, a.u2);
  }
  if (V == 4) return;
  const double qx = s.qx - t.q0, qy = s.qy - t.q1, qz = s.qz - t.q2;
  const double dq = fma(dx, qx, fma(dy, qy, dz * qz));
  const double dm = fma(dx, s.mx, fma(dy, s.my, dz * s.mz));
  const double c = (dq * dm) * (ri2 * ri2 * ri);
  a.v0 = fma(dx, c, a.v0);
  a.v1 = fma(dy, c, a.v1);
  a.v2 = fma(dz, c, a.v2);
}
template <int T, int U, int V>
__global__ void __launch_bounds__(128) k(const double* __restrict__ src, int nsrc, double* out) {
  __shared__ double sm[256 * 12];
  for (int i = threadIdx.x; i < 256 * 12; i += blockDim.x) sm[i] = src[i];
  __syncthreads();
  Tgt tg[T]; Acc acc[T];
  for (int j = 0; j < T; ++j) {
    double b = 0.37 + 0.01 * threadIdx.x + j;
    tg[j] = Tgt{b, 2 * b, -b, 0.3, 0.1, 0.2, 0.3};
    acc[j] = Acc{0, 0, 0, 0, 0, 0};
  }
  for (int rep = 0; rep < nsrc / 256; ++rep) {
#pragma unroll U
    for (int k2 = 0; k2 < 256; ++k2) {
      const double2* p = reinterpret_cast<const double2*>(sm + k2 * 12);
      double2 a = p[0], b = p[1], c = p[2], d = p[3], e = p[4], f = p[5];
      Src s{a.x, a.y, b.x, b.y, c.x, c.y, d.x, d.y, e.x, e.y, f.x, f.y};
#pragma unroll
      for (int j = 0; j < T; ++j) far_pair<V>(s, tg[j], acc[j]);
    }
  }
  double t = 0;
  for (int j = 0; j < T; ++j) t += acc[j].u0 + acc[j].u1 + acc[j].u2 + acc[j].v0 + acc[j].v1 + acc[j].v2;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int T, int U, int V> void run(const double* src, double* out, int sms, int ctas_per_sm) {
  int blocks = sms * ctas_per_sm, nsrc = 256 * 64;
  k<T, U, V><<<blocks, 128>>>(src, 256, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); k<T, U, V><<<blocks, 128>>>(src, nsrc, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double pairs = (double)nsrc * T * 128 * blocks;
  printf("V=%d T=%d U=%d ctas/SM=%d: %.3e pairs/s  FP64 pipe %.1f%% (41 instr/pair at 1965 MHz)\n", V, T, U, ctas_per_sm,
         pairs / ms * 1e3, 100.0 * pairs * 41 / (ms * 1e-3) / sms / 64 / 1.965e9);
}

// software-pipelined variant: geometry + rsqrt of source k+1 overlap the accumulation of source k
struct Geo { double dx, dy, dz, ri; };
__device__ __forceinline__ Geo geo(const Src& s, const Tgt& t) {
  Geo g; g.dx = t.y0 - s.x; g.dy = t.y1 - s.y; g.dz = t.y2 - s.z;
  const double r2 = fma(g.dx, g.dx, fma(g.dy, g.dy, g.dz * g.dz));
  g.ri = ser::rsqrt_nr(r2);
  return g;
}
__device__ __forceinline__ void acc_pair(const Src& s, const Tgt& t, const Geo& g, Acc& a) {
  const double dx = g.dx, dy = g.dy, dz = g.dz, ri = g.ri, ri2 = ri * ri;
  const double gx = fma(-t.alpha, s.mx, s.fx), gy = fma(-t.alpha, s.my, s.fy), gz = fma(-t.alpha, s.mz, s.fz);
  const double a3 = fma(dx, gx, fma(dy, gy, dz * gz)) * ri2;
  a.u0 = fma(fma(dx, a3, gx), ri, a.u0);
  a.u1 = fma(fma(dy, a3, gy), ri, a.u1);
  a.u2 = fma(fma(dz, a3, gz), ri, a.u2);
  const double qx = s.qx - t.q0, qy = s.qy - t.q1, qz = s.qz - t.q2;
  const double dq = fma(dx, qx, fma(dy, qy, dz * qz));
  const double dm = fma(dx, s.mx, fma(dy, s.my, dz * s.mz));
  const double c = (dq * dm) * (ri2 * ri2 * ri);
  a.v0 = fma(dx, c, a.v0);
  a.v1 = fma(dy, c, a.v1);
  a.v2 = fma(dz, c, a.v2);
}
__device__ __forceinline__ Src lds(const double* sm, int k) {
  const double2* p = reinterpret_cast<const double2*>(sm + k * 12);
  double2 a = p[0], b = p[1], c = p[2], d = p[3], e = p[4], f = p[5];
  return Src{a.x, a.y, b.x, b.y, c.x, c.y, d.x, d.y, e.x, e.y, f.x, f.y};
}
template <int T, int U>
__global__ void __launch_bounds__(128) kp(const double* __restrict__ src, int nsrc, double* out) {
  __shared__ double sm[256 * 12];
  for (int i = threadIdx.x; i < 256 * 12; i += blockDim.x) sm[i] = src[i];
  __syncthreads();
  Tgt tg[T]; Acc acc[T];
  for (int j = 0; j < T; ++j) {
    double b = 0.37 + 0.01 * threadIdx.x + j;
    tg[j] = Tgt{b, 2 * b, -b, 0.3, 0.1, 0.2, 0.3};
    acc[j] = Acc{0, 0, 0, 0, 0, 0};
  }
  for (int rep = 0; rep < nsrc / 256; ++rep) {
    Src s = lds(sm, 0);
    Geo g[T];
#pragma unroll
    for (int j = 0; j < T; ++j) g[j] = geo(s, tg[j]);
#pragma unroll U
    for (int k2 = 0; k2 < 256; ++k2) {
      const Src sn = lds(sm, (k2 + 1) & 255);
      Geo gn[T];
#pragma unroll
      for (int j = 0; j < T; ++j) gn[j] = geo(sn, tg[j]);
#pragma unroll
      for (int j = 0; j < T; ++j) acc_pair(s, tg[j], g[j], acc[j]);
      s = sn;
#pragma unroll
      for (int j = 0; j < T; ++j) g[j] = gn[j];
    }
  }
  double t = 0;
  for (int j = 0; j < T; ++j) t += acc[j].u0 + acc[j].u1 + acc[j].u2 + acc[j].v0 + acc[j].v1 + acc[j].v2;
  out[blockIdx.x * blockDim.x + threadIdx.x] = t;
}
template <int T, int U> void runp(const double* src, double* out, int sms, int ctas_per_sm) {
  int blocks = sms * ctas_per_sm, nsrc = 256 * 64;
  kp<T, U><<<blocks, 128>>>(src, 256, out);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0); kp<T, U><<<blocks, 128>>>(src, nsrc, out); cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double pairs = (double)nsrc * T * 128 * blocks;
  printf("pipelined T=%d U=%d ctas/SM=%d: %.3e pairs/s  FP64 pipe %.1f%% (41 instr/pair at 1965 MHz)\n", T, U, ctas_per_sm,
         pairs / ms * 1e3, 100.0 * pairs * 41 / (ms * 1e-3) / sms / 64 / 1.965e9);
}

int main() {
  cudaDeviceProp p; cudaGetDeviceProperties(&p, 0);
  double h[256 * 12];
  for (int i = 0; i < 256 * 12; ++i) h[i] = 0.5 + 0.001 * i;
  double *src, *out; cudaMalloc(&src, sizeof(h)); cudaMalloc(&out, 1 << 24);
  cudaMemcpy(src, h, sizeof(h), cudaMemcpyHostToDevice);
  run<2, 4, 0>(src, out, p.multiProcessorCount, 4);
  runp<2, 2>(src, out, p.multiProcessorCount, 4);
  runp<2, 4>(src, out, p.multiProcessorCount, 4);
  runp<2, 2>(src, out, p.multiProcessorCount, 3);
  runp<1, 4>(src, out, p.multiProcessorCount, 6);
  return 0;
}
