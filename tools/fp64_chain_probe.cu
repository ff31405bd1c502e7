// Probe: dependent fp64 chain latency through the ADDEND (acc = fma(x_i, w_i, acc)), as in the
// router, versus through the multiplicand; and DADD chains.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_addend(const double* in, double* out, long long* cyc, int n) {
  double x[8], w[8];
  for (int i = 0; i < 8; ++i) { x[i] = in[i]; w[i] = in[8 + i]; }
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < n; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = fma(x[i], w[i], acc);
  long long t1 = clock64();
  out[0] = acc;
  cyc[0] = t1 - t0;
}
__global__ void k_dadd(const double* in, double* out, long long* cyc, int n) {
  double p[8];
  for (int i = 0; i < 8; ++i) p[i] = in[i] * in[8 + i];
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < n; ++r)
#pragma unroll
    for (int i = 0; i < 8; ++i) acc = acc + p[i];
  long long t1 = clock64();
  out[1] = acc;
  cyc[1] = t1 - t0;
}
__global__ void k_mult(const double* in, double* out, long long* cyc, int n) {
  double a = in[0], b = 1.0000001, c = 0.5;
  long long t0 = clock64();
  for (int r = 0; r < n * 8; ++r) a = fma(a, b, c);
  long long t1 = clock64();
  out[2] = a;
  cyc[2] = t1 - t0;
}
int main() {
  double *in, *out; long long* cyc;
  cudaMalloc(&in, 16 * 8); cudaMalloc(&out, 8 * 8); cudaMalloc(&cyc, 3 * 8);
  double h[16]; for (int i = 0; i < 16; ++i) h[i] = 1.0 + i * 1e-3;
  cudaMemcpy(in, h, sizeof h, cudaMemcpyHostToDevice);
  const int n = 1 << 14;
  for (int rep = 0; rep < 2; ++rep) {
    k_addend<<<1, 32>>>(in, out, cyc, n);
    k_dadd<<<1, 32>>>(in, out, cyc, n);
    k_mult<<<1, 32>>>(in, out, cyc, n);
    cudaDeviceSynchronize();
  }
  long long c[3]; cudaMemcpy(c, cyc, sizeof c, cudaMemcpyDeviceToHost);
  printf("fma chain via addend: %.2f cyc/step\\n", (double)c[0] / (8.0 * n));
  printf("dadd chain:           %.2f cyc/step\\n", (double)c[1] / (8.0 * n));
  printf("fma chain via mult:   %.2f cyc/step\\n", (double)c[2] / (8.0 * n));
  return 0;
}
