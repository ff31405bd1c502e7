// Microbenchmark: DFMA dependent-chain latency, DFMA throughput, F2F.F64.F32 throughput on this GPU.
#include <cstdio>
#include <cuda_runtime.h>

__global__ void lat_kernel(double* out, long long* cyc, int n) {
  double a = out[0], b = 1.0000001, c = 0.5;
  long long t0 = clock64();
  for (int i = 0; i < n; ++i) a = fma(a, b, c);
  long long t1 = clock64();
  out[1] = a;
  *cyc = t1 - t0;
}
template <int CH>
__global__ void tput_kernel(double* out, int n) {
  double a[CH];
  for (int j = 0; j < CH; ++j) a[j] = out[j] + threadIdx.x;
  const double b = 1.0000001, c = 0.5;
  for (int i = 0; i < n; ++i)
#pragma unroll
    for (int j = 0; j < CH; ++j) a[j] = fma(a[j], b, c);
  double s = 0;
  for (int j = 0; j < CH; ++j) s += a[j];
  if (s == 12345.0) out[0] = s;
}
__global__ void f2f_kernel(const float* in, double* out, int n) {
  float v[8];
  for (int j = 0; j < 8; ++j) v[j] = in[j] + threadIdx.x;
  double s = 0;
  for (int i = 0; i < n; ++i) {
#pragma unroll
    for (int j = 0; j < 8; ++j) { s += (double)v[j]; v[j] += 1.0f; }
  }
  if (s == 12345.0) out[0] = s;
}
int main() {
  double* d; long long* c; float* f;
  cudaMalloc(&d, 1024 * sizeof(double)); cudaMalloc(&c, 8); cudaMalloc(&f, 64);
  cudaMemset(d, 0, 1024 * 8); cudaMemset(f, 0, 64);
  int n = 1 << 16;
  lat_kernel<<<1, 1>>>(d, c, n); cudaDeviceSynchronize();
  long long cyc; cudaMemcpy(&cyc, c, 8, cudaMemcpyDeviceToHost);
  printf("DFMA dependent latency: %.2f cycles\n", (double)cyc / n);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  for (int warps : {4, 8, 16, 32}) {
    tput_kernel<8><<<sms, 32 * warps>>>(d, 1024);
    cudaEventRecord(e0);
    tput_kernel<8><<<sms, 32 * warps>>>(d, 8192);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double fmas = (double)sms * 32 * warps * 8 * 8192;
    printf("DFMA tput, %2d warps/SM x 8 chains: %.2f TFMA/s = %.1f FMA/clk/SM (at %d MHz nominal)\n", warps,
           fmas / ms / 1e9, fmas / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
  }
  f2f_kernel<<<sms, 512>>>(f, d, 1024);
  cudaEventRecord(e0);
  f2f_kernel<<<sms, 512>>>(f, d, 8192);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double cv = (double)sms * 512 * 8 * 8192;
  printf("F2F.F64.F32 (+DADD) tput: %.1f conv/clk/SM\n", cv / (ms * 1e-3) / sms / (clk * 1e3));
  return 0;
}
