// Probe: fp64 chains with operands streamed from shared memory (router latency variant pattern).
// 128-thread CTAs, thread = (token, expert) chain over L steps; x[tok][l] and w[l][e] in smem.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N4 = 16, TPC = 8, L = 128;
template <int V>
__global__ void __launch_bounds__(128) chain(const double* gx, const double* gw, double* out, long long* cyc, int reps) {
  __shared__ double sx[TPC * L];
  __shared__ double sw[L * N4];
  __shared__ __align__(16) double swT[N4 * (L + 2)];
  for (int i = threadIdx.x; i < TPC * L; i += 128) sx[i] = gx[i];
  for (int i = threadIdx.x; i < L * N4; i += 128) sw[i] = gw[i];
  for (int i = threadIdx.x; i < L * N4; i += 128) swT[(i % N4) * (L + 2) + i / N4] = gw[i];
  __syncthreads();
  const int tl = threadIdx.x / N4, e = threadIdx.x % N4;
  const double* xr = sx + tl * L;
  const double* wc = sw + e;
  double acc = 0.0;
  long long t0 = clock64();
  for (int r = 0; r < reps; ++r) {
    if (V == 0) {  // plain
#pragma unroll 16
      for (int l = 0; l < L; ++l) acc = fma(xr[l], wc[l * N4], acc);
    } else if (V == 1) {  // products first (DMUL off the chain), then DADD chain
#pragma unroll 1
      for (int b = 0; b < L; b += 16) {
        double p[16];
#pragma unroll
        for (int i = 0; i < 16; ++i) p[i] = xr[b + i] * wc[(b + i) * N4];
#pragma unroll
        for (int i = 0; i < 16; ++i) acc += p[i];
      }
    } else if (V == 3) {  // expert-major W ([e][l], padded rows), 2 steps per LDS.128 for both operands
      const double* we = swT + e * (L + 2);
#pragma unroll 16
      for (int l = 0; l < L; l += 2) {
        const double2 xx = *reinterpret_cast<const double2*>(xr + l);
        const double2 ww = *reinterpret_cast<const double2*>(we + l);
        acc = fma(xx.x, ww.x, acc);
        acc = fma(xx.y, ww.y, acc);
      }
    } else {  // registers only: loads once, chain over registers (upper bound)
      double xv[16], wv[16];
#pragma unroll
      for (int i = 0; i < 16; ++i) { xv[i] = xr[i]; wv[i] = wc[i * N4]; }
#pragma unroll 1
      for (int b = 0; b < L; b += 16)
#pragma unroll
        for (int i = 0; i < 16; ++i) acc = fma(xv[i], wv[i], acc);
    }
  }
  long long t1 = clock64();
  out[blockIdx.x * 128 + threadIdx.x] = acc;
  if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}
int main() {
  double *gx, *gw, *out; long long* cyc;
  cudaMalloc(&gx, TPC * L * 8); cudaMalloc(&gw, L * N4 * 8); cudaMalloc(&out, 64 * 128 * 8); cudaMalloc(&cyc, 64 * 8);
  cudaMemset(gx, 0, TPC * L * 8); cudaMemset(gw, 0, L * N4 * 8);
  const int reps = 16;
  long long h[64];
  chain<0><<<64, 128>>>(gx, gw, out, cyc, reps); cudaDeviceSynchronize();
  chain<0><<<64, 128>>>(gx, gw, out, cyc, reps); cudaMemcpy(h, cyc, 8 * 64, cudaMemcpyDeviceToHost);
  printf("fma chain, smem operands:        %.2f cyc/step\n", (double)h[0] / (reps * L));
  chain<1><<<64, 128>>>(gx, gw, out, cyc, reps); cudaMemcpy(h, cyc, 8 * 64, cudaMemcpyDeviceToHost);
  printf("dmul then dadd chain, smem:      %.2f cyc/step\n", (double)h[0] / (reps * L));
  chain<3><<<64, 128>>>(gx, gw, out, cyc, reps); cudaMemcpy(h, cyc, 8 * 64, cudaMemcpyDeviceToHost);
  printf("fma chain, expert-major W, LDS.128: %.2f cyc/step\n", (double)h[0] / (reps * L));
  chain<2><<<64, 128>>>(gx, gw, out, cyc, reps); cudaMemcpy(h, cyc, 8 * 64, cudaMemcpyDeviceToHost);
  printf("fma chain, register operands:    %.2f cyc/step\n", (double)h[0] / (reps * L));
  return 0;
}
