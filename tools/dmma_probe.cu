// Probe: does the fp64 tensor-core MMA (mma.sync.m8n8k4.f64) accumulate like a sequential chain of
// fp64 FMAs, d = fma(a3, b3, fma(a2, b2, fma(a1, b1, fma(a0, b0, c))))? For the router's operands
// (bf16 x fp32 products, exact in fp64) the only difference can be the addition order / rounding.
// Compares, per output element, the MMA result against three candidate evaluation orders.
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ void dmma(double& d0, double& d1, double a, double b, double c0, double c1) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%4, %5};"
               : "=d"(d0), "=d"(d1) : "d"(a), "d"(b), "d"(c0), "d"(c1));
}

__device__ uint64_t mix(uint64_t z) {
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
// bf16-representable / fp32-representable values with a wide exponent spread (cancellation-heavy)
__device__ double rnd_bf16(uint64_t r) {
  const int e = (int)(r % 40) - 20;
  const float m = (float)((r >> 8) & 0xff) / 256.0f + 1.0f;
  float v = ldexpf(m, e) * ((r >> 20) & 1 ? -1.f : 1.f);
  uint32_t u = __float_as_uint(v) & 0xffff0000u;
  return (double)__uint_as_float(u);
}
__device__ double rnd_f32(uint64_t r) {
  const int e = (int)(r % 40) - 20;
  const float m = (float)((r >> 8) & 0xffffff) / 16777216.0f + 1.0f;
  return (double)(ldexpf(m, e) * ((r >> 40) & 1 ? -1.f : 1.f));
}

// each warp: one 8x8x4 MMA with accumulator C; A[8x4] row-major (x), B[4x8] col-major (w)
__global__ void probe(long long iters, unsigned long long* bad, unsigned long long seed, int mode) {
  const int lane = threadIdx.x & 31;
  const uint64_t base = seed ^ ((uint64_t)(blockIdx.x * blockDim.x + threadIdx.x) << 20);
  unsigned long long nb[3] = {0, 0, 0};
  for (long long it = 0; it < iters; ++it) {
    const uint64_t k = mix(base + it);
    // fragment layouts (m8n8k4 f64): A: lane holds A[lane/4][lane%4]; B: lane holds B[lane%4][lane/4];
    // C/D: lane holds C[lane/4][2*(lane%4) + {0,1}]
    const double a = rnd_bf16(mix(k ^ (uint64_t)lane));
    const double b = rnd_f32(mix(k ^ ((uint64_t)lane << 8) ^ 0x55));
    double c0 = mode ? rnd_f32(mix(k ^ ((uint64_t)lane << 16) ^ 0x77)) * 64.0 : rnd_f32(mix(k ^ ((uint64_t)lane << 16)));
    double c1 = rnd_f32(mix(k ^ ((uint64_t)lane << 24) ^ 0x99));
    double d0, d1;
    dmma(d0, d1, a, b, c0, c1);
    // gather the row of A and the columns of B this lane's outputs need
    const int row = lane / 4, col0 = 2 * (lane % 4);
    double ar[4], b0[4], b1[4];
    for (int q = 0; q < 4; ++q) {
      ar[q] = __shfl_sync(0xffffffffu, a, row * 4 + q);
      b0[q] = __shfl_sync(0xffffffffu, b, col0 * 4 + q);
      b1[q] = __shfl_sync(0xffffffffu, b, (col0 + 1) * 4 + q);
    }
    double s0 = c0, s1 = c1;  // sequential ascending-k FMA chain
    for (int q = 0; q < 4; ++q) { s0 = __fma_rn(ar[q], b0[q], s0); s1 = __fma_rn(ar[q], b1[q], s1); }
    double r0 = c0, r1 = c1;  // descending k
    for (int q = 3; q >= 0; --q) { r0 = __fma_rn(ar[q], b0[q], r0); r1 = __fma_rn(ar[q], b1[q], r1); }
    // products summed first (pairwise), then added to c
    const double p0 = __dadd_rn(__dadd_rn(__dmul_rn(ar[0], b0[0]), __dmul_rn(ar[1], b0[1])),
                                __dadd_rn(__dmul_rn(ar[2], b0[2]), __dmul_rn(ar[3], b0[3])));
    const double p1 = __dadd_rn(__dadd_rn(__dmul_rn(ar[0], b1[0]), __dmul_rn(ar[1], b1[1])),
                                __dadd_rn(__dmul_rn(ar[2], b1[2]), __dmul_rn(ar[3], b1[3])));
    const double t0 = __dadd_rn(c0, p0), t1 = __dadd_rn(c1, p1);
    nb[0] += (__double_as_longlong(d0) != __double_as_longlong(s0)) + (__double_as_longlong(d1) != __double_as_longlong(s1));
    nb[1] += (__double_as_longlong(d0) != __double_as_longlong(r0)) + (__double_as_longlong(d1) != __double_as_longlong(r1));
    nb[2] += (__double_as_longlong(d0) != __double_as_longlong(t0)) + (__double_as_longlong(d1) != __double_as_longlong(t1));
  }
  for (int i = 0; i < 3; ++i) atomicAdd(&bad[i], nb[i]);
}

// throughput / latency: each warp runs `chains` independent accumulator chains of `steps` DMMAs
template <int kChains>
__global__ void rate(int steps, double* out) {
  const int lane = threadIdx.x & 31;
  double a = 1.0 + lane * 1e-3, b = 1.0 - lane * 1e-3;
  double c[kChains][2];
#pragma unroll
  for (int i = 0; i < kChains; ++i) c[i][0] = c[i][1] = i;
  for (int s = 0; s < steps; ++s)
#pragma unroll
    for (int i = 0; i < kChains; ++i) dmma(c[i][0], c[i][1], a, b, c[i][0], c[i][1]);
  double t = 0;
#pragma unroll
  for (int i = 0; i < kChains; ++i) t += c[i][0] + c[i][1];
  if (t == 12345.678) out[0] = t;
}
template <int kChains>
void time_rate(int blocks, int warps, int steps) {
  double* o;
  cudaMalloc(&o, 8);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  rate<kChains><<<blocks, warps * 32>>>(steps, o);
  cudaEventRecord(e0);
  rate<kChains><<<blocks, warps * 32>>>(steps, o);
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double dmmas = (double)blocks * warps * steps * kChains;
  printf("chains %d blocks %d warps %d: %.3f ms, %.1f TFLOP/s fp64, %.1f ns per dependent DMMA\n", kChains, blocks,
         warps, ms, dmmas * 512 / (ms * 1e-3) / 1e12, ms * 1e6 / steps);
  cudaFree(o);
}

int main(int argc, char** argv) {
  time_rate<1>(1, 1, 100000);
  time_rate<4>(1, 1, 100000);
  time_rate<8>(148, 4, 20000);
  time_rate<4>(148, 8, 20000);
  time_rate<4>(148 * 2, 8, 20000);
  const long long iters = argc > 1 ? atoll(argv[1]) : 2000;
  unsigned long long* bad;
  cudaMalloc(&bad, 3 * sizeof(unsigned long long));
  for (int mode = 0; mode < 2; ++mode) {
    cudaMemset(bad, 0, 3 * sizeof(unsigned long long));
    probe<<<148 * 4, 256>>>(iters, bad, 12345 + mode, mode);
    unsigned long long h[3];
    cudaMemcpy(h, bad, sizeof(h), cudaMemcpyDeviceToHost);
    const double n = 148.0 * 4 * 256 * iters * 2;
    printf("mode %d: %.3g outputs; mismatches vs sequential-ascending %llu, descending %llu, products-first %llu (%s)\n",
           mode, n, h[0], h[1], h[2], cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
