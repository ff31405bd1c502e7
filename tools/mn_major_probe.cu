// Probe (not part of the library): tcgen05.mma with MN-major A and B operands in the 128-byte
// swizzled layout a TMA box {64 elements (MN, inner), K rows} produces. Checks D = A B against a
// host reference for a few descriptor conventions. One CTA, cta_group::1, M=128, N=256, K=64.
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2509_09121_b200/csrc mn_major_probe.cu -o mn_major_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "ptx.cuh"

using namespace cmoe;

constexpr int M = 128, N = 256, K = 64;

// element (k, j) of an MN-major operand with MN extent `mn`: 64-element MN chunks of K rows x 128 B
__host__ __device__ inline int mn_off(int k, int j) {
  const int ch = j / 64, jj = j % 64;
  const int byte = jj * 2;
  return ch * (K * 128) + (k / 8) * 1024 + (k % 8) * 128 + (((byte / 16) ^ (k % 8)) * 16) + byte % 16;
}

__device__ uint64_t desc_mn(uint32_t saddr, uint32_t lbo, uint32_t sbo) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFFu);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFFu) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFFu) << 32;
  d |= static_cast<uint64_t>(1u) << 46;  // version
  d |= static_cast<uint64_t>(2u) << 61;  // SWIZZLE_128B
  return d;
}

__global__ void __launch_bounds__(128) probe(const __nv_bfloat16* A, const __nv_bfloat16* B, float* out, int lbo,
                                             int sbo, int kstep_bytes, int majbits) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                     // 2 chunks x 8 KB
  uint8_t* sB = smem + (M / 64) * K * 128;  // 4 chunks x 8 KB
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  // A logical [M][K] given row-major as At [K][M]; B logical [N][K] given as Bt [K][N]
  for (int i = threadIdx.x; i < K * M; i += 128) {
    const int k = i / M, m = i % M;
    *reinterpret_cast<__nv_bfloat16*>(sA + mn_off(k, m)) = A[k * M + m];
  }
  for (int i = threadIdx.x; i < K * N; i += 128) {
    const int k = i / N, n = i % N;
    *reinterpret_cast<__nv_bfloat16*>(sB + mn_off(k, n)) = B[k * N + n];
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp_id() == 0) tmem_alloc<1>(&tslot, 256);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tslot;
  if (threadIdx.x == 0) {
    const uint32_t idesc = idesc_f32acc<false>(M, N) | static_cast<uint32_t>(majbits);
    for (int k = 0; k < K / 16; ++k) {
      const uint64_t ad = desc_mn(smem_u32(sA) + k * kstep_bytes, lbo, sbo);
      const uint64_t bd = desc_mn(smem_u32(sB) + k * kstep_bytes, lbo, sbo);
      mma_ss<1, false>(tbase, ad, bd, idesc, k > 0);
    }
    mma_commit<1>(&bar);
  }
  mbar_wait(&bar, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const int w = warp_id(), lane = lane_id();
  for (int c = 0; c < N / 32; ++c) {
    uint32_t a[32];
    tmem_ld32(tbase + ((uint32_t)(w * 32) << 16) + c * 32, a);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) out[(w * 32 + lane) * N + c * 32 + i] = __uint_as_float(a[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp_id() == 0) tmem_dealloc<1>(tbase, 256);
}

int main() {
  std::vector<float> a(M * K), b(N * K);
  std::vector<__nv_bfloat16> at(K * M), bt(K * N);
  srand(1);
  for (int m = 0; m < M; ++m)
    for (int k = 0; k < K; ++k) {
      const float v = (float)((rand() % 17) - 8) / 8.0f;
      a[m * K + k] = v;
      at[k * M + m] = __float2bfloat16(v);
    }
  for (int n = 0; n < N; ++n)
    for (int k = 0; k < K; ++k) {
      const float v = (float)((rand() % 13) - 6) / 4.0f;
      b[n * K + k] = v;
      bt[k * N + n] = __float2bfloat16(v);
    }
  std::vector<float> ref(M * N, 0.f);
  for (int m = 0; m < M; ++m)
    for (int n = 0; n < N; ++n) {
      double s = 0;
      for (int k = 0; k < K; ++k) s += (double)a[m * K + k] * b[n * K + k];
      ref[m * N + n] = (float)s;
    }
  __nv_bfloat16 *dA, *dB;
  float* dO;
  cudaMalloc(&dA, at.size() * 2);
  cudaMalloc(&dB, bt.size() * 2);
  cudaMalloc(&dO, M * N * 4);
  cudaMemcpy(dA, at.data(), at.size() * 2, cudaMemcpyHostToDevice);
  cudaMemcpy(dB, bt.data(), bt.size() * 2, cudaMemcpyHostToDevice);
  cudaFuncSetAttribute(probe, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  struct Cfg { int lbo, sbo, kstep, maj; const char* name; };
  const int kMaj = (1 << 15) | (1 << 16);
  const Cfg cfgs[] = {
      {K * 128, 1024, 16 * 128, kMaj, "LBO=chunk(8KB) SBO=1KB kstep=2KB"},
      {1024, K * 128, 16 * 128, kMaj, "LBO=1KB SBO=chunk(8KB) kstep=2KB"},
  };
  for (const Cfg& c : cfgs) {
    cudaMemset(dO, 0, M * N * 4);
    probe<<<1, 128, 64 * 1024>>>(dA, dB, dO, c.lbo, c.sbo, c.kstep, c.maj);
    const cudaError_t e = cudaDeviceSynchronize();
    std::vector<float> o(M * N);
    cudaMemcpy(o.data(), dO, M * N * 4, cudaMemcpyDeviceToHost);
    int bad = 0;
    double maxe = 0;
    for (int i = 0; i < M * N; ++i) {
      const double d = std::abs((double)o[i] - ref[i]);
      if (d > 1e-3) ++bad;
      if (d > maxe) maxe = d;
    }
    printf("%-40s status=%s mismatches=%d max|err|=%.3g  o[0]=%g ref[0]=%g o[1]=%g ref[1]=%g\n", c.name,
           cudaGetErrorString(e), bad, maxe, o[0], ref[0], o[N + 1], ref[N + 1]);
  }
  return 0;
}
