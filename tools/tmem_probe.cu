// Probe (not part of the library): where does tcgen05.mma.cta_group::2 put the accumulator rows
// for M = 128 (64 rows per CTA) versus M = 256? A[r][0] = unique id of (CTA, smem row),
// A[r][1] = 1; B[n][0] = 1000, B[n][1] = unique id of (CTA, smem B row). So D = 1000*aid + bid
// identifies the A row and B row behind every TMEM (lane, column). Build:
//   nvcc -gencode arch=compute_100a,code=sm_100a -std=c++17 -I../paper_2509_09121_b200/csrc tmem_probe.cu -o tmem_probe
#include <cuda.h>
#include <cuda_bf16.h>
#include <cstdio>
#include <vector>

#include "ptx.cuh"

using namespace cmoe;

constexpr int kN = 256;

__device__ void put(uint8_t* base, int row, int k, float v) {
  const int byte = k * 2;
  const int chunk = (byte / 16) ^ (row % 8);
  __nv_bfloat16* p = reinterpret_cast<__nv_bfloat16*>(base + (row / 8) * 1024 + (row % 8) * 128 + chunk * 16 + byte % 16);
  *p = __float2bfloat16(v);
}

template <int M>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128) probe(float* out, int tag, long long* cyc) {
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;                 // 128 rows x 128 B
  uint8_t* sB = smem + 128 * 128;     // 128 rows x 128 B
  __shared__ uint64_t bar;
  __shared__ uint32_t tslot;
  const int cta = cluster_ctarank();
  for (int i = threadIdx.x; i < 2 * 128 * 128 / 4; i += blockDim.x) reinterpret_cast<uint32_t*>(smem)[i] = 0;
  __syncthreads();
  if (threadIdx.x < 128) {
    const int r = threadIdx.x;
    put(sA, r, 0, float(cta * 128 + r + 1));
    put(sA, r, 2, float(tag));
    put(sB, r, 2, 65536.0f);
    put(sA, r, 1, 1.0f);
    put(sB, r, 0, 1000.0f);
    put(sB, r, 1, float(cta * 128 + r));
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  if (threadIdx.x == 0) {
    mbar_init(&bar, 1);
    fence_mbar_init();
  }
  if (warp_id() == 0) tmem_alloc<2>(&tslot, 512);
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tbase = tslot;
  if (cta == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_f32acc<false>(M, kN);
    mma_ss<2, false>(tbase, sdesc_k_sw128(smem_u32(sA)), sdesc_k_sw128(smem_u32(sB)), idesc, 0);
    mma_commit<2>(&bar, 3);
  }
  mbar_wait(&bar, 0);
  // throughput: 4096 back-to-back MMAs (K=16 each) into columns 256.., then one commit
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (cta == 0 && threadIdx.x == 0) {
    const uint32_t idesc = idesc_f32acc<false>(M, kN);
    const long long t0 = clock64();
    for (int i = 0; i < 4096; ++i)
      mma_ss<2, false>(tbase + 256, sdesc_k_sw128(smem_u32(sA)) + 2 * (i & 3), sdesc_k_sw128(smem_u32(sB)) + 2 * (i & 3),
                       idesc, 1);
    mma_commit<2>(&bar, 3);
    mbar_wait(&bar, 1);
    cyc[0] = clock64() - t0;
  } else {
    mbar_wait(&bar, 1);
  }
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (threadIdx.x == 0) printf("kernel M=%d cta %d tbase %u\n", M, cta, tbase);
  const int w = warp_id(), lane = lane_id();
  for (int c = 0; c < 512 / 32; ++c) {
    uint32_t a[32];
    tmem_ld32(tbase + ((uint32_t)(w * 32) << 16) + c * 32, a);
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    for (int i = 0; i < 32; ++i) out[((size_t)cta * 128 + w * 32 + lane) * 512 + c * 32 + i] = __uint_as_float(a[i]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  cluster_sync();
  if (warp_id() == 0) tmem_dealloc<2>(tbase, 512);
}

template <int M>
void run() {
  float* d;
  long long* cyc;
  cudaMalloc(&cyc, 8);
  cudaMalloc(&d, sizeof(float) * 2 * 128 * 512);
  cudaMemset(d, 0xff, sizeof(float) * 2 * 128 * 512);
  cudaFuncSetAttribute(probe<M>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
  probe<M><<<2, 128, 64 * 1024>>>(d, M == 128 ? 1 : 0, cyc);
  cudaError_t e = cudaDeviceSynchronize();
  std::vector<float> h(2 * 128 * 512);
  cudaMemcpy(h.data(), d, h.size() * 4, cudaMemcpyDeviceToHost);
  long long hc = 0;
  cudaMemcpy(&hc, cyc, 8, cudaMemcpyDeviceToHost);
  printf("M=%d status=%s  4096 MMAs (N=256, K=16): %lld cycles = %.1f cycles/MMA\n", M, cudaGetErrorString(e), hc,
         hc / 4096.0);
  for (int cta = 0; cta < 2; ++cta)
    for (int lane = 0; lane < 128; ++lane) {
      if (!(lane == 0 || lane == 63 || lane == 64 || lane == 127)) continue;
      const float* row = &h[((size_t)cta * 128 + lane) * 512];
      printf("cta %d lane %3d:", cta, lane);
      int c = 0;
      while (c < 256) {
        const int iv = (int)row[c];
        const int t = iv >= 65536, a = (iv % 65536) / 1000, b = (iv % 65536) % 1000;
        int e = c + 1;
        while (e < 512 && (int)row[e] == iv + (e - c)) ++e;
        printf(" [%d..%d: run%d a=%d b=%d..%d]", c, e - 1, t, a, b, b + (e - c) - 1);
        c = e;
      }
      printf("\n");
    }
  cudaFree(d);
}

int main() {
  run<256>();
  run<128>();
  return 0;
}
