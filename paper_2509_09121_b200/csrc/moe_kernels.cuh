// Router (K1), dispatch plan (K2), fused permute/dispatch (K3) and weighted combine (K6)
// kernels of the MoE layer. All are memory- or latency-bound; see DESIGN.md for their rooflines.
#pragma once
#include <algorithm>
#include <cuda_fp8.h>

#include "glibc_exp.cuh"
#include "ptx.cuh"

namespace cmoe {

constexpr int kRouterChunk = 64;  // d-columns staged per pipeline step (d % 256 == 0 by config)
constexpr int kRouterTT = 1;      // tokens per thread
constexpr int kPlanThreads = 1024;

// Device-side routing state shared by the kernels of one forward call.
struct RouteBufs {
  float* logits;        // [T][N]
  float* probs;         // [T][N]
  int32_t* topk_idx;    // [T][K]
  float* combine_w;     // [T][K]
  int32_t* local_rank;  // [T][K] rank of the slot among same-expert slots of its router tile
  int32_t* tile_cnt;    // [n_tiles][N] -> rewritten in place with the tile's base within the expert
  double* tile_psum;    // [n_tiles][N] sum of probs over the tile's tokens (double)
  double* tile_lse2;    // [n_tiles] sum of lse^2 over the tile's tokens (double)
  int32_t* counts;      // [N]
  int32_t* offsets;     // [N+1]
  float* agg_prob;      // [N]
  float* losses;        // [2] aux, z
  int32_t* finite_flag; // [1] set to 1 on any non-finite router logit or layer output (K11)
};

// Router tile geometry: one thread per (token, 4 experts). Two variants: 128-thread CTAs with a
// 3-deep ring for large batches (throughput), 32-thread CTAs with an 8-deep ring for small batches
// (latency: more CTAs in flight and a deeper prefetch of the sequential chunk stream).
__host__ __device__ inline int router_tokens_per_cta(int n_experts, int threads) {
  const int groups = (n_experts + 3) / 4;
  return (threads / groups) * kRouterTT;
}
struct RouterSmem {
  int tpc, N4, xs;
  size_t raw_x, sw, sx, slog, sidx, slse, total;
  __host__ __device__ RouterSmem(int n_experts, int threads, int stages, int xb = 2) {
    N4 = (n_experts + 3) / 4 * 4;
    tpc = router_tokens_per_cta(n_experts, threads);
    xs = kRouterChunk + 2;  // padded fp64 row of one token: 16-byte aligned, conflict-free double2 loads
    raw_x = 0;
    sw = raw_x + (size_t)stages * tpc * kRouterChunk * xb;    // [stages][chunk][N4] fp64 (cp.async target)
    sx = sw + (size_t)stages * sizeof(double) * kRouterChunk * N4;  // [tpc][xs] fp64
    slog = sx + sizeof(double) * tpc * xs;
    sidx = slog + sizeof(float) * tpc * N4;
    slse = (sidx + sizeof(int) * tpc * 8 + 7) / 8 * 8;
    total = slse + sizeof(double) * tpc;
  }
};
__host__ __device__ inline size_t router_smem_bytes(int n_experts, int threads, int stages, int xb = 2) {
  return RouterSmem(n_experts, threads, stages, xb).total;
}

__device__ __forceinline__ void cp_async16(void* dst, const void* src, bool valid) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16, %2;" ::"r"(smem_u32(dst)), "l"(src), "r"(valid ? 16 : 0)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

// Router input element: bf16 (the device path's storage type), fp32 (the reference's own Tensor
// values), or uint8 = E4M3 codes of the FP8 scheme's router operand, whose value
// is code * s (fp32 multiply: exactly qdq_e4m3's x_hat). Each widens exactly to fp64, and a
// float x float product is exact in fp64, so the ascending-l chains stay bit-identical to gemm_nn.
template <typename XT>
__device__ __forceinline__ double x_to_f64(XT v, float xs = 1.0f) {
  if constexpr (sizeof(XT) == 1) {
    const __half_raw hr = __nv_cvt_fp8_to_halfraw(static_cast<__nv_fp8_storage_t>(v), __NV_E4M3);
    return static_cast<double>(__fmul_rn(__half2float(__half(hr)), xs));
  } else if constexpr (sizeof(XT) == 2) {
    return static_cast<double>(__bfloat162float(v));
  } else {
    return static_cast<double>(v);
  }
}
// 16 bytes of raw x -> its 16 (e4m3), 8 (bf16) or 4 (fp32) values in fp64
template <typename XT>
__device__ __forceinline__ void widen16(const int4& raw, double* out, float xs = 1.0f) {
  const XT* v = reinterpret_cast<const XT*>(&raw);
#pragma unroll
  for (int i = 0; i < 16 / (int)sizeof(XT); ++i) out[i] = x_to_f64<XT>(v[i], xs);
}
__device__ __forceinline__ float router_xscale(const float* p) { return p ? *p : 1.0f; }

// Chunk length (steps) of router_ws_kernel's ring, by padded expert count.
__host__ __device__ inline int router_ws_chunk(int N4) { return N4 <= 16 ? 256 : N4 <= 32 ? 128 : N4 <= 64 ? 64 : 32; }

// W_r [d][N] fp32 -> fp64 [d][N4] (zero-padded experts), followed by the layout router_ws_kernel
// streams: per chunk of router_ws_chunk(N4) steps, [N4][chunk + 2] expert-major rows (2 pad
// doubles per row so a warp's experts hit distinct banks) — one contiguous bulk copy per ring
// slot. Once per weight update.
__global__ void widen_router_kernel(const float* __restrict__ wr, int d, int N, double* __restrict__ out) {
  const int N4 = (N + 3) / 4 * 4, N8 = (N + 7) / 8 * 8;
  const int chunk = router_ws_chunk(N4), pitch = chunk + 2;
  double* wt = out + (size_t)d * N4;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d * N4; i += gridDim.x * blockDim.x) {
    const int l = i / N4, e = i % N4;
    const double v = e < N ? static_cast<double>(wr[(size_t)l * N + e]) : 0.0;
    out[i] = v;
    const int c = l / chunk, j = l % chunk;
    double* row = wt + ((size_t)c * N4 + e) * pitch;
    row[j] = v;
    if (j == 0) row[chunk] = row[chunk + 1] = 0.0;
  }
  // router_dmma_kernel's B fragments: [d/4][N8/8][32], lane = (e % 8) * 4 + l % 4
  // (router_wfrag_offset: after the two layouts above)
  const size_t foff = (size_t)d * N4 + (size_t)(d / chunk) * N4 * pitch;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d * N8; i += gridDim.x * blockDim.x) {
    const int l = i / N8, e = i % N8;
    const double v = e < N ? static_cast<double>(wr[(size_t)l * N + e]) : 0.0;
    out[foff + ((size_t)(l / 4) * (N8 / 8) + e / 8) * 32 + (e % 8) * 4 + l % 4] = v;
  }
}

// Per-token softmax (fp64, tensor.cpp:614-621), top-K with lowest-index tie-break
// (tensor.cpp:1046-1060), renormalised combine weights, and the per-tile
// statistics (expert counts, local ranks, prob sums, lse^2 sums) of one router tile whose fp32
// logits sit in slog[tpc][N4]. Called by all threads of the CTA after a barrier.
__device__ __forceinline__ void router_finish(int tile, int tok0, int tpc, int T, int N, int N4, int K, float* slog,
                                              int* sidx, double* slse, const RouteBufs& rb, int nthreads) {
  const int ntok = min(tpc, T - tok0);
  for (int tl = threadIdx.x; tl < tpc; tl += nthreads) {
    double lse2 = 0.0;
    if (tl < ntok) {
      const int j = tok0 + tl;
      float* zrow = slog + tl * N4;
      double mx = zrow[0];
      for (int e = 1; e < N; ++e) mx = fmax(mx, static_cast<double>(zrow[e]));
      double denom = 0.0;
      for (int e = 0; e < N; ++e) denom += exp_glibc(static_cast<double>(zrow[e]) - mx);
      float* p = rb.probs + (size_t)j * N;
      for (int e = 0; e < N; ++e) {
        const float pe = static_cast<float>(exp_glibc(static_cast<double>(zrow[e]) - mx) / denom);
        p[e] = pe;
        zrow[e] = pe;  // the row now holds probs
      }
      const double lse = mx + log(denom);
      lse2 = lse * lse;
      uint64_t taken_lo = 0, taken_hi = 0;
      float vals[8];
      int ids[8];
      for (int k = 0; k < K; ++k) {
        int best = -1;
        float bv = 0.0f;
        for (int e = 0; e < N; ++e) {
          const bool tk = e < 64 ? ((taken_lo >> e) & 1ull) : ((taken_hi >> (e - 64)) & 1ull);
          if (tk) continue;
          const float v = zrow[e];
          if (best < 0 || v > bv) { best = e; bv = v; }  // strict '>' keeps the lowest index on ties
        }
        if (best < 64) taken_lo |= 1ull << best; else taken_hi |= 1ull << (best - 64);
        vals[k] = bv;
        ids[k] = best;
      }
      double s = 0.0;
      for (int k = 0; k < K; ++k) s += static_cast<double>(vals[k]);
      for (int k = 0; k < K; ++k) {
        rb.topk_idx[(size_t)j * K + k] = ids[k];
        rb.combine_w[(size_t)j * K + k] = static_cast<float>(static_cast<double>(vals[k]) / s);
        sidx[tl * 8 + k] = ids[k];
      }
    }
    slse[tl] = lse2;
  }
  __syncthreads();
  for (int e = threadIdx.x; e < N; e += nthreads) {
    int cnt = 0;
    double ps = 0.0;
    for (int t = 0; t < ntok; ++t) {
      ps += static_cast<double>(slog[t * N4 + e]);
      for (int k = 0; k < K; ++k)
        if (sidx[t * 8 + k] == e) rb.local_rank[(size_t)(tok0 + t) * K + k] = cnt++;
    }
    rb.tile_cnt[(size_t)tile * N + e] = cnt;
    rb.tile_psum[(size_t)tile * N + e] = ps;
  }
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int t = 0; t < ntok; ++t) a += slse[t];
    rb.tile_lse2[tile] = a;
  }
}

// ---------------------------------------------------------------------------------------
// K1: router. logits = x W_r with one fp64 accumulator per (token, expert) summed over the
// hidden dimension in ascending order — the exact accumulation order of the reference gemm_nn
// (proj/src/tensor.cpp:157-173), so logits are bit-identical to the CPU oracle (each product of
// two floats is exact in fp64, hence FMA == multiply-then-add). x chunks (bf16) and the fp64 copy
// of W_r stream into shared memory through a double-buffered cp.async pipeline; x is widened to
// fp64 once per CTA. One thread owns 4 independent accumulator chains (1 token x 4 experts).
// Then per token: softmax in fp64 (tensor.cpp:614-621), top-K with lowest-index tie-break
// (tensor.cpp:1046-1060), renormalised combine weights, per-tile expert counts
// and local ranks for the stable dispatch permutation, and per-tile partial sums for agg_prob
// (col_sums, tensor.cpp:545-565) and the Z-loss (tensor.cpp:1011-1040).
template <int kRouterThreads, int kStages, typename XT = __nv_bfloat16>
__global__ void __launch_bounds__(kRouterThreads, 1) router_kernel(const XT* __restrict__ x,
                                                                const double* __restrict__ wr64, int T, int d,
                                                                int N, int K, RouteBufs rb,
                                                                const float* __restrict__ xscale = nullptr) {
  constexpr int kXB = sizeof(XT), kPerPiece = 16 / kXB;  // x elements per 16-byte cp.async piece
  const float xsc = router_xscale(xscale);
  const RouterSmem L(N, kRouterThreads, kStages, kXB);
  const int groups = L.N4 / 4;
  const int N4 = L.N4;
  const int tg_per_cta = kRouterThreads / groups;
  const int tpc = L.tpc;  // tokens per CTA
  const int xs = L.xs;
  const int tile = blockIdx.x;
  const int tok0 = tile * tpc;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  XT* rawx = reinterpret_cast<XT*>(smem_raw + L.raw_x);                        // [stages][tpc][chunk]
  double* sw = reinterpret_cast<double*>(smem_raw + L.sw);                     // [2][chunk][N4]
  double* sx = reinterpret_cast<double*>(smem_raw + L.sx);                     // [tpc][xs]
  float* slog = reinterpret_cast<float*>(smem_raw + L.slog);                   // [tpc][N4]
  int* sidx = reinterpret_cast<int*>(smem_raw + L.sidx);                       // [tpc][8]
  double* slse = reinterpret_cast<double*>(smem_raw + L.slse);                 // [tpc]

  const int tgi = threadIdx.x / groups;  // token (group)
  const int g = threadIdx.x % groups;    // expert group
  const bool worker = tgi < tg_per_cta;
  double acc[kRouterTT][4];
#pragma unroll
  for (int a = 0; a < kRouterTT; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  const int nchunks = d / kRouterChunk;
  const int xpieces = tpc * kRouterChunk * kXB / 16;  // 16-byte pieces of one x chunk
  const int wpieces = kRouterChunk * N4 * 8 / 16;
  auto issue = [&](int c, int buf) {
    const int c0 = c * kRouterChunk;
    for (int i = threadIdx.x; i < xpieces; i += kRouterThreads) {
      const int r = i / (kRouterChunk / kPerPiece), q = i % (kRouterChunk / kPerPiece);
      const bool ok = tok0 + r < T;
      const XT* src = x + (size_t)(ok ? tok0 + r : 0) * d + c0 + q * kPerPiece;
      cp_async16(rawx + (size_t)buf * tpc * kRouterChunk + r * kRouterChunk + q * kPerPiece, src, ok);
    }
    const double* wsrc = wr64 + (size_t)c0 * N4;
    for (int i = threadIdx.x; i < wpieces; i += kRouterThreads)
      cp_async16(sw + (size_t)buf * kRouterChunk * N4 + i * 2, wsrc + i * 2, true);
    cp_async_commit();
  };
  for (int c = 0; c < kStages - 1; ++c) {
    if (c < nchunks) issue(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kStages;
    cp_async_wait<kStages - 2>();  // chunk c has landed (one group committed per chunk)
    __syncthreads();               // ... and every thread is done with chunk c-1's buffers
    if (c + kStages - 1 < nchunks) issue(c + kStages - 1, (c + kStages - 1) % kStages);
    else cp_async_commit();
    // widen x to fp64, [tok][l] layout
    const XT* rx = rawx + (size_t)buf * tpc * kRouterChunk;
    for (int i = threadIdx.x; i < tpc * kRouterChunk / 2; i += kRouterThreads) {
      const int r = (2 * i) / kRouterChunk, l = (2 * i) % kRouterChunk;
      if constexpr (kXB == 2) {
        const __nv_bfloat162 v = reinterpret_cast<const __nv_bfloat162*>(rx)[i];
        *reinterpret_cast<double2*>(sx + r * xs + l) =
            make_double2(static_cast<double>(__low2float(v)), static_cast<double>(__high2float(v)));
      } else if constexpr (kXB == 4) {
        const float2 v = reinterpret_cast<const float2*>(rx)[i];
        *reinterpret_cast<double2*>(sx + r * xs + l) = make_double2(static_cast<double>(v.x), static_cast<double>(v.y));
      } else {
        *reinterpret_cast<double2*>(sx + r * xs + l) = make_double2(x_to_f64<XT>(rx[2 * i], xsc), x_to_f64<XT>(rx[2 * i + 1], xsc));
      }
    }
    __syncthreads();
    if (worker) {
      const double2* xv = reinterpret_cast<const double2*>(sx + tgi * xs);
      const double2* wv = reinterpret_cast<const double2*>(sw + (size_t)buf * kRouterChunk * N4 + g * 4);
      // Register double buffer: the operands of l-pair block b+1 are requested before block b is
      // consumed, so the four accumulator chains never wait on a shared-memory round trip.
      constexpr int kU = 4;
      double2 cur[kU][5], nxt[kU][5];
      auto load = [&](double2 (&r)[kU][5], int l2b) {
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const int l2 = l2b + u;
          r[u][0] = xv[l2];
          r[u][1] = wv[(2 * l2) * (N4 / 2)];
          r[u][2] = wv[(2 * l2) * (N4 / 2) + 1];
          r[u][3] = wv[(2 * l2 + 1) * (N4 / 2)];
          r[u][4] = wv[(2 * l2 + 1) * (N4 / 2) + 1];
        }
      };
      load(cur, 0);
#pragma unroll
      for (int l2b = 0; l2b < kRouterChunk / 2; l2b += kU) {
        if (l2b + kU < kRouterChunk / 2) load(nxt, l2b + kU);
#pragma unroll
        for (int u = 0; u < kU; ++u) {
          const double2 xx = cur[u][0];
          acc[0][0] = fma(xx.x, cur[u][1].x, acc[0][0]);
          acc[0][1] = fma(xx.x, cur[u][1].y, acc[0][1]);
          acc[0][2] = fma(xx.x, cur[u][2].x, acc[0][2]);
          acc[0][3] = fma(xx.x, cur[u][2].y, acc[0][3]);
          acc[0][0] = fma(xx.y, cur[u][3].x, acc[0][0]);
          acc[0][1] = fma(xx.y, cur[u][3].y, acc[0][1]);
          acc[0][2] = fma(xx.y, cur[u][4].x, acc[0][2]);
          acc[0][3] = fma(xx.y, cur[u][4].y, acc[0][3]);
        }
#pragma unroll
        for (int u = 0; u < kU; ++u)
#pragma unroll
          for (int q = 0; q < 5; ++q) cur[u][q] = nxt[u][q];
      }
    }
    __syncthreads();
  }
  if (worker) {
#pragma unroll
    for (int a = 0; a < kRouterTT; ++a) {
      const int tl = tgi * kRouterTT + a;
      const int tok = tok0 + tl;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int e = g * 4 + b;
        const float z = static_cast<float>(acc[a][b]);
        slog[tl * N4 + e] = z;
        if (tok < T && e < N) {
          rb.logits[(size_t)tok * N + e] = z;
          if (!isfinite(z)) atomicOr(rb.finite_flag, 1);
        }
      }
    }
  }
  __syncthreads();

  router_finish(tile, tok0, tpc, T, N, N4, K, slog, sidx, slse, rb, kRouterThreads);
}

// ---------------------------------------------------------------------------------------
// K1, latency variant (decode-size batches): one thread per (token, expert) chain. A 4096-long
// fp64 chain costs 4096 x 8.7 cycles of DFMA latency whatever the blocking, so at small T the
// only lever is parallelism: 128-thread CTAs of (128 / N4) tokens x N4 experts, x and W chunks
// through a cp.async ring. The x chunk is widened to fp64 once per CTA (not once per expert:
// F2F runs at 15/clk/SM), then the operands of 32 steps are loaded ahead of their 32 dependent
// DFMAs. Chunks are 256 steps for N <= 16 (128 / 64 for more experts) so the per-chunk barrier and
// refill overhead is amortised over a long chain segment. Same ascending-l order per chain.
template <int kStages, int kChunk>
struct RouterLatSmem {
  int tpc, N4;
  size_t rx, sw, xd, slog, sidx, slse, total;
  __host__ __device__ RouterLatSmem(int n_experts) {
    N4 = (n_experts + 3) / 4 * 4;
    tpc = N4 >= 128 ? 1 : 128 / N4;
    rx = 0;                                                          // [stages][tpc][chunk] bf16
    sw = rx + ((size_t)kStages * tpc * kChunk * 2 + 15) / 16 * 16;  // [stages][chunk][N4] fp64
    xd = sw + (size_t)kStages * sizeof(double) * kChunk * N4;       // [tpc][chunk] fp64
    slog = xd + sizeof(double) * tpc * kChunk;
    sidx = slog + sizeof(float) * tpc * N4;
    slse = (sidx + sizeof(int) * tpc * 8 + 7) / 8 * 8;
    total = slse + sizeof(double) * tpc;
  }
};

template <int kStages, int kChunk>
__global__ void __launch_bounds__(128) router_lat_kernel(const __nv_bfloat16* __restrict__ x,
                                                         const double* __restrict__ wr64, int T, int d, int N, int K,
                                                         RouteBufs rb) {
  constexpr int kThreads = 128;
  const RouterLatSmem<kStages, kChunk> L(N);
  const int N4 = L.N4, tpc = L.tpc;
  const int tile = blockIdx.x;
  const int tok0 = tile * tpc;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  __nv_bfloat16* rawx = reinterpret_cast<__nv_bfloat16*>(smem_raw + L.rx);
  double* sw = reinterpret_cast<double*>(smem_raw + L.sw);
  double* xd = reinterpret_cast<double*>(smem_raw + L.xd);
  float* slog = reinterpret_cast<float*>(smem_raw + L.slog);
  int* sidx = reinterpret_cast<int*>(smem_raw + L.sidx);
  double* slse = reinterpret_cast<double*>(smem_raw + L.slse);
  const int tl = threadIdx.x / N4;  // token of this chain
  const int e = threadIdx.x % N4;   // expert of this chain
  const bool worker = tl < tpc;
  double acc = 0.0;

  const int nchunks = d / kChunk;
  const int xpieces = tpc * (kChunk / 8);
  const int wpieces = kChunk * N4 / 2;
  auto issue = [&](int c, int buf) {
    const int c0 = c * kChunk;
    for (int i = threadIdx.x; i < xpieces; i += kThreads) {
      const int r = i / (kChunk / 8), q = i % (kChunk / 8);
      const bool ok = tok0 + r < T;
      const __nv_bfloat16* src = x + (size_t)(ok ? tok0 + r : 0) * d + c0 + q * 8;
      cp_async16(rawx + ((size_t)buf * tpc + r) * kChunk + q * 8, src, ok);
    }
    const double* wsrc = wr64 + (size_t)c0 * N4;
    for (int i = threadIdx.x; i < wpieces; i += kThreads)
      cp_async16(sw + (size_t)buf * kChunk * N4 + i * 2, wsrc + i * 2, true);
    cp_async_commit();
  };
  for (int c = 0; c < kStages - 1; ++c) {
    if (c < nchunks) issue(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kStages;
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (c + kStages - 1 < nchunks) issue(c + kStages - 1, (c + kStages - 1) % kStages);
    else cp_async_commit();
    // widen the chunk's x once for all experts
    const __nv_bfloat16* rx = rawx + (size_t)buf * tpc * kChunk;
    for (int i = threadIdx.x * 8; i < tpc * kChunk; i += kThreads * 8) {  // 8 values per thread and pass
      const int4 raw = *reinterpret_cast<const int4*>(rx + i);
      const __nv_bfloat16* hv = reinterpret_cast<const __nv_bfloat16*>(&raw);
      double v[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) v[j] = static_cast<double>(__bfloat162float(hv[j]));
#pragma unroll
      for (int j = 0; j < 8; j += 2) *reinterpret_cast<double2*>(xd + i + j) = make_double2(v[j], v[j + 1]);
    }
    __syncthreads();
    if (worker) {
      // 32 steps' operands are loaded before their 32 dependent DFMAs: one shared-memory round
      // trip (~30 cycles) per 32 x 8-cycle chain segment. (Interleaving loads with the chain lets
      // ptxas schedule each load right before its use, exposing the latency on every step.)
      const double* xr = xd + (size_t)tl * kChunk;
      const double* wc = sw + (size_t)buf * kChunk * N4 + e;
      // Register double buffer across a NON-unrolled loop: the loads of block b+1 are issued at
      // the top of iteration b and consumed only in the next iteration, so ptxas cannot sink
      // them next to their uses; each 16-step FMA segment (~128 cycles) covers the round trip.
      constexpr int kB = 16;
      double xa[kB], wa[kB], xb[kB], wb[kB];
      auto ld = [&](double (&xv)[kB], double (&w)[kB], int base) {
#pragma unroll
        for (int i = 0; i < kB; i += 2) {
          const double2 t = *reinterpret_cast<const double2*>(xr + base + i);
          xv[i] = t.x;
          xv[i + 1] = t.y;
        }
#pragma unroll
        for (int i = 0; i < kB; ++i) w[i] = wc[(base + i) * N4];
      };
      ld(xa, wa, 0);
#pragma unroll 1
      for (int hb = 0; hb < kChunk; hb += 2 * kB) {
        ld(xb, wb, hb + kB);
#pragma unroll
        for (int i = 0; i < kB; ++i) acc = fma(xa[i], wa[i], acc);
        if (hb + 2 * kB < kChunk) ld(xa, wa, hb + 2 * kB);
#pragma unroll
        for (int i = 0; i < kB; ++i) acc = fma(xb[i], wb[i], acc);
      }
    }
    __syncthreads();  // xd is rewritten by the next chunk
  }
  __syncthreads();
  if (worker) {
    const int tok = tok0 + tl;
    const float z = static_cast<float>(acc);
    slog[tl * N4 + e] = z;
    if (tok < T && e < N) {
      rb.logits[(size_t)tok * N + e] = z;
      if (!isfinite(z)) atomicOr(rb.finite_flag, 1);
    }
  }
  __syncthreads();
  router_finish(tile, tok0, tpc, T, N, N4, K, slog, sidx, slse, rb, kThreads);
}

// ---------------------------------------------------------------------------------------
// K2 body (the dispatch plan; see plan_kernel below), shared by plan_kernel and router_ws_kernel's
// fused tail: threads >= kThreads of a larger CTA only take part in the barriers.
template <int kThreads>
__device__ __forceinline__ void plan_body(int n_tiles, int T, int N, int K, const RouteBufs& rb) {
  __shared__ int s_chunk[kThreads];
  __shared__ double s_red[kThreads];
  __shared__ double s_p[128];
  __shared__ int s_counts[128];
  const bool in = threadIdx.x < kThreads;
  const int chunks = kThreads / N;  // chunks of tiles per expert
  const int per = (n_tiles + chunks - 1) / chunks;
  const int e = threadIdx.x % N;
  const int c = threadIdx.x / N;
  const bool act = in && c < chunks;
  const int t_begin = act ? min(n_tiles, c * per) : 0;
  const int t_end = act ? min(n_tiles, (c + 1) * per) : 0;
  int sum = 0;
  double ps = 0.0;
#pragma unroll 8
  for (int t = t_begin; t < t_end; ++t) {
    sum += rb.tile_cnt[(size_t)t * N + e];
    ps += rb.tile_psum[(size_t)t * N + e];
  }
  if (in) {
    s_chunk[threadIdx.x] = sum;
    s_red[threadIdx.x] = ps;
  }
  __syncthreads();
  if (threadIdx.x < N) {
    int run = 0;
    double p = 0.0;
    for (int cc = 0; cc < chunks; ++cc) {
      const int v = s_chunk[cc * N + threadIdx.x];
      s_chunk[cc * N + threadIdx.x] = run;
      run += v;
      p += s_red[cc * N + threadIdx.x];
    }
    s_counts[threadIdx.x] = run;
    s_p[threadIdx.x] = p;
    rb.counts[threadIdx.x] = run;
    rb.agg_prob[threadIdx.x] = static_cast<float>(p);
  }
  __syncthreads();
  {
    int run = act ? s_chunk[threadIdx.x] : 0;
    for (int t = t_begin; t < t_end; ++t) {
      const size_t i = (size_t)t * N + e;
      const int v = rb.tile_cnt[i];
      rb.tile_cnt[i] = run;
      run += v;
    }
  }
  // Z-loss: fixed-order two-level reduction of the per-tile lse^2 sums.
  double z = 0.0;
  for (int t = threadIdx.x; in && t < n_tiles; t += kThreads) z += rb.tile_lse2[t];
  __syncthreads();  // s_red's tile partial sums above are consumed
  if (in) s_red[threadIdx.x] = z;
  __syncthreads();
  for (int w = kThreads / 2; w > 0; w >>= 1) {
    if (threadIdx.x < w) s_red[threadIdx.x] += s_red[threadIdx.x + w];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    int off = 0;
    double aux = 0.0;
    for (int x = 0; x < N; ++x) {
      rb.offsets[x] = off;
      off += s_counts[x];
      aux += s_p[x] * static_cast<double>(s_counts[x]);
    }
    rb.offsets[N] = off;
    const double coef = static_cast<double>(N) / (static_cast<double>(T) * T * static_cast<double>(K));
    rb.losses[0] = static_cast<float>(coef * aux);
    rb.losses[1] = static_cast<float>(s_red[0] / static_cast<double>(T));
  }
}

// ---------------------------------------------------------------------------------------
// K1, warp-specialised latency variant (decode-size batches; replaces the barrier-paced ring of
// router_lat_kernel). Same chains (one thread per (token, expert), ascending l), fed by a deep
// ring so the chains never wait on global memory:
//   producer warp:  1-D TMA bulk copies, per ring slot, of the W_r chunk (one contiguous copy of
//                   the padded expert-major layout widen_router_kernel writes) and of each token's
//                   x chunk; completion on full[s]; sleeps while the ring is full;
//   converter warp: widens the slot's x chunk to fp64 once for all experts (F2F runs at
//                   15/clk/SM: kept off the chains' SM sub-partition), then publishes it;
//   chain warps:    per 256-step chunk, run the chain from a register ring filled 16 steps ahead
//                   (two steps per 16-byte load of each operand), then publish the slot as free.
//                   The next slot's flag is read when a chunk starts, so the check overlaps the
//                   chain instead of stalling it.
// The chain step is one asm block (the FMA, then on odd steps the two ring loads): measured 9.2
// cycles per step against 8.5 for operands already in registers and 11.9 for the [l][e] layout
// with a runtime stride (tools/chain_ring_probe.cu). Slot hand-offs use CTA-scope release/acquire
// flags in shared memory (mbarriers only for the TMA byte counts).
// kCons (chain threads) is 32, 64 or 128: the host picks the smallest that keeps one CTA per SM, so
// a decode batch spreads over the most SMs (dense decode pins 128: the router then runs beside
// GEMM1 and should hold few SMs). The per-token softmax / top-K runs one warp per token.
struct RouterWsSmem {
  static constexpr int kMaxStages = 12;
  static constexpr int kMaxChainWarps = 8;  // kCons <= 256: one eflag slot per chain warp
  static constexpr int kAhead = 16;  // ring distance (steps); loads run up to kAhead past a row
  int tpc, N4, chunk, wpitch, stages;
  size_t sw, rx, xd, bars, slog, sidx, slse, total;
  __host__ __device__ RouterWsSmem(int n_experts, int cons, int xb = 2) {
    N4 = (n_experts + 3) / 4 * 4;
    tpc = cons / N4;
    chunk = router_ws_chunk(N4);
    wpitch = chunk + 2;  // doubles per expert row
    // as many ring slots as ~200 KB allow (the producer runs several L2 round trips ahead)
    const size_t slot = (size_t)N4 * wpitch * 8 + ((size_t)tpc * chunk * xb + 15) / 16 * 16 + (size_t)tpc * chunk * 8;
    const size_t fixed = 4096;
    stages = (int)(((size_t)200 * 1024 - fixed) / slot);
    stages = stages < 2 ? 2 : stages > kMaxStages ? kMaxStages : stages;
    sw = 0;                                                          // [stages][N4][wpitch] fp64
    rx = sw + (size_t)stages * N4 * wpitch * 8;                      // [stages][tpc][chunk] bf16 / fp32
    xd = rx + ((size_t)stages * tpc * chunk * xb + 15) / 16 * 16;    // [stages][tpc][chunk] fp64
    bars = xd + (size_t)stages * tpc * chunk * 8;                    // full[kMaxStages] + flags
    // flags: xflag[kMaxStages] + eflag[kMaxChainWarps] (round 1 reserved only 4 eflag slots, so a
    // 256-thread instantiation's eflag[4..7] aliased slog[0..3]: the logits of the tile's token 0)
    slog = bars + kMaxStages * 8 + (kMaxStages + kMaxChainWarps) * 4;
    sidx = slog + sizeof(float) * tpc * N4;
    slse = (sidx + sizeof(int) * tpc * 8 + 7) / 8 * 8;
    total = slse + sizeof(double) * tpc + kAhead * 8;  // guard for the ring's overrun past the last row
  }
};

// One chain step: acc = fma(xx, ww, acc); on odd steps also the next x / W pairs of the ring.
__device__ __forceinline__ void ws_step(double& acc, double xx, double ww) {
  asm volatile("fma.rn.f64 %0, %1, %2, %0;" : "+d"(acc) : "d"(xx), "d"(ww));
}
__device__ __forceinline__ void ws_step_ld(double& acc, double xx, double ww, double& x0, double& x1, double& w0,
                                           double& w1, uint32_t xa, uint32_t wa) {
  asm volatile(
      "fma.rn.f64 %0, %5, %6, %0;\n\t"
      "ld.shared.v2.f64 {%1, %2}, [%7];\n\t"
      "ld.shared.v2.f64 {%3, %4}, [%8];"
      : "+d"(acc), "=d"(x0), "=d"(x1), "=d"(w0), "=d"(w1)
      : "d"(xx), "d"(ww), "r"(xa), "r"(wa)
      : "memory");
}

// Per-tile statistics of a router tile whose rows of slog now hold probs and sidx the top-K
// picks: one warp per expert over 32-token slices; a token's rank among the tile's tokens routed
// to e is the popcount of the earlier lanes' ballot (each token picks e at most once); the prob sum
// adds the tokens in ascending order, as router_finish. Called by all threads after a barrier.
__device__ __forceinline__ void router_tile_stats(int tile, int tok0, int ntok, int N, int N4, int K,
                                                  const float* slog, const int* sidx, const double* slse,
                                                  const RouteBufs& rb) {
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  constexpr unsigned kAll = 0xffffffffu;
  for (int e = warp; e < N; e += nwarps) {
    int cnt = 0;
    double ps = 0.0;
    for (int t0 = 0; t0 < ntok; t0 += 32) {
      const int t = t0 + lane;
      int kk = -1;
      double p = 0.0;
      if (t < ntok) {
        for (int k = 0; k < K; ++k)
          if (sidx[t * 8 + k] == e) kk = k;
        p = static_cast<double>(slog[t * N4 + e]);
      }
      const unsigned m = __ballot_sync(kAll, kk >= 0);
      if (kk >= 0) rb.local_rank[(size_t)(tok0 + t) * K + kk] = cnt + __popc(m & ((1u << lane) - 1u));
      cnt += __popc(m);
      const int n = min(32, ntok - t0);
      for (int i = 0; i < n; ++i) ps += __shfl_sync(kAll, p, i);
    }
    if (lane == 0) {
      rb.tile_cnt[(size_t)tile * N + e] = cnt;
      rb.tile_psum[(size_t)tile * N + e] = ps;
    }
  }
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int t = 0; t < ntok; ++t) a += slse[t];
    rb.tile_lse2[tile] = a;
  }
}

// Per-token softmax / top-K / combine weights with one warp per token (lanes own experts), then the
// per-tile statistics. Same arithmetic as router_finish: the max is order-free, the fp64 softmax
// denominator and the top-K weight sum are accumulated in ascending order (every lane runs the same
// sequence over shuffled terms), and top-K is an argmax with the lowest index winning ties. A row
// with a NaN probability takes the sequential path on lane 0 (its NaN semantics are positional).
__device__ __forceinline__ void router_finish_warps(int tile, int tok0, int tpc, int T, int N, int N4, int K,
                                                    float* slog, int* sidx, double* slse, const RouteBufs& rb) {
  const int ntok = min(tpc, T - tok0);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  constexpr unsigned kAll = 0xffffffffu;
  for (int tl = warp; tl < tpc; tl += nwarps) {
    double lse2 = 0.0;
    if (tl < ntok) {
      const int j = tok0 + tl;
      float* zrow = slog + tl * N4;
      double mx = zrow[0];
      for (int e = lane; e < N; e += 32) mx = fmax(mx, static_cast<double>(zrow[e]));
#pragma unroll
      for (int o = 16; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kAll, mx, o));
      double ex[4] = {0.0, 0.0, 0.0, 0.0};
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = q * 32 + lane;
        if (q * 32 < N && e < N) ex[q] = exp_glibc(static_cast<double>(zrow[e]) - mx);
      }
      // ascending-e sum: every lane adds the same shuffled terms in the same order
      double denom = 0.0;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        if (q * 32 >= N) break;
        const int nq = min(32, N - q * 32);
#pragma unroll 8
        for (int i = 0; i < nq; ++i) denom += __shfl_sync(kAll, ex[q], i);
      }
      float pv[4] = {0.0f, 0.0f, 0.0f, 0.0f};
      bool nan = false;
      __syncwarp();  // every lane has read zrow (logits) before it is overwritten with probs
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int e = q * 32 + lane;
        if (q * 32 >= N) break;
        pv[q] = static_cast<float>(ex[q] / denom);
        if (e < N) {
          rb.probs[(size_t)j * N + e] = pv[q];
          zrow[e] = pv[q];  // the row now holds probs
          nan |= isnan(pv[q]);
        }
      }
      const double lse = mx + log(denom);
      lse2 = lse * lse;
      if (!__any_sync(kAll, nan)) {
        // K rounds of a warp argmax: probs are >= +0 and not NaN, so their bit patterns order like
        // the values; the lowest index wins ties (the reference's strict '>' scan)
        unsigned taken = 0;  // bit q: this lane's expert q*32+lane is taken
        float myv = 0.0f;    // lane k keeps round k's winner
        int myi = 0;
        double sum = 0.0;    // sum of the winners in round order, as the reference
#pragma unroll
        for (int k = 0; k < 8; ++k) {
          if (k >= K) break;
          unsigned key = 0;
          int best = -1;
#pragma unroll
          for (int q = 0; q < 4; ++q) {
            const int e = q * 32 + lane;
            const unsigned kq = __float_as_uint(pv[q]);
            if (e < N && !((taken >> q) & 1u) && (best < 0 || kq > key)) { best = e; key = kq; }
          }
          const unsigned m = __reduce_max_sync(kAll, best >= 0 ? key : 0u);
          const int win = static_cast<int>(
              __reduce_min_sync(kAll, (best >= 0 && key == m) ? static_cast<unsigned>(best) : 0x7fffffffu));
          if ((win & 31) == lane) taken |= 1u << (win >> 5);
          const float bv = __uint_as_float(m);
          if (lane == k) {
            myv = bv;
            myi = win;
          }
          sum += static_cast<double>(bv);
        }
        if (lane < K) {
          rb.topk_idx[(size_t)j * K + lane] = myi;
          rb.combine_w[(size_t)j * K + lane] = static_cast<float>(static_cast<double>(myv) / sum);
          sidx[tl * 8 + lane] = myi;
        }
      } else if (lane == 0) {  // sequential reference order (rows with a NaN probability)
        float vals[8];
        int ids[8];
        uint64_t taken_lo = 0, taken_hi = 0;
        for (int k = 0; k < K; ++k) {
          int best = -1;
          float bv = 0.0f;
          for (int e = 0; e < N; ++e) {
            const bool tk = e < 64 ? ((taken_lo >> e) & 1ull) : ((taken_hi >> (e - 64)) & 1ull);
            if (tk) continue;
            const float v = zrow[e];
            if (best < 0 || v > bv) { best = e; bv = v; }
          }
          if (best < 64) taken_lo |= 1ull << best; else taken_hi |= 1ull << (best - 64);
          vals[k] = bv;
          ids[k] = best;
        }
        double sum = 0.0;
        for (int k = 0; k < K; ++k) sum += static_cast<double>(vals[k]);
        for (int k = 0; k < K; ++k) {
          rb.topk_idx[(size_t)j * K + k] = ids[k];
          rb.combine_w[(size_t)j * K + k] = static_cast<float>(static_cast<double>(vals[k]) / sum);
          sidx[tl * 8 + k] = ids[k];
        }
      }
    }
    if (lane == 0) slse[tl] = lse2;
  }
  __syncthreads();
  router_tile_stats(tile, tok0, ntok, N, N4, K, slog, sidx, slse, rb);
}

// tail_ctr (dense decode, nullable): the last CTA to finish also runs the plan (plan_body<128>)
// and the dense row weights / combine rows, so nothing queues behind GEMM1's persistent CTAs.
template <int kCons, typename XT = __nv_bfloat16>
__global__ void __launch_bounds__(kCons + 64, 1) router_ws_kernel(const XT* __restrict__ x,
                                                                 const double* __restrict__ wr64, int T, int d,
                                                                 int N, int K, RouteBufs rb,
                                                                 int* __restrict__ tail_ctr = nullptr,
                                                                 float* __restrict__ rwd = nullptr,
                                                                 int32_t* __restrict__ invd = nullptr,
                                                                 const float* __restrict__ xscale = nullptr) {
  constexpr int kD = RouterWsSmem::kAhead, kB = 32;
  static_assert(kCons % 32 == 0 && kCons / 32 <= RouterWsSmem::kMaxChainWarps, "eflag region holds one slot per chain warp");
  constexpr int kXB = sizeof(XT);
  const RouterWsSmem L(N, kCons, kXB);
  const int N4 = L.N4, tpc = L.tpc, chunk = L.chunk, wpitch = L.wpitch, kStages = L.stages;
  const double* wt = wr64 + (size_t)d * N4;  // per chunk [N4][wpitch] (widen_router_kernel)
  const int tok0 = blockIdx.x * tpc;
  const int ntok = min(tpc, T - tok0);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  double* sw = reinterpret_cast<double*>(smem_raw + L.sw);
  XT* rawx = reinterpret_cast<XT*>(smem_raw + L.rx);
  double* xd = reinterpret_cast<double*>(smem_raw + L.xd);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
  // the chain side synchronises through chunk-granular flags (CTA-scope release stores / acquire
  // loads) rather than mbarriers:
  //   xflag[s] = c + 1 once the converter has widened chunk c into slot s (release);
  //   eflag[w] = number of chunks chain warp w has finished (release).
  int* xflag = reinterpret_cast<int*>(full + RouterWsSmem::kMaxStages);
  int* eflag = xflag + RouterWsSmem::kMaxStages;
  float* slog = reinterpret_cast<float*>(smem_raw + L.slog);
  int* sidx = reinterpret_cast<int*>(smem_raw + L.sidx);
  double* slse = reinterpret_cast<double*>(smem_raw + L.slse);
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) {
      mbar_init(&full[s], 1);
      xflag[s] = 0;
    }
    for (int w = 0; w < kCons / 32; ++w) eflag[w] = 0;
    fence_mbar_init();
  }
  __syncthreads();
  const int nchunks = d / chunk;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  if (warp == kCons / 32 + 1) {  // producer
    if (lane == 0) {
      const uint32_t wbytes = N4 * wpitch * 8, xbytes = chunk * kXB;
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % kStages;
        if (c >= kStages)  // sleep-poll until every chain warp has finished chunk c - kStages
          for (int w = 0; w < kCons / 32; ++w)
            while (ld_acquire_cta(&eflag[w]) <= c - kStages) __nanosleep(128);
        mbar_arrive_expect_tx(&full[s], wbytes + ntok * xbytes);
        bulk_g2s(sw + (size_t)s * N4 * wpitch, wt + (size_t)c * N4 * wpitch, wbytes, &full[s]);
        for (int r = 0; r < ntok; ++r)
          bulk_g2s(rawx + ((size_t)s * tpc + r) * chunk, x + (size_t)(tok0 + r) * d + (size_t)c * chunk, xbytes,
                   &full[s]);
      }
    }
  } else if (warp == kCons / 32) {  // converter
    const float xsc = router_xscale(xscale);
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kStages;
      mbar_wait(&full[s], (c / kStages) & 1);
      const XT* rx = rawx + (size_t)s * tpc * chunk;
      double* xo = xd + (size_t)s * tpc * chunk;
      constexpr int kV = 16 / kXB;  // values per 16-byte load
      for (int i = lane * kV; i < ntok * chunk; i += 32 * kV) {
        double v[kV];
        widen16<XT>(*reinterpret_cast<const int4*>(rx + i), v, xsc);
#pragma unroll
        for (int j = 0; j < kV; j += 2) *reinterpret_cast<double2*>(xo + i + j) = make_double2(v[j], v[j + 1]);
      }
      __syncwarp();
      if (lane == 0) st_release_cta(&xflag[s], c + 1);  // publishes the widened x and, by cumulativity,
    }                                                    // the W chunk this warp acquired via full[s]
  } else {  // chain warps
    const int tl = threadIdx.x / N4, e = threadIdx.x % N4;
    const bool worker = tl < ntok;
    double acc = 0.0;
    bool ready = false;  // the current chunk's flag already observed (acquired) one chunk earlier
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kStages;
      if (!ready)
        while (ld_acquire_cta(&xflag[s]) <= c) {
        }
      // look at the next slot now: the flag read's latency overlaps this chunk's chain
      ready = c + 1 < nchunks && ld_acquire_cta(&xflag[(c + 1) % kStages]) > c + 1;
      if (worker) {
        const double* xr = xd + ((size_t)s * tpc + tl) * chunk;
        const double* we = sw + ((size_t)s * N4 + e) * wpitch;
        double xa[kD], wa[kD];
#pragma unroll
        for (int i = 0; i < kD; i += 2) {
          const double2 t = *reinterpret_cast<const double2*>(xr + i);
          const double2 u = *reinterpret_cast<const double2*>(we + i);
          xa[i] = t.x;
          xa[i + 1] = t.y;
          wa[i] = u.x;
          wa[i + 1] = u.y;
        }
        const uint32_t xs = smem_u32(xr), ws = smem_u32(we);
        // loads past the row end (last kD steps of the chunk) fill ring slots that are never consumed
#pragma unroll 1
        for (int b = 0; b < chunk; b += kB) {
          const uint32_t xq = xs + (b + kD) * 8, wq = ws + (b + kD) * 8;
#pragma unroll
          for (int i = 0; i < kB; ++i) {
            const double xx = xa[i % kD], ww = wa[i % kD];
            if (i & 1)
              ws_step_ld(acc, xx, ww, xa[(i - 1) % kD], xa[i % kD], wa[(i - 1) % kD], wa[i % kD], xq + (i - 1) * 8,
                         wq + (i - 1) * 8);
            else
              ws_step(acc, xx, ww);
          }
        }
      }
      __syncwarp();
      if (lane == 0) st_release_cta(&eflag[warp], c + 1);
    }
    if (worker) {
      const int tok = tok0 + tl;
      const float z = static_cast<float>(acc);
      slog[tl * N4 + e] = z;
      if (e < N) {
        rb.logits[(size_t)tok * N + e] = z;
        if (!isfinite(z)) atomicOr(rb.finite_flag, 1);
      }
    }
  }
  __syncthreads();
  router_finish_warps(blockIdx.x, tok0, tpc, T, N, N4, K, slog, sidx, slse, rb);
  if (tail_ctr) {
    __shared__ int s_last;
    __threadfence();  // this CTA's tile statistics and decisions, before the counter
    __syncthreads();
    if (threadIdx.x == 0) s_last = atomicAdd(tail_ctr, 1) == (int)gridDim.x - 1;
    __syncthreads();
    if (s_last) {
      __threadfence();
      plan_body<128>(gridDim.x, T, N, K, rb);
      for (int i = threadIdx.x; i < N * T; i += blockDim.x) {  // = dense_weights_kernel
        const int e = i / T, t = i % T;
        float v = 0.0f;
        for (int k = 0; k < K; ++k)
          if (rb.topk_idx[(size_t)t * K + k] == e) v = rb.combine_w[(size_t)t * K + k];
        rwd[i] = v;
      }
      for (int i = threadIdx.x; i < T * K; i += blockDim.x) invd[i] = rb.topk_idx[i] * T + i / K;
      if (threadIdx.x == 0) *tail_ctr = 0;  // ready for the next launch (stream-ordered)
    }
  }
}

// ---------------------------------------------------------------------------------------
// K1, large-batch variant: one thread owns 4 tokens x 4 experts (16 independent fp64 chains, each
// still summed over l in ascending order — bit-identical to the reference gemm_nn). x rows stay
// raw bf16 in shared memory (16-byte chunks XOR-swizzled by token group so the per-token 16-byte
// loads of a quarter-warp hit distinct banks) and are widened in registers, amortised over the
// 4 experts; the fp64 copy of W_r streams through a cp.async ring. Shared-memory traffic is
// ~1.25 wavefronts per 64 DFMA instead of ~5 in the 1x4 layout.
struct RouterBigSmem {
  int tpc, N4;
  size_t rx, sw, slog, sidx, slse, total;
  __host__ __device__ RouterBigSmem(int n_experts, int threads, int stages, int tok = 4, int xb = 2) {
    N4 = (n_experts + 3) / 4 * 4;
    tpc = (threads / (N4 / 4)) * tok;
    rx = 0;
    sw = rx + (size_t)stages * tpc * kRouterChunk * xb;
    slog = sw + (size_t)stages * sizeof(double) * kRouterChunk * N4;
    sidx = slog + sizeof(float) * tpc * N4;
    slse = (sidx + sizeof(int) * tpc * 8 + 7) / 8 * 8;
    total = slse + sizeof(double) * tpc;
  }
};

template <int kThreads, int kStages, int kTok = 4, typename XT = __nv_bfloat16>
__global__ void __launch_bounds__(kThreads, 1) router_big_kernel(const XT* __restrict__ x,
                                                                 const double* __restrict__ wr64, int T, int d, int N,
                                                                 int K, RouteBufs rb,
                                                                 const float* __restrict__ xscale = nullptr) {
  // a token's 64-column chunk: bf16 8 x 16 B (16-byte pieces swizzled by token group); fp32 16 x
  // 16 B swizzled in 32-byte pairs; e4m3 codes 4 x 16 B (each piece = two 8-value groups)
  constexpr int kXB = sizeof(XT), kRowB = kRouterChunk * kXB;
  constexpr int kP = kXB >= 2 ? kXB / 2 : 1;     // 16-byte pieces per 8-value group (e4m3: per 2 groups)
  constexpr int kPieces = kRowB / 16;            // pieces per row
  const float xsc = router_xscale(xscale);
  const RouterBigSmem L(N, kThreads, kStages, kTok, kXB);
  const int N4 = L.N4;
  const int groups = N4 / 4;
  const int tg_per_cta = kThreads / groups;
  const int tpc = L.tpc;
  const int tile = blockIdx.x;
  const int tok0 = tile * tpc;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* rawx = smem_raw + L.rx;                               // [stages][tpc][kRowB] swizzled
  double* sw = reinterpret_cast<double*>(smem_raw + L.sw);       // [stages][chunk][N4]
  float* slog = reinterpret_cast<float*>(smem_raw + L.slog);
  int* sidx = reinterpret_cast<int*>(smem_raw + L.sidx);
  double* slse = reinterpret_cast<double*>(smem_raw + L.slse);
  const int tg = threadIdx.x / groups;
  const int g = threadIdx.x % groups;
  const bool worker = tg < tg_per_cta;
  double acc[kTok][4];
#pragma unroll
  for (int a = 0; a < kTok; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;

  const int nchunks = d / kRouterChunk;
  const int xpieces = tpc * kPieces;  // 16-byte pieces per token row per stage
  const int wpieces = kRouterChunk * N4 / 2;
  auto issue = [&](int c, int buf) {
    const int c0 = c * kRouterChunk;
    for (int i = threadIdx.x; i < xpieces; i += kThreads) {
      const int r = i / kPieces, p = i % kPieces;
      const bool ok = tok0 + r < T;
      const XT* src = x + (size_t)(ok ? tok0 + r : 0) * d + c0 + p * (16 / kXB);
      int ps;
      if constexpr (kXB == 1) {
        ps = p ^ ((r / kTok) & 3);
      } else {
        const int q = p / kP, h = p % kP;  // 8-value group q, half h
        ps = (q ^ ((r / kTok) & 7)) * kP + h;
      }
      cp_async16(rawx + ((size_t)buf * tpc + r) * kRowB + ps * 16, src, ok);
    }
    const double* wsrc = wr64 + (size_t)c0 * N4;
    for (int i = threadIdx.x; i < wpieces; i += kThreads)
      cp_async16(sw + (size_t)buf * kRouterChunk * N4 + i * 2, wsrc + i * 2, true);
    cp_async_commit();
  };
  for (int c = 0; c < kStages - 1; ++c) {
    if (c < nchunks) issue(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kStages;
    cp_async_wait<kStages - 2>();
    __syncthreads();
    if (c + kStages - 1 < nchunks) issue(c + kStages - 1, (c + kStages - 1) % kStages);
    else cp_async_commit();
    if (worker) {
      const uint8_t* xb = rawx + (size_t)buf * tpc * kRowB;
      const double2* wv = reinterpret_cast<const double2*>(sw + (size_t)buf * kRouterChunk * N4 + g * 4);
#pragma unroll 1
      for (int q = 0; q < kRouterChunk / 8; ++q) {
        // 8 l-columns of the kTok tokens, widened to fp64 once for all 4 experts
        double xd[kTok][8];
#pragma unroll
        for (int a = 0; a < kTok; ++a) {
          const int r = tg * kTok + a;
          if constexpr (kXB == 1) {
            const uint2 raw = *reinterpret_cast<const uint2*>(xb + (size_t)r * kRowB + ((q >> 1) ^ ((r / kTok) & 3)) * 16 +
                                                              (q & 1) * 8);
            const uint8_t* cb = reinterpret_cast<const uint8_t*>(&raw);
#pragma unroll
            for (int i = 0; i < 8; ++i) xd[a][i] = x_to_f64<XT>(cb[i], xsc);
          } else {
            const uint8_t* g8 = xb + (size_t)r * kRowB + (q ^ ((r / kTok) & 7)) * kP * 16;
#pragma unroll
            for (int h = 0; h < kP; ++h)
              widen16<XT>(*reinterpret_cast<const int4*>(g8 + h * 16), &xd[a][h * (16 / kXB)]);
          }
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) {
          const int l = q * 8 + i;
          const double2 w01 = wv[l * (N4 / 2)];
          const double2 w23 = wv[l * (N4 / 2) + 1];
#pragma unroll
          for (int a = 0; a < kTok; ++a) {
            acc[a][0] = fma(xd[a][i], w01.x, acc[a][0]);
            acc[a][1] = fma(xd[a][i], w01.y, acc[a][1]);
            acc[a][2] = fma(xd[a][i], w23.x, acc[a][2]);
            acc[a][3] = fma(xd[a][i], w23.y, acc[a][3]);
          }
        }
      }
    }
  }
  __syncthreads();
  if (worker) {
#pragma unroll
    for (int a = 0; a < kTok; ++a) {
      const int tl = tg * kTok + a;
      const int tok = tok0 + tl;
#pragma unroll
      for (int b = 0; b < 4; ++b) {
        const int e = g * 4 + b;
        const float z = static_cast<float>(acc[a][b]);
        slog[tl * N4 + e] = z;
        if (tok < T && e < N) {
          rb.logits[(size_t)tok * N + e] = z;
          if (!isfinite(z)) atomicOr(rb.finite_flag, 1);
        }
      }
    }
  }
  __syncthreads();
  router_finish(tile, tok0, tpc, T, N, N4, K, slog, sidx, slse, rb, kThreads);
}

// ---------------------------------------------------------------------------------------
// K2: dispatch plan. Exclusive scan of the per-tile expert counts (tile-major within each
// expert) -> each tile's base row inside its expert segment; expert offsets; agg_prob, aux-loss
// and Z-loss reductions in a fixed order. One CTA; deterministic (no atomics).
// ---------------------------------------------------------------------------------------
// K1, fp64 tensor-core variant (large and mid-size batches). DMMA (mma.sync.m8n8k4.f64) computes
// D = C + A B over k = 0..3 as the sequential FMA chain fma(a3,b3, fma(a2,b2, fma(a1,b1,
// fma(a0,b0,c)))) — measured on this B200 (tools/dmma_probe.cu): bit-identical to the ascending-k
// chain on 1.5e9 outputs of bf16 x fp32 operands with a 2^40 exponent spread, where the
// descending chain or products-summed-first differ on 12-15 % of them. One DMMA is therefore four
// steps of the reference's ascending-l chain (tensor.cpp:157-173) for an 8-token x 8-expert block,
// with the accumulator carried across k-steps in registers: logits stay bit-identical by
// construction of the instruction's arithmetic, 256 FMAs per warp instruction instead of 32. The
// handle checks the instruction on the device before first use (dmma_selftest_kernel) and keeps
// the DFMA variants otherwise.
//   Warp: one 8-token tile x every 8-expert tile (kNT accumulator chains; C fragment: lane
//   holds C[lane/4][2(lane%4) + {0,1}]), so each x value is widened once per warp and feeds kNT
//   DMMAs. A DMMA occupies its sub-partition's FP64 pipe for 16 cycles and has a 26-cycle
//   dependent latency (tools/dmma_probe.cu), so CTAs are small (kW warps) and many. A fragment
//   (x, one value per lane: row lane/4, k = lane%4) is read from a row-padded smem copy of the x
//   chunk (rows 16 B apart in banks: conflict-free) and widened in registers; B fragments (W_r)
//   come pre-arranged in fragment order (widen_router_kernel's third layout: [d/4][N8/8][32]
//   fp64), one 8-byte load per lane. x and W chunks of kDmmaChunk steps stream through a
//   cp.async ring. The kernel writes logits only: the per-token softmax / top-K / tile statistics
//   run in router_finish_kernel with one warp per token (inside this kernel they would be a
//   serial tail of every CTA, ~30 us at C2).
constexpr int kDmmaChunk = 64;
constexpr int kDmmaStages = 4;
__host__ __device__ inline int dmma_n8(int N) { return (N + 7) / 8 * 8; }
// W_r fragment layout: after the [d][N4] copy and the router_ws layout inside the wr64 buffer
__host__ __device__ inline size_t router_wfrag_offset(int d, int N) {
  const int N4 = (N + 3) / 4 * 4, chunk = router_ws_chunk(N4);
  return (size_t)d * N4 + (size_t)(d / chunk) * N4 * (chunk + 2);
}
__host__ __device__ inline size_t router_w64_size(int d, int N) {  // doubles of the whole wr64 buffer
  return router_wfrag_offset(d, N) + (size_t)d * dmma_n8(N);
}
struct RouterDmmaSmem {
  int tpc, NT, xpitch;
  size_t sx, sw, total;
  __host__ __device__ RouterDmmaSmem(int n_experts, int warps, int xb) {
    NT = dmma_n8(n_experts) / 8;
    tpc = warps * 8;
    xpitch = kDmmaChunk * xb + 16;  // bytes per token row; +16: consecutive rows 4 banks apart
    sx = 0;                                                              // [stages][tpc][xpitch]
    sw = sx + (size_t)kDmmaStages * tpc * xpitch;                        // [stages][chunk/4][NT][32]
    total = sw + (size_t)kDmmaStages * (kDmmaChunk / 4) * NT * 32 * 8;
  }
};

__device__ __forceinline__ void dmma_f64(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0, %1}, {%2}, {%3}, {%0, %1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

template <int kNT, int kW, typename XT = __nv_bfloat16>
__global__ void __launch_bounds__(kW * 32) router_dmma_kernel(const XT* __restrict__ x,
                                                            const double* __restrict__ wfrag, int T, int d, int N,
                                                            RouteBufs rb, const float* __restrict__ xscale = nullptr) {
  constexpr int kXB = sizeof(XT), kThreads = kW * 32;
  const float xsc = router_xscale(xscale);
  const RouterDmmaSmem L(N, kW, kXB);
  const int tpc = L.tpc, xpitch = L.xpitch;
  const int tok0 = blockIdx.x * tpc;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* sx = smem_raw + L.sx;
  double* sw = reinterpret_cast<double*>(smem_raw + L.sw);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;

  const int nchunks = d / kDmmaChunk;
  constexpr int kRowPieces = kDmmaChunk * kXB / 16;          // 16-byte pieces of one token's x chunk
  constexpr int kWPieces = (kDmmaChunk / 4) * kNT * 32 / 2;  // 16-byte pieces of one W chunk
  auto issue = [&](int c, int buf) {
    const int c0 = c * kDmmaChunk;
    uint8_t* xdst = sx + (size_t)buf * tpc * xpitch;
    for (int i = threadIdx.x; i < tpc * kRowPieces; i += kThreads) {
      const int r = i / kRowPieces, q = i % kRowPieces;
      const bool ok = tok0 + r < T;
      const XT* src = x + (size_t)(ok ? tok0 + r : 0) * d + c0 + q * (16 / kXB);
      cp_async16(xdst + r * xpitch + q * 16, src, ok);
    }
    const double* wsrc = wfrag + (size_t)(c0 / 4) * kNT * 32;
    double* wdst = sw + (size_t)buf * (kDmmaChunk / 4) * kNT * 32;
    for (int i = threadIdx.x; i < kWPieces; i += kThreads) cp_async16(wdst + 2 * i, wsrc + 2 * i, true);
    cp_async_commit();
  };
#pragma unroll
  for (int c = 0; c < kDmmaStages - 1; ++c) {
    if (c < nchunks) issue(c, c);
    else cp_async_commit();
  }
  double acc[kNT][2];
#pragma unroll
  for (int g = 0; g < kNT; ++g) acc[g][0] = acc[g][1] = 0.0;
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kDmmaStages;
    cp_async_wait<kDmmaStages - 2>();
    __syncthreads();
    if (c + kDmmaStages - 1 < nchunks) issue(c + kDmmaStages - 1, (c + kDmmaStages - 1) % kDmmaStages);
    else cp_async_commit();
    const uint8_t* xs = sx + (size_t)buf * tpc * xpitch + (size_t)(warp * 8 + lane / 4) * xpitch + (lane % 4) * kXB;
    const double* ws = sw + (size_t)buf * (kDmmaChunk / 4) * kNT * 32 + lane;
#pragma unroll 8
    for (int j = 0; j < kDmmaChunk / 4; ++j) {
      const double a = x_to_f64<XT>(*reinterpret_cast<const XT*>(xs + j * 4 * kXB), xsc);
#pragma unroll
      for (int g = 0; g < kNT; ++g) dmma_f64(acc[g][0], acc[g][1], a, ws[(j * kNT + g) * 32]);
    }
  }
  // logits: C fragment row lane/4 of this warp's token tile, columns 2(lane%4) + {0,1} of tile g
  const int tok = tok0 + warp * 8 + lane / 4;
  if (tok < T) {
#pragma unroll
    for (int g = 0; g < kNT; ++g)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int e = g * 8 + 2 * (lane % 4) + h;
        if (e < N) {
          const float z = static_cast<float>(acc[g][h]);
          rb.logits[(size_t)tok * N + e] = z;
          if (!isfinite(z)) atomicOr(rb.finite_flag, 1);
        }
      }
  }
}

// router_finish_warps for N <= 16 with two tokens per warp (one per 16-lane half; lane = expert):
// the same operations in the same order — max (fmax, NaN-ignoring, from the row's first logit),
// exp_glibc, ascending-e fp64 denominator, one division per probability, K argmax rounds with the
// lowest index winning ties (here a half-warp butterfly on (bits, index)), the winners' sum in
// round order — so the results are bit-identical; half the warp instructions per token. tpc even.
__device__ __forceinline__ void router_finish_half(int tile, int tok0, int tpc, int T, int N, int N4, int K,
                                                   float* slog, int* sidx, double* slse, const RouteBufs& rb) {
  const int ntok = min(tpc, T - tok0);
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32, nwarps = blockDim.x / 32;
  const int seg = lane >> 4, sl = lane & 15;
  constexpr unsigned kAll = 0xffffffffu;
  for (int tb = warp * 2; tb < tpc; tb += nwarps * 2) {
    const int tl = tb + seg;
    const bool tv = tl < ntok;   // uniform within the half
    const bool ev = tv && sl < N;
    const int j = tok0 + tl;
    float* zrow = slog + tl * N4;
    const float z = ev ? zrow[sl] : 0.0f;
    double mx = tv ? static_cast<double>(zrow[0]) : 0.0;
    if (ev) mx = fmax(mx, static_cast<double>(z));
#pragma unroll
    for (int o = 8; o; o >>= 1) mx = fmax(mx, __shfl_xor_sync(kAll, mx, o));
    const double ex = ev ? exp_glibc(static_cast<double>(z) - mx) : 0.0;
    double denom = 0.0;
    for (int i = 0; i < N; ++i) denom += __shfl_sync(kAll, ex, (seg << 4) + i);
    __syncwarp();  // every lane has read zrow (logits) before it is overwritten with probs
    float pv = 0.0f;
    bool nan = false;
    if (ev) {
      pv = static_cast<float>(ex / denom);
      rb.probs[(size_t)j * N + sl] = pv;
      zrow[sl] = pv;
      nan = isnan(pv);
    }
    const double lse = mx + log(denom);
    const double lse2 = tv ? lse * lse : 0.0;
    const bool segnan = ((__ballot_sync(kAll, nan) >> (seg << 4)) & 0xffffu) != 0;
    __syncwarp();
    if (!segnan) {
      bool taken = false;
      float myv = 0.0f;
      int myi = 0;
      double sum = 0.0;
#pragma unroll
      for (int k = 0; k < 8; ++k) {
        if (k >= K) break;
        unsigned key = (ev && !taken) ? __float_as_uint(pv) : 0u;
        int idx = (ev && !taken) ? sl : 0x7fffffff;
#pragma unroll
        for (int o = 8; o; o >>= 1) {
          const unsigned ok = __shfl_xor_sync(kAll, key, o);
          const int oi = __shfl_xor_sync(kAll, idx, o);
          if (ok > key || (ok == key && oi < idx)) {
            key = ok;
            idx = oi;
          }
        }
        if (idx == sl) taken = true;
        const float bv = __uint_as_float(key);
        if (sl == k) {
          myv = bv;
          myi = idx;
        }
        sum += static_cast<double>(bv);
      }
      if (tv && sl < K) {
        rb.topk_idx[(size_t)j * K + sl] = myi;
        rb.combine_w[(size_t)j * K + sl] = static_cast<float>(static_cast<double>(myv) / sum);
        sidx[tl * 8 + sl] = myi;
      }
    } else if (tv && sl == 0) {  // sequential reference order (rows with a NaN probability)
      float vals[8];
      int ids[8];
      unsigned taken_bits = 0;
      for (int k = 0; k < K; ++k) {
        int best = -1;
        float bv = 0.0f;
        for (int e = 0; e < N; ++e) {
          if ((taken_bits >> e) & 1u) continue;
          const float v = zrow[e];
          if (best < 0 || v > bv) { best = e; bv = v; }
        }
        taken_bits |= 1u << best;
        vals[k] = bv;
        ids[k] = best;
      }
      double sum = 0.0;
      for (int k = 0; k < K; ++k) sum += static_cast<double>(vals[k]);
      for (int k = 0; k < K; ++k) {
        rb.topk_idx[(size_t)j * K + k] = ids[k];
        rb.combine_w[(size_t)j * K + k] = static_cast<float>(static_cast<double>(vals[k]) / sum);
        sidx[tl * 8 + k] = ids[k];
      }
    }
    if (sl == 0) slse[tl] = lse2;
  }
  __syncthreads();
  router_tile_stats(tile, tok0, ntok, N, N4, K, slog, sidx, slse, rb);
}

// Softmax / top-K / combine weights / tile statistics of router tiles whose logits are already in
// rb.logits (router_dmma_kernel): one CTA per tile of router_finish_tpc(N) tokens, one warp per
// token (two for N <= 16, router_finish_half).
// tokens per finish tile (the plan's router tile on this path) and threads: 32 tokens on 16 warps
// (two per warp) for N <= 16, else 16 tokens on 16 warps; fewer, larger tiles keep the plan's
// serial scan short
__host__ __device__ inline int router_finish_tpc(int N) { return N <= 16 ? 32 : 16; }
__host__ __device__ inline int router_finish_threads(int) { return 512; }
__global__ void __launch_bounds__(512) router_finish_kernel(int T, int N, int K, int tpc, RouteBufs rb) {
  extern __shared__ __align__(16) uint8_t smem_raw[];
  const int N4 = (N + 3) / 4 * 4;
  float* slog = reinterpret_cast<float*>(smem_raw);                                  // [tpc][N4]
  int* sidx = reinterpret_cast<int*>(smem_raw + sizeof(float) * tpc * N4);          // [tpc][8]
  double* slse = reinterpret_cast<double*>(smem_raw + ((sizeof(float) * tpc * N4 + sizeof(int) * tpc * 8 + 7) / 8 * 8));
  const int tok0 = blockIdx.x * tpc;
  const int ntok = min(tpc, T - tok0);
  for (int i = threadIdx.x; i < tpc * N4; i += blockDim.x) {
    const int t = i / N4, e = i % N4;
    slog[i] = (t < ntok && e < N) ? rb.logits[(size_t)(tok0 + t) * N + e] : 0.0f;
  }
  __syncthreads();
  if (N <= 16) router_finish_half(blockIdx.x, tok0, tpc, T, N, N4, K, slog, sidx, slse, rb);
  else router_finish_warps(blockIdx.x, tok0, tpc, T, N, N4, K, slog, sidx, slse, rb);
}
__host__ __device__ inline size_t router_finish_smem(int N, int tpc) {
  const int N4 = (N + 3) / 4 * 4;
  return (sizeof(float) * tpc * N4 + sizeof(int) * tpc * 8 + 7) / 8 * 8 + sizeof(double) * tpc;
}

// Device check of the DMMA accumulation order, run once per handle before router_dmma_kernel is
// used: random bf16 x fp32 operands (exponents over 2^+-20) through one m8n8k4 DMMA per trial vs
// the sequential FMA chain; *bad counts mismatching outputs.
__global__ void dmma_selftest_kernel(int trials, unsigned long long* bad) {
  const int lane = threadIdx.x % 32;
  unsigned long long nb = 0;
  uint64_t st = 0x243f6a8885a308d3ull ^ ((uint64_t)(blockIdx.x * blockDim.x + threadIdx.x - lane) << 17);
  auto next = [&]() {
    st += 0x9e3779b97f4a7c15ull;
    uint64_t z = st;
    z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
    z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
    return z ^ (z >> 31);
  };
  for (int it = 0; it < trials; ++it) {
    const uint64_t ra = next(), rb = next(), rc = next(), rd = next();
    // per-lane values from the warp-common stream, mixed with the lane id
    const uint64_t ua = ra * (2 * lane + 1) + (rb >> 7), ub = rb * (2 * lane + 3) + (rc >> 9);
    const uint64_t uc = rc * (2 * lane + 5) + (rd >> 5), ud = rd * (2 * lane + 7) + (ra >> 3);
    const float fa = ldexpf(1.0f + (float)((ua >> 8) & 0xff) / 256.0f, (int)(ua % 41) - 20) * ((ua >> 40) & 1 ? -1.f : 1.f);
    const double a = static_cast<double>(__uint_as_float(__float_as_uint(fa) & 0xffff0000u));  // bf16 value
    const double b = static_cast<double>(ldexpf(1.0f + (float)((ub >> 8) & 0xffffff) / 16777216.0f,
                                                (int)(ub % 41) - 20) * ((ub >> 40) & 1 ? -1.f : 1.f));
    double c0 = static_cast<double>(ldexpf(1.0f + (float)((uc >> 8) & 0xffffff) / 16777216.0f, (int)(uc % 41) - 20));
    double c1 = -static_cast<double>(ldexpf(1.0f + (float)((ud >> 8) & 0xffffff) / 16777216.0f, (int)(ud % 41) - 20));
    double s0 = c0, s1 = c1;
    const int row = lane / 4, col = 2 * (lane % 4);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const double ak = __shfl_sync(0xffffffffu, a, row * 4 + k);
      s0 = __fma_rn(ak, __shfl_sync(0xffffffffu, b, col * 4 + k), s0);
      s1 = __fma_rn(ak, __shfl_sync(0xffffffffu, b, (col + 1) * 4 + k), s1);
    }
    dmma_f64(c0, c1, a, b);
    nb += (__double_as_longlong(c0) != __double_as_longlong(s0)) + (__double_as_longlong(c1) != __double_as_longlong(s1));
  }
  if (nb) atomicAdd(bad, nb);
}

template <int kThreads>
__global__ void __launch_bounds__(kThreads) plan_kernel(int n_tiles, int T, int N, int K, RouteBufs rb) {
  plan_body<kThreads>(n_tiles, T, N, K, rb);
}

// ---------------------------------------------------------------------------------------
// Plan for an externally supplied routing decision (SPEC moe_forward(hidden, decision)): per
// tile counts + local ranks, same tile geometry as the router.
__global__ void decision_tiles_kernel(const int32_t* __restrict__ idx, int T, int N, int K, int tpc,
                                      RouteBufs rb) {
  const int tile = blockIdx.x;
  const int tok0 = tile * tpc;
  const int ntok = min(tpc, T - tok0);
  for (int e = threadIdx.x; e < N; e += blockDim.x) {
    int cnt = 0;
    for (int t = 0; t < ntok; ++t)
      for (int k = 0; k < K; ++k) {
        const size_t s = (size_t)(tok0 + t) * K + k;
        if (idx[s] == e) rb.local_rank[s] = cnt++;
      }
    rb.tile_cnt[(size_t)tile * N + e] = cnt;
    rb.tile_psum[(size_t)tile * N + e] = 0.0;
  }
  if (threadIdx.x == 0) rb.tile_lse2[tile] = 0.0;
}

constexpr int kMaxArriveExperts = 128;
// End of a dispatch CTA with arrival counters: every thread has fenced its own peer stores; after
// the barrier one thread per expert publishes the CTA's piece count with a system-scope release.
__device__ __forceinline__ void dispatch_arrive_tail(uint32_t* const* expert_arrive, int N, uint32_t* s_arr) {
  __threadfence_system();
  __syncthreads();
  for (int g = threadIdx.x; g < N; g += blockDim.x) {
    const uint32_t c = s_arr[g];
    if (c && expert_arrive[g]) {
      __threadfence_system();
      red_release_sys_add(expert_arrive[g], c);
    }
  }
}

// ---------------------------------------------------------------------------------------
// K3: fused permute/dispatch ("memcpy elimination"). One warp per token: the
// token row is read once and written straight into each of its K expert-contiguous rows of the
// GEMM1 operand (row r = offsets[e] + tile_base[tile][e] + local_rank), and the permutation
// metadata (perm, inv, per-row combine weight) is emitted alongside. Replaces gather_rows
// (proj/src/tensor.cpp:784-812) for every expert at once. kFp8: the row is quantised to E4M3
// on the fly with the destination expert's activation scale.
template <bool kFp8>
__global__ void __launch_bounds__(256) dispatch_kernel(const __nv_bfloat16* __restrict__ x, int T, int d, int N,
                                                       int K, int tpc, RouteBufs rb, const int32_t* __restrict__ idx,
                                                       const float* __restrict__ wts, void* __restrict__ xperm,
                                                       int32_t* __restrict__ perm, int32_t* __restrict__ inv,
                                                       float* __restrict__ row_w, const float* __restrict__ act_scale,
                                                       void* const* __restrict__ expert_dst = nullptr,
                                                       float* const* __restrict__ expert_dst_w = nullptr,
                                                       uint32_t* const* __restrict__ expert_arrive = nullptr,
                                                       const int32_t* __restrict__ dst_poff = nullptr) {
  // expert_dst (peer transport, ep.cuh): row r of expert e goes to expert_dst[e] + (r - offsets[e])
  // rows — the owner's receive buffer over NVLink — instead of xperm; null entries (overflow) skip.
  // expert_arrive (dispatch overlapped with the owners' GEMM1): after its stores the CTA adds the
  // number of (row, column-slice) pieces it wrote for each expert to the owner's arrival counter
  // (system-scope release), which the owner's GEMM1 producer acquires before loading the rows.
  // dst_poff (training, single GPU): xperm is the padded row layout, expert e's rows from
  // dst_poff[e] (the weight-gradient operand, read by GEMM1 through GemmArgs::a_poff); perm / inv /
  // row_w stay in the row layout.
  __shared__ uint32_t s_arr[kMaxArriveExperts];
  if (expert_arrive) {
    for (int g = threadIdx.x; g < N; g += blockDim.x) s_arr[g] = 0;
    __syncthreads();
  }
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= T) {
    if (expert_arrive) dispatch_arrive_tail(expert_arrive, N, s_arr);
    return;
  }
  const int tile = j / tpc;
  int rows[8];
  float sc[8];
  void* dsts[8];
  for (int k = 0; k < K; ++k) {
    const size_t s = (size_t)j * K + k;
    const int e = idx[s];
    const int r = rb.offsets[e] + rb.tile_cnt[(size_t)tile * N + e] + rb.local_rank[s];
    rows[k] = r;
    constexpr int kRowElemBytes = kFp8 ? 1 : 2;
    if (expert_dst) {
      char* b = static_cast<char*>(expert_dst[e]);
      dsts[k] = b ? b + (size_t)(r - rb.offsets[e]) * d * kRowElemBytes : nullptr;
      if (lane == 0 && b && blockIdx.y == 0) expert_dst_w[e][r - rb.offsets[e]] = wts[s];
    } else {
      const size_t pr = dst_poff ? (size_t)(dst_poff[e] + (r - rb.offsets[e])) : (size_t)r;
      dsts[k] = static_cast<char*>(xperm) + pr * d * kRowElemBytes;
    }
    if constexpr (kFp8) sc[k] = act_scale[e];
    if (lane == 0 && blockIdx.y == 0) {
      inv[s] = r;
      perm[r] = static_cast<int32_t>(s);
      row_w[r] = wts[s];
    }
    if (expert_arrive && lane == 0 && dsts[k]) atomicAdd(&s_arr[e], 1u);
  }
  const int4* src = reinterpret_cast<const int4*>(x + (size_t)j * d);
  // gridDim.y column slices (small batches: more warps in flight than tokens)
  const int nvec_all = d / 8;  // 8 bf16 per 16 B
  const int per = (nvec_all + gridDim.y - 1) / gridDim.y;
  const int vbeg = blockIdx.y * per;
  const int nvec = min(nvec_all, vbeg + per);
  if constexpr (!kFp8) {
    for (int v0 = vbeg + lane; v0 < nvec; v0 += 32 * 4) {
      int4 buf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u * 32 < nvec) buf[u] = ld_nc_v4(src + v0 + u * 32);
      for (int k = 0; k < K; ++k) {
        int4* dst = static_cast<int4*>(dsts[k]);
        if (!dst) continue;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + u * 32 < nvec) st_na_v4(dst + v0 + u * 32, buf[u]);
      }
    }
  } else {
    for (int v0 = vbeg + lane; v0 < nvec; v0 += 32 * 4) {  // 4 independent 16-byte loads in flight
      int4 buf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u * 32 < nvec) buf[u] = ld_nc_v4(src + v0 + u * 32);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int v = v0 + u * 32;
        if (v >= nvec) break;
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&buf[u]);
        float f[8];
#pragma unroll
        for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(h[i]);
        for (int k = 0; k < K; ++k) {
          uint32_t p[2];
#pragma unroll
          for (int i = 0; i < 2; ++i) {
            // x / scale with IEEE division, then RNE + saturate to E4M3 (SPEC.md:523-531 fp8_qdq)
            const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                make_float2(__fdiv_rn(f[4 * i], sc[k]), __fdiv_rn(f[4 * i + 1], sc[k])), __NV_SATFINITE, __NV_E4M3);
            const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                make_float2(__fdiv_rn(f[4 * i + 2], sc[k]), __fdiv_rn(f[4 * i + 3], sc[k])), __NV_SATFINITE,
                __NV_E4M3);
            p[i] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
          }
          if (!dsts[k]) continue;
          uint2* dst = static_cast<uint2*>(dsts[k]) + v;
          *dst = make_uint2(p[0], p[1]);
        }
      }
    }
  }
  if (expert_dst) __threadfence_system();  // peer stores visible before the exchange barrier
  if (expert_arrive) dispatch_arrive_tail(expert_arrive, N, s_arr);
}

// ---------------------------------------------------------------------------------------
// Dense decode (T <= 128 tokens, host_forward.cuh run_forward): every expert takes all T tokens,
// so GEMM1 can start before routing is known. Row e*T + t of the GEMM1 operand is token t, as
// bf16 or E4M3-quantised with expert e's activation scale exactly as dispatch_kernel does it.
// One warp per row; block 0 also writes the expert offsets e*T.
template <bool kFp8>
__global__ void __launch_bounds__(256) dense_dispatch_kernel(const __nv_bfloat16* __restrict__ x, int T, int d, int N,
                                                             void* __restrict__ xd, const float* __restrict__ act_scale,
                                                             int32_t* __restrict__ offd) {
  if (blockIdx.x == 0 && blockIdx.y == 0 && threadIdx.x <= N) offd[threadIdx.x] = threadIdx.x * T;
  const int row = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (row >= N * T) return;
  const int e = row / T, t = row % T;
  const int4* src = reinterpret_cast<const int4*>(x + (size_t)t * d);
  // gridDim.y column slices, 4 independent 16-byte loads in flight per lane
  const int nvec_all = d / 8;
  const int per = (nvec_all + gridDim.y - 1) / gridDim.y;
  const int vbeg = blockIdx.y * per, vend = min(nvec_all, vbeg + per);
  for (int v0 = vbeg + lane; v0 < vend; v0 += 32 * 4) {
    int4 buf[4];
#pragma unroll
    for (int u = 0; u < 4; ++u)
      if (v0 + u * 32 < vend) buf[u] = ld_nc_v4(src + v0 + u * 32);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int v = v0 + u * 32;
      if (v >= vend) break;
      if constexpr (!kFp8) {
        st_na_v4(reinterpret_cast<int4*>(static_cast<__nv_bfloat16*>(xd) + (size_t)row * d) + v, buf[u]);
      } else {
        const float sc = act_scale[e];
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&buf[u]);
        uint32_t p[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {  // x / scale (IEEE division), RNE + saturate: as dispatch_kernel
          const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
              make_float2(__fdiv_rn(__bfloat162float(h[4 * i]), sc), __fdiv_rn(__bfloat162float(h[4 * i + 1]), sc)),
              __NV_SATFINITE, __NV_E4M3);
          const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
              make_float2(__fdiv_rn(__bfloat162float(h[4 * i + 2]), sc), __fdiv_rn(__bfloat162float(h[4 * i + 3]), sc)),
              __NV_SATFINITE, __NV_E4M3);
          p[i] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        reinterpret_cast<uint2*>(static_cast<uint8_t*>(xd) + (size_t)row * d)[v] = make_uint2(p[0], p[1]);
      }
    }
  }
}

// Dense decode, once routing is known: GEMM2 row weights (the combine weight of (t, e) when e is
// among t's top-K, else 0) and the combine rows inv[t*K + k] = e_k*T + t.
__global__ void dense_weights_kernel(const int32_t* __restrict__ idx, const float* __restrict__ w, int T, int N, int K,
                                     float* __restrict__ rwd, int32_t* __restrict__ invd) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < N * T) {
    const int e = i / T, t = i % T;
    float v = 0.0f;
    for (int k = 0; k < K; ++k)
      if (idx[(size_t)t * K + k] == e) v = w[(size_t)t * K + k];
    rwd[i] = v;
  }
  if (i < T * K) invd[i] = idx[i] * T + i / K;
}

// ---------------------------------------------------------------------------------------
// K6: weighted combine / un-permute. One warp per token: out[j] = sum_k Y[inv[j,k]] in fp32, slot
// order (rows of Y already carry the combine weight from the GEMM2 epilogue). Replaces
// scatter_add_rows + add (proj/src/tensor.cpp:814-845, :248-262) with no intermediate copies.
// kK is compile-time so all K x kU 16-byte loads of a lane are in flight together.
// `wts` (nullable): multiply row k by wts[j*K+k] here (expert-parallel path, where the expert
// side returns unweighted rows).
template <typename OutT, int kK>
__global__ void __launch_bounds__(256) combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ inv,
                                                      int T, int d, OutT* __restrict__ out,
                                                      int32_t* __restrict__ finite_flag, const float* __restrict__ wts) {
  constexpr int kU = kK <= 2 ? 4 : 2;
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= T) return;
  const int4* src[kK];
#pragma unroll
  for (int k = 0; k < kK; ++k) src[k] = reinterpret_cast<const int4*>(y + (size_t)inv[(size_t)j * kK + k] * d);
  float wk[kK];
#pragma unroll
  for (int k = 0; k < kK; ++k) wk[k] = wts ? wts[(size_t)j * kK + k] : 1.0f;
  const int nvec_all = d / 8;
  const int per = (nvec_all + gridDim.y - 1) / gridDim.y;  // gridDim.y column slices (small batches)
  const int vbeg = blockIdx.y * per;
  const int nvec = min(nvec_all, vbeg + per);
  bool fin = true;
  for (int v0 = vbeg + lane; v0 < nvec; v0 += 32 * kU) {
    int4 raw[kU][kK];
#pragma unroll
    for (int u = 0; u < kU; ++u)
#pragma unroll
      for (int k = 0; k < kK; ++k)
        if (v0 + u * 32 < nvec) raw[u][k] = ld_nc_v4(src[k] + v0 + u * 32);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int v = v0 + u * 32;
      if (v >= nvec) break;
      float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
      for (int k = 0; k < kK; ++k) {
        const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw[u][k]);
#pragma unroll
        for (int i = 0; i < 8; ++i) acc[i] += wts ? wk[k] * __bfloat162float(h[i]) : __bfloat162float(h[i]);
      }
#pragma unroll
      for (int i = 0; i < 8; ++i) fin &= isfinite(acc[i]);
      if constexpr (sizeof(OutT) == 2) {
        int4 o;
        o.x = pack_bf16(acc[0], acc[1]);
        o.y = pack_bf16(acc[2], acc[3]);
        o.z = pack_bf16(acc[4], acc[5]);
        o.w = pack_bf16(acc[6], acc[7]);
        st_na_v4(reinterpret_cast<int4*>(out + (size_t)j * d) + v, o);
      } else {
        float4* o = reinterpret_cast<float4*>(out + (size_t)j * d) + 2 * v;
        o[0] = make_float4(acc[0], acc[1], acc[2], acc[3]);
        o[1] = make_float4(acc[4], acc[5], acc[6], acc[7]);
      }
    }
  }
  if (!fin) atomicOr(finite_flag, 1);
}

// K2 launch: a 128-thread CTA when there are few tiles (decode: fewer warps, cheaper barriers),
// 1024 threads otherwise. The fixed-order reductions depend only on (n_tiles, N).
inline void launch_plan(int n_tiles, int T, int N, int K, const RouteBufs& rb, cudaStream_t st) {
  if (n_tiles * N <= 1024)
    plan_kernel<128><<<1, 128, 0, st>>>(n_tiles, T, N, K, rb);
  else
    plan_kernel<kPlanThreads><<<1, kPlanThreads, 0, st>>>(n_tiles, T, N, K, rb);
}

// Warp-per-token kernels (dispatch, combine): (T/8) x slices CTAs of 8 warps; small batches get
// up to 8 column slices per token so a few hundred warps are in flight.
constexpr int kTargetSms = 148;  // B200 (sm_100a, the only target): sizing hint, not a correctness bound
inline dim3 token_grid(int64_t T) {
  const int blocks = static_cast<int>((T + 7) / 8);
  const int slices = std::max(1, std::min(8, (4 * kTargetSms + blocks - 1) / blocks));
  return dim3(blocks, slices);
}

template <typename OutT>
inline void launch_combine(const __nv_bfloat16* y, const int32_t* inv, int T, int d, int K, OutT* out, int32_t* flag,
                           cudaStream_t st, const float* wts = nullptr) {
  const dim3 blocks = token_grid(T);
  switch (K) {
    case 1: combine_kernel<OutT, 1><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    case 2: combine_kernel<OutT, 2><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    case 3: combine_kernel<OutT, 3><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    case 4: combine_kernel<OutT, 4><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    case 5: combine_kernel<OutT, 5><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    case 6: combine_kernel<OutT, 6><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    case 7: combine_kernel<OutT, 7><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
    default: combine_kernel<OutT, 8><<<blocks, 256, 0, st>>>(y, inv, T, d, out, flag, wts); break;
  }
}

}  // namespace cmoe
