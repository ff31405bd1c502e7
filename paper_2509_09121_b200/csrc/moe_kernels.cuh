// Router (K1), dispatch plan (K2), fused permute/dispatch (K3) and weighted combine (K6)
// kernels of the MoE layer. All are memory- or latency-bound; see DESIGN.md for their rooflines.
#pragma once
#include <cuda_fp8.h>

#include "ptx.cuh"

namespace cmoe {

constexpr int kRouterThreads = 128;
constexpr int kRouterChunk = 64;  // d-columns staged per step
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
  int32_t* finite_flag; // [1] set to 1 on any non-finite router logit (K11)
};

__host__ __device__ inline int router_tokens_per_cta(int n_experts) {
  const int groups = (n_experts + 3) / 4;  // one thread per (token, 4 experts)
  return kRouterThreads / groups;
}

// ---------------------------------------------------------------------------------------
// K1: router. logits = x W_r with one fp64 accumulator per (token, expert) summed over the
// hidden dimension in ascending order — the exact accumulation order of the reference gemm_nn
// (proj/src/tensor.cpp:157-173), so logits are bit-identical to the CPU oracle (each product of
// two floats is exact in fp64, hence FMA == multiply-then-add). Then per token: softmax in fp64
// (tensor.cpp:614-621), top-K with lowest-index tie-break (tensor.cpp:1046-1060), renormalised
// combine weights, per-tile expert counts and local ranks for the stable
// dispatch permutation, and per-tile partial sums for agg_prob (col_sums, tensor.cpp:545-565) and
// the Z-loss (tensor.cpp:1011-1040).
__global__ void __launch_bounds__(kRouterThreads) router_kernel(const __nv_bfloat16* __restrict__ x,
                                                                const float* __restrict__ wr, int T, int d,
                                                                int N, int K, RouteBufs rb) {
  const int groups = (N + 3) / 4;
  const int tpc = kRouterThreads / groups;  // tokens per CTA
  const int tile = blockIdx.x;
  const int tok0 = tile * tpc;
  extern __shared__ uint8_t smem_raw[];
  float* sx = reinterpret_cast<float*>(smem_raw);                      // [tpc][kRouterChunk+1]
  float* sw = sx + tpc * (kRouterChunk + 1);                           // [kRouterChunk][N4]
  const int N4 = groups * 4;
  float* slog = sw + kRouterChunk * N4;                                // [tpc][N4]

  const int t_local = threadIdx.x / groups;
  const int g = threadIdx.x % groups;
  const int tok = tok0 + t_local;
  const bool active = t_local < tpc && tok < T;
  double acc[4] = {0.0, 0.0, 0.0, 0.0};

  for (int c0 = 0; c0 < d; c0 += kRouterChunk) {
    const int cw = min(kRouterChunk, d - c0);
    // stage x[tok0 .. tok0+tpc) x [c0, c0+cw) as fp32, padded rows (bank-conflict free)
    for (int i = threadIdx.x; i < tpc * kRouterChunk; i += kRouterThreads) {
      const int r = i / kRouterChunk, c = i % kRouterChunk;
      float v = 0.0f;
      if (tok0 + r < T && c < cw) v = __bfloat162float(x[(size_t)(tok0 + r) * d + c0 + c]);
      sx[r * (kRouterChunk + 1) + c] = v;
    }
    for (int i = threadIdx.x; i < kRouterChunk * N4; i += kRouterThreads) {
      const int l = i / N4, e = i % N4;
      sw[i] = (l < cw && e < N) ? wr[(size_t)(c0 + l) * N + e] : 0.0f;
    }
    __syncthreads();
    if (t_local < tpc) {
      const float* xr = sx + t_local * (kRouterChunk + 1);
      const float4* wv = reinterpret_cast<const float4*>(sw) + g;
      for (int l = 0; l < cw; ++l) {
        const double xv = static_cast<double>(xr[l]);
        const float4 w4 = wv[l * groups];
        acc[0] = fma(xv, static_cast<double>(w4.x), acc[0]);
        acc[1] = fma(xv, static_cast<double>(w4.y), acc[1]);
        acc[2] = fma(xv, static_cast<double>(w4.z), acc[2]);
        acc[3] = fma(xv, static_cast<double>(w4.w), acc[3]);
      }
    }
    __syncthreads();
  }
  if (t_local < tpc) {
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int e = g * 4 + i;
      const float z = static_cast<float>(acc[i]);
      slog[t_local * N4 + e] = z;
      if (active && e < N) {
        rb.logits[(size_t)tok * N + e] = z;
        if (!isfinite(z)) atomicExch(rb.finite_flag, 1);
      }
    }
  }
  __syncthreads();

  // ---- per-token softmax / top-K (one thread per token of the tile) ----
  double lse2 = 0.0;
  if (threadIdx.x < tpc && tok0 + threadIdx.x < T) {
    const int j = tok0 + threadIdx.x;
    const float* z = slog + threadIdx.x * N4;
    double mx = z[0];
    for (int e = 1; e < N; ++e) mx = fmax(mx, static_cast<double>(z[e]));
    double denom = 0.0;
    for (int e = 0; e < N; ++e) denom += exp(static_cast<double>(z[e]) - mx);
    float* p = rb.probs + (size_t)j * N;
    for (int e = 0; e < N; ++e) {
      const float pe = static_cast<float>(exp(static_cast<double>(z[e]) - mx) / denom);
      p[e] = pe;
      slog[threadIdx.x * N4 + e] = pe;  // reuse the row for probs
    }
    const double lse = mx + log(denom);
    lse2 = lse * lse;
    // top-K by repeated selection: strict '>' keeps the lowest index among equal values.
    uint64_t taken_lo = 0, taken_hi = 0;  // up to 128 experts tracked in bits; larger N loops
    float vals[8];
    int ids[8];
    const float* prow = slog + threadIdx.x * N4;
    for (int k = 0; k < K; ++k) {
      int best = -1;
      float bv = 0.0f;
      for (int e = 0; e < N; ++e) {
        const bool tk = e < 64 ? ((taken_lo >> e) & 1ull) : ((taken_hi >> (e - 64)) & 1ull);
        if (tk) continue;
        const float v = prow[e];
        if (best < 0 || v > bv) { best = e; bv = v; }
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
    }
  }
  __syncthreads();

  // ---- per-tile statistics: expert counts, local ranks, prob sums (one thread per expert) ----
  const int ntok = min(tpc, T - tok0);
  for (int e = threadIdx.x; e < N; e += kRouterThreads) {
    int cnt = 0;
    double ps = 0.0;
    for (int t = 0; t < ntok; ++t) {
      ps += static_cast<double>(slog[t * N4 + e]);
      for (int k = 0; k < K; ++k) {
        const size_t s = (size_t)(tok0 + t) * K + k;
        if (rb.topk_idx[s] == e) rb.local_rank[s] = cnt++;
      }
    }
    rb.tile_cnt[(size_t)tile * N + e] = cnt;
    rb.tile_psum[(size_t)tile * N + e] = ps;
  }
  // tile sum of lse^2 in token order (warp 0 holds the tile's tokens when tpc <= 32; general
  // case goes through shared memory)
  __shared__ double s_lse[kRouterThreads];
  s_lse[threadIdx.x] = lse2;
  __syncthreads();
  if (threadIdx.x == 0) {
    double a = 0.0;
    for (int t = 0; t < ntok; ++t) a += s_lse[t];
    rb.tile_lse2[tile] = a;
  }
}

// ---------------------------------------------------------------------------------------
// K2: dispatch plan. Exclusive scan of the per-tile expert counts (tile-major within each
// expert) -> each tile's base row inside its expert segment; expert offsets; agg_prob, aux-loss
// and Z-loss reductions in a fixed order. One CTA; deterministic (no atomics).
__global__ void __launch_bounds__(kPlanThreads) plan_kernel(int n_tiles, int T, int N, int K, RouteBufs rb) {
  __shared__ int s_chunk[kPlanThreads];
  __shared__ double s_pchunk[kPlanThreads];
  __shared__ int s_counts[256];
  const int chunks = kPlanThreads / N;  // chunks of tiles per expert
  const int per = (n_tiles + chunks - 1) / chunks;
  const int e = threadIdx.x % N;
  const int c = threadIdx.x / N;
  const bool act = c < chunks;
  int sum = 0;
  double ps = 0.0;
  if (act) {
    for (int t = c * per; t < min(n_tiles, (c + 1) * per); ++t) {
      sum += rb.tile_cnt[(size_t)t * N + e];
      ps += rb.tile_psum[(size_t)t * N + e];
    }
  }
  s_chunk[threadIdx.x] = sum;
  s_pchunk[threadIdx.x] = ps;
  __syncthreads();
  if (threadIdx.x < N) {
    int run = 0;
    double p = 0.0;
    for (int cc = 0; cc < chunks; ++cc) {
      const int v = s_chunk[cc * N + threadIdx.x];
      s_chunk[cc * N + threadIdx.x] = run;
      run += v;
      p += s_pchunk[cc * N + threadIdx.x];
    }
    s_counts[threadIdx.x] = run;
    s_pchunk[threadIdx.x] = p;  // chunk 0 slot of this expert now holds the expert's prob sum
    rb.counts[threadIdx.x] = run;
    rb.agg_prob[threadIdx.x] = static_cast<float>(p);
  }
  __syncthreads();
  if (act) {
    int run = s_chunk[threadIdx.x];
    for (int t = c * per; t < min(n_tiles, (c + 1) * per); ++t) {
      const size_t i = (size_t)t * N + e;
      const int v = rb.tile_cnt[i];
      rb.tile_cnt[i] = run;
      run += v;
    }
  }
  if (threadIdx.x == 0) {
    int off = 0;
    double aux = 0.0;
    for (int x = 0; x < N; ++x) {
      rb.offsets[x] = off;
      off += s_counts[x];
      aux += s_pchunk[x] * static_cast<double>(s_counts[x]);
    }
    rb.offsets[N] = off;
    double z = 0.0;
    for (int t = 0; t < n_tiles; ++t) z += rb.tile_lse2[t];
    const double coef = static_cast<double>(N) / (static_cast<double>(T) * T * static_cast<double>(K));
    rb.losses[0] = static_cast<float>(coef * aux);
    rb.losses[1] = static_cast<float>(z / static_cast<double>(T));
  }
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
                                                       float* __restrict__ row_w, const float* __restrict__ act_scale) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= T) return;
  const int tile = j / tpc;
  int rows[8];
  float inv_s[8];
  for (int k = 0; k < K; ++k) {
    const size_t s = (size_t)j * K + k;
    const int e = idx[s];
    const int r = rb.offsets[e] + rb.tile_cnt[(size_t)tile * N + e] + rb.local_rank[s];
    rows[k] = r;
    if constexpr (kFp8) inv_s[k] = 1.0f / act_scale[e];
    if (lane == 0) {
      inv[s] = r;
      perm[r] = static_cast<int32_t>(s);
      row_w[r] = wts[s];
    }
  }
  const int4* src = reinterpret_cast<const int4*>(x + (size_t)j * d);
  const int nvec = d / 8;  // 8 bf16 per 16 B
  if constexpr (!kFp8) {
    for (int v0 = lane; v0 < nvec; v0 += 32 * 4) {
      int4 buf[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        if (v0 + u * 32 < nvec) buf[u] = ld_nc_v4(src + v0 + u * 32);
      for (int k = 0; k < K; ++k) {
        int4* dst = reinterpret_cast<int4*>(reinterpret_cast<__nv_bfloat16*>(xperm) + (size_t)rows[k] * d);
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (v0 + u * 32 < nvec) st_na_v4(dst + v0 + u * 32, buf[u]);
      }
    }
  } else {
    for (int v = lane; v < nvec; v += 32) {
      const int4 raw = ld_nc_v4(src + v);
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
      float f[8];
#pragma unroll
      for (int i = 0; i < 8; ++i) f[i] = __bfloat162float(h[i]);
      for (int k = 0; k < K; ++k) {
        uint32_t p[2];
#pragma unroll
        for (int i = 0; i < 2; ++i) {
          const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
              make_float2(f[4 * i] * inv_s[k], f[4 * i + 1] * inv_s[k]), __NV_SATFINITE, __NV_E4M3);
          const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
              make_float2(f[4 * i + 2] * inv_s[k], f[4 * i + 3] * inv_s[k]), __NV_SATFINITE, __NV_E4M3);
          p[i] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
        }
        uint2* dst = reinterpret_cast<uint2*>(reinterpret_cast<uint8_t*>(xperm) + (size_t)rows[k] * d) + v;
        *dst = make_uint2(p[0], p[1]);
      }
    }
  }
}

// ---------------------------------------------------------------------------------------
// K6: weighted combine / un-permute. One warp per token: out[j] = sum_k Y[inv[j,k]] in fp32, slot
// order (rows of Y already carry the combine weight from the GEMM2 epilogue). Replaces
// scatter_add_rows + add (proj/src/tensor.cpp:814-845, :248-262) with no intermediate copies.
template <typename OutT>
__global__ void __launch_bounds__(256) combine_kernel(const __nv_bfloat16* __restrict__ y, const int32_t* __restrict__ inv,
                                                      int T, int d, int K, OutT* __restrict__ out,
                                                      int32_t* __restrict__ finite_flag) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= T) return;
  int rows[8];
  for (int k = 0; k < K; ++k) rows[k] = inv[(size_t)j * K + k];
  const int nvec = d / 8;
  for (int v = lane; v < nvec; v += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    int4 raw[8];
    for (int k = 0; k < K; ++k) raw[k] = ld_nc_v4(reinterpret_cast<const int4*>(y + (size_t)rows[k] * d) + v);
    for (int k = 0; k < K; ++k) {
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw[k]);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(h[i]);
    }
    bool fin = true;
#pragma unroll
    for (int i = 0; i < 8; ++i) fin &= isfinite(acc[i]);
    if (!fin) atomicExch(finite_flag, 1);
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

}  // namespace cmoe
