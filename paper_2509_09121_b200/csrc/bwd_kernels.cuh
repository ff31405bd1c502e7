// Expert-FFN backward helpers (the Tape closures of the reference composition):
//  * combine backward  = scatter_add_rows bwd (tensor.cpp:834-842) + mul_rowwise bwd (:587-607):
//      dY[r] = w[s] * dOut[j],  d_w[s] = <dOut[j], Y[r]>   (s = perm[r], j = s / K)
//  * padded transposes feeding the variable-K weight-gradient GEMMs (dW = Lhs^T Rhs over the
//    rows of one expert; each expert's rows start at a 64-aligned column so a k-block never
//    straddles two experts; padding columns are zero);
//  * reference-layout bf16 weight copies (W_in [d][2f], W_out [f][d]) derived on device from the
//    packed forward layouts — the K-major B operands of the two dgrad GEMMs.
#pragma once
#include "ptx.cuh"

namespace cmoe {

// One warp per permuted row.
__global__ void __launch_bounds__(256) combine_bwd_kernel(const __nv_bfloat16* __restrict__ d_out,
                                                          const __nv_bfloat16* __restrict__ y,
                                                          const int32_t* __restrict__ perm,
                                                          const float* __restrict__ cw, int rows, int d, int K,
                                                          __nv_bfloat16* __restrict__ dy, float* __restrict__ d_cw,
                                                          void* const* __restrict__ expert_dst = nullptr,
                                                          const int32_t* __restrict__ idx = nullptr,
                                                          const int32_t* __restrict__ offsets = nullptr,
                                                          const int32_t* __restrict__ dst_poff = nullptr) {
  // expert_dst (EP peer transport): the dY row of expert g goes straight into the owner's dYbuf at
  // expert_dst[g] + (r - offsets[g]) rows instead of dy[r]. dst_poff (single GPU): dy is the padded
  // row layout, expert g's rows from dst_poff[g] (dgrad-1 and dW_out read it there).
  const int r = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const int s = perm[r];
  const int j = s / K;
  const float w = cw[s];
  const int4* g = reinterpret_cast<const int4*>(d_out + (size_t)j * d);
  const int4* yr = reinterpret_cast<const int4*>(y + (size_t)r * d);
  int4* o = reinterpret_cast<int4*>(dy + (size_t)r * d);
  if (dst_poff) {
    const int e = idx[s];
    o = reinterpret_cast<int4*>(dy + (size_t)(dst_poff[e] + (r - offsets[e])) * d);
  } else if (expert_dst) {
    const int e = idx[s];
    char* b = static_cast<char*>(expert_dst[e]);
    o = b ? reinterpret_cast<int4*>(b + (size_t)(r - offsets[e]) * d * 2) : nullptr;
  }
  float acc = 0.0f;
  for (int v = lane; v < d / 8; v += 32) {
    const int4 gv = ld_nc_v4(g + v);
    const int4 yv = ld_nc_v4(yr + v);
    const __nv_bfloat16* gh = reinterpret_cast<const __nv_bfloat16*>(&gv);
    const __nv_bfloat16* yh = reinterpret_cast<const __nv_bfloat16*>(&yv);
    float f[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const float gg = __bfloat162float(gh[i]);
      acc = fmaf(gg, __bfloat162float(yh[i]), acc);
      f[i] = w * gg;
    }
    int4 ov;
    ov.x = pack_bf16(f[0], f[1]);
    ov.y = pack_bf16(f[2], f[3]);
    ov.z = pack_bf16(f[4], f[5]);
    ov.w = pack_bf16(f[6], f[7]);
    if (o) st_na_v4(o + v, ov);
  }
  for (int off = 16; off; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
  if (lane == 0) d_cw[s] = acc;
  if (expert_dst) __threadfence_system();  // peer stores visible before the exchange barrier
}

// poff[e] = 64-aligned first padded row of expert e; kb_off[e] = poff[e] / 64 (k-blocks of the
// bf16 K-major transposes). One thread.
__global__ void pad_plan_kernel(const int32_t* __restrict__ offsets, int n, int32_t* __restrict__ poff,
                                int32_t* __restrict__ kb_off) {
  if (threadIdx.x || blockIdx.x) return;
  int p = 0;
  for (int e = 0; e < n; ++e) {
    poff[e] = p;
    kb_off[e] = p / 64;
    p += (offsets[e + 1] - offsets[e] + 63) / 64 * 64;
  }
  poff[n] = p;
  kb_off[n] = p / 64;
}

// dst[p][:] = src[offsets[e] + p - poff[e]][:] inside expert e's padded row range, zeros in its
// padding rows: the row-major padded layout the weight-gradient GEMMs read MN-major. One warp per
// padded row, 16-byte accesses.
__global__ void __launch_bounds__(256) pad_rows_kernel(const __nv_bfloat16* __restrict__ src, int C,
                                                       const int32_t* __restrict__ offsets,
                                                       const int32_t* __restrict__ poff, int n,
                                                       __nv_bfloat16* __restrict__ dst) {
  const int p = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (p >= poff[n]) return;
  int e = 0;
  while (p >= poff[e + 1]) ++e;
  const int r = p - poff[e];
  const bool live = r < offsets[e + 1] - offsets[e];
  const int4* s4 = reinterpret_cast<const int4*>(src + (size_t)(offsets[e] + (live ? r : 0)) * C);
  int4* d4 = reinterpret_cast<int4*>(dst + (size_t)p * C);
  for (int v = lane; v < C / 8; v += 32) d4[v] = live ? ld_nc_v4(s4 + v) : make_int4(0, 0, 0, 0);
}

// Zero the padding rows [poff[e] + cnt_e, poff[e+1]) of a padded row-major buffer [rp][C] whose
// live rows are written by a GEMM epilogue. Grid (64 / 8, n_experts), 256 threads.
__global__ void __launch_bounds__(256) zero_pad_rows_kernel(__nv_bfloat16* __restrict__ buf, int C,
                                                            const int32_t* __restrict__ offsets,
                                                            const int32_t* __restrict__ poff) {
  const int e = blockIdx.y;
  const int start = poff[e] + (offsets[e + 1] - offsets[e]);
  const int p = start + blockIdx.x * 8 + (threadIdx.x >> 5);
  if (p >= poff[e + 1]) return;
  int4* d4 = reinterpret_cast<int4*>(buf + (size_t)p * C);
  for (int v = threadIdx.x & 31; v < C / 8; v += 32) d4[v] = make_int4(0, 0, 0, 0);
}

// dst[i][j] = src[rowmap(j)][i]: src [rows_src][cols_src] bf16 -> dst [cols_src][rows_src].
// kWinMap: rowmap(c) = packed W_in row of reference column c (inverse of win_col_of_packed_row).
template <bool kWinMap>
__global__ void __launch_bounds__(256) transpose_weight_kernel(const __nv_bfloat16* __restrict__ src, int rows_src,
                                                               int cols_src, int f, __nv_bfloat16* __restrict__ dst) {
  __shared__ __nv_bfloat16 tile[32][34];
  const int j0 = blockIdx.x * 32;  // dst column block = source (mapped) row block
  const int i0 = blockIdx.y * 32;  // dst row block = source column block
  for (int t = threadIdx.x; t < 32 * 32; t += 256) {
    const int jj = t / 32, ii = t % 32;
    const int j = j0 + jj;
    __nv_bfloat16 v = __float2bfloat16_rn(0.0f);
    if (j < rows_src && i0 + ii < cols_src) {
      int r = j;
      if constexpr (kWinMap) {
        const int up = j >= f;
        const int c = up ? j - f : j;
        r = (c / 128) * 256 + (up ? 128 : 0) + c % 128;
      }
      v = src[(size_t)r * cols_src + i0 + ii];
    }
    tile[jj][ii] = v;
  }
  __syncthreads();
  for (int t = threadIdx.x; t < 32 * 32; t += 256) {
    const int ii = t / 32, jj = t % 32;
    if (i0 + ii < cols_src && j0 + jj < rows_src) dst[(size_t)(i0 + ii) * rows_src + j0 + jj] = tile[jj][ii];
  }
}

// ---------------------------------------------------------------------------------------
// Router backward. One thread per token:
//   dv_k = (d_cw_k - sum_k' d_cw_k' w_k') / s,  s = sum_k p[idx_k]      (renormalised top-K)
//   dp_i = sum_{k: idx_k=i} dv_k + g_aux * N/(B^2 K) * c_i             (moe_aux_loss bwd)
//   dz_i = p_i (dp_i - <dp, p>) + g_z * 2 lse / B * p_i                (softmax / z_loss bwd)
__global__ void router_bwd_dz_kernel(const float* __restrict__ probs, const float* __restrict__ logits,
                                     const int32_t* __restrict__ idx, const float* __restrict__ d_cw,
                                     const int32_t* __restrict__ counts, int T, int N, int K, float g_aux, float g_z,
                                     float* __restrict__ dz) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= T) return;
  const float* p = probs + (size_t)j * N;
  const float* zr = logits + (size_t)j * N;
  double s = 0.0;
  for (int k = 0; k < K; ++k) s += p[idx[(size_t)j * K + k]];
  double dot_w = 0.0;
  for (int k = 0; k < K; ++k) dot_w += static_cast<double>(d_cw[(size_t)j * K + k]) * (p[idx[(size_t)j * K + k]] / s);
  const double coef = static_cast<double>(N) / (static_cast<double>(T) * T * static_cast<double>(K));
  double mx = zr[0];
  for (int i = 1; i < N; ++i) mx = fmax(mx, static_cast<double>(zr[i]));
  double den = 0.0;
  for (int i = 0; i < N; ++i) den += exp_glibc(static_cast<double>(zr[i]) - mx);
  const double lse = mx + log(den);
  // dp is sparse except for the dense aux term: dot = sum_i dp_i p_i computed on the fly
  double dot = 0.0;
  for (int i = 0; i < N; ++i) dot += g_aux * coef * static_cast<double>(counts[i]) * p[i];
  for (int k = 0; k < K; ++k) {
    const int i = idx[(size_t)j * K + k];
    dot += (static_cast<double>(d_cw[(size_t)j * K + k]) - dot_w) / s * p[i];
  }
  for (int i = 0; i < N; ++i) {
    double dpi = g_aux * coef * static_cast<double>(counts[i]);
    for (int k = 0; k < K; ++k)
      if (idx[(size_t)j * K + k] == i) dpi += (static_cast<double>(d_cw[(size_t)j * K + k]) - dot_w) / s;
    dz[(size_t)j * N + i] =
        static_cast<float>(p[i] * (dpi - dot) + g_z * 2.0 * lse / static_cast<double>(T) * p[i]);
  }
}

// dW_r partials: grid (d/64, T-chunks, ceil(N4/16)); thread = (l, 4 experts); fp32 partial sums over
// the chunk's tokens, reduced in a fixed order by router_wgrad_reduce_kernel (deterministic).
constexpr int kRwTokens = 512;
__global__ void __launch_bounds__(256) router_wgrad_partial_kernel(const __nv_bfloat16* __restrict__ x,
                                                                   const float* __restrict__ dz, int T, int d, int N,
                                                                   float* __restrict__ part) {
  const int l = blockIdx.x * 64 + threadIdx.x / 4;
  const int e0 = blockIdx.z * 16 + (threadIdx.x % 4) * 4;
  const int t0 = blockIdx.y * kRwTokens;
  const int t1 = min(T, t0 + kRwTokens);
  float acc[4] = {0.f, 0.f, 0.f, 0.f};
  if (l < d) {
    for (int j = t0; j < t1; ++j) {
      const float xv = __bfloat162float(x[(size_t)j * d + l]);
#pragma unroll
      for (int b = 0; b < 4; ++b)
        if (e0 + b < N) acc[b] = fmaf(xv, dz[(size_t)j * N + e0 + b], acc[b]);
    }
#pragma unroll
    for (int b = 0; b < 4; ++b)
      if (e0 + b < N) part[((size_t)blockIdx.y * d + l) * N + e0 + b] = acc[b];
  }
}
__global__ void router_wgrad_reduce_kernel(const float* __restrict__ part, int chunks, int dn, float* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= dn) return;
  float a = 0.0f;
  for (int c = 0; c < chunks; ++c) a += part[(size_t)c * dn + i];
  out[i] = a;
}

// Dispatch backward with the router term fused: d_hidden[j] = sum_k dX[inv[j,k]] +
// sum_e dz[j][e] W_r[:, e]  (fp32 accumulation, one rounding to bf16). One warp per token.
template <int kK>
__global__ void __launch_bounds__(256) dispatch_bwd_router_kernel(const __nv_bfloat16* __restrict__ dx,
                                                                  const int32_t* __restrict__ inv, int T, int d,
                                                                  const float* __restrict__ dz,
                                                                  const float* __restrict__ wr, int N,
                                                                  __nv_bfloat16* __restrict__ out) {
  const int j = blockIdx.x * 8 + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= T) return;
  const int4* src[kK];
#pragma unroll
  for (int k = 0; k < kK; ++k) src[k] = reinterpret_cast<const int4*>(dx + (size_t)inv[(size_t)j * kK + k] * d);
  const float* dzj = dz + (size_t)j * N;
  for (int v = lane; v < d / 8; v += 32) {
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
    for (int k = 0; k < kK; ++k) {
      const int4 raw = ld_nc_v4(src[k] + v);
      const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] += __bfloat162float(h[i]);
    }
    for (int e = 0; e < N; ++e) {
      const float g = dzj[e];
#pragma unroll
      for (int i = 0; i < 8; ++i) acc[i] = fmaf(g, wr[(size_t)(8 * v + i) * N + e], acc[i]);
    }
    int4 o;
    o.x = pack_bf16(acc[0], acc[1]);
    o.y = pack_bf16(acc[2], acc[3]);
    o.z = pack_bf16(acc[4], acc[5]);
    o.w = pack_bf16(acc[6], acc[7]);
    st_na_v4(reinterpret_cast<int4*>(out + (size_t)j * d) + v, o);
  }
}

}  // namespace cmoe
