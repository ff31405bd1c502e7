// Weight preparation kernels: device-side synthetic generation with the reference counter PRNG
// (proj/include/compasslab/prng.hpp:15-70) and repacking of reference-layout fp32 weights into
// the K-major bf16 / e4m3 operand layouts of the grouped GEMMs.
//
// Packed layouts (per expert e):
//   W_in  [2f][d]  row p: block b = p/256, i = p%256; i < 128 -> gate column b*128+i,
//                  else up column f + b*128 + (i-128). A 256-row n-block therefore holds the gate
//                  and up columns of the same 128 FFN channels, so the SwiGLU runs in the GEMM1
//                  epilogue straight from TMEM (no slice_cols copies, tensor.cpp:398-420).
//   W_out [d][f]   transpose of the reference [f][d].
#pragma once
#include <cuda_fp8.h>

#include "ptx.cuh"

namespace cmoe {

__host__ __device__ inline uint64_t mix64(uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
constexpr uint64_t kGolden = 0x9e3779b97f4a7c15ull;
__host__ __device__ inline uint64_t split_seed(uint64_t root, uint64_t stream) {
  return mix64(root ^ mix64(stream * kGolden + 0x632be59bd9b4e019ull));
}
// Value i of Prng(seed).next_normal_f(0, stddev): Box-Muller over draws 2i+1, 2i+2.
__device__ __forceinline__ float prng_normal_f(uint64_t seed, uint64_t i, float stddev) {
  const uint64_t c = 2 * i;
  const double u1 = 1.0 - static_cast<double>(mix64(seed + (c + 1) * kGolden) >> 11) * 0x1.0p-53;
  const double u2 = static_cast<double>(mix64(seed + (c + 2) * kGolden) >> 11) * 0x1.0p-53;
  const double z = sqrt(-2.0 * log(u1)) * cos(2.0 * 3.14159265358979323846 * u2);
  return 0.0f + stddev * static_cast<float>(z);
}

__device__ __forceinline__ int win_col_of_packed_row(int p, int f) {
  const int b = p >> 8, i = p & 255;
  return i < 128 ? b * 128 + i : f + b * 128 + (i - 128);
}

__global__ void synth_bf16_kernel(uint64_t seed, int64_t n, float stddev, __nv_bfloat16* out, float shift = 0.0f) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(prng_normal_f(seed, i, stddev) + shift);
}
__global__ void synth_f32_kernel(uint64_t seed, int64_t n, float stddev, float* out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = prng_normal_f(seed, i, stddev);
}
// Packed W_in[e] element (p, l) is reference element (l, c(p)) = draw l*2f + c of stream seed.
__global__ void synth_pack_win_kernel(uint64_t seed, int d, int f, float stddev, __nv_bfloat16* out) {
  const int64_t n = (int64_t)2 * f * d;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int p = static_cast<int>(i / d), l = static_cast<int>(i % d);
    const int c = win_col_of_packed_row(p, f);
    out[i] = __float2bfloat16_rn(prng_normal_f(seed, (uint64_t)l * 2 * f + c, stddev));
  }
}
// Packed W_out[e] element (n, l) is reference element (l, n) = draw l*d + n.
__global__ void synth_pack_wout_kernel(uint64_t seed, int d, int f, float stddev, __nv_bfloat16* out) {
  const int64_t total = (int64_t)d * f;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += (int64_t)gridDim.x * blockDim.x) {
    const int nrow = static_cast<int>(i / f), l = static_cast<int>(i % f);
    out[i] = __float2bfloat16_rn(prng_normal_f(seed, (uint64_t)l * d + nrow, stddev));
  }
}

// Transpose-and-convert of one expert's reference-layout fp32 matrix src[rows][cols] into
// dst[cols'][rows] bf16, where dst row q takes source column map(q). 32x32 smem tiles.
template <bool kWin>
__global__ void pack_transpose_kernel(const float* __restrict__ src, int rows, int cols, int f,
                                      __nv_bfloat16* __restrict__ dst) {
  __shared__ float tile[32][33];
  const int q0 = blockIdx.x * 32;  // dst row block (source column space)
  const int r0 = blockIdx.y * 32;  // source row block (= dst column)
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int r = r0 + i;
    const int q = q0 + threadIdx.x;
    float v = 0.0f;
    if (r < rows && q < cols) {
      const int c = kWin ? win_col_of_packed_row(q, f) : q;
      v = src[(size_t)r * cols + c];
    }
    tile[i][threadIdx.x] = v;
  }
  __syncthreads();
  for (int i = threadIdx.y; i < 32; i += blockDim.y) {
    const int q = q0 + i;
    const int r = r0 + threadIdx.x;
    if (q < cols && r < rows) dst[(size_t)q * rows + r] = __float2bfloat16_rn(tile[threadIdx.x][i]);
  }
}

// Per-output-channel FP8 weight quantisation: scale = absmax/448 over the
// packed row (a K-major row is one output channel), q = e4m3_satfinite(w / scale). One warp/row.
// given = true: the scales are inputs (a loaded scheme file), not recomputed.
__global__ void quantize_rows_e4m3_kernel(const __nv_bfloat16* __restrict__ w, int64_t rows, int kdim,
                                          uint8_t* __restrict__ q, float* __restrict__ scale, bool given = false) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= rows) return;
  const __nv_bfloat16* src = w + r * kdim;
  float s;
  if (given) {
    s = scale[r];
  } else {
    float m = 0.0f;
    for (int i = lane; i < kdim; i += 32) m = fmaxf(m, fabsf(__bfloat162float(src[i])));
    for (int o = 16; o; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
    s = m > 0.0f ? __fdiv_rn(m, 448.0f) : 1.0f;
    if (lane == 0) scale[r] = s;
  }
  uint8_t* dst = q + r * kdim;
  for (int i = lane; i < kdim; i += 32)
    dst[i] = static_cast<uint8_t>(__nv_cvt_float_to_fp8(__fdiv_rn(__bfloat162float(src[i]), s), __NV_SATFINITE, __NV_E4M3));
}

// Calibration (collect_calibration): per-expert max |value| over the rows of
// each expert segment. Non-negative floats order like their bit patterns -> atomicMax on ints.
__global__ void segment_absmax_kernel(const __nv_bfloat16* __restrict__ m, int cols, const int32_t* __restrict__ offsets,
                                      int n_experts, float* __restrict__ out) {
  const int64_t r = blockIdx.x * (int64_t)(blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (r >= offsets[n_experts]) return;
  int e = 0;
  while (r >= offsets[e + 1]) ++e;
  float mx = 0.0f;
  const __nv_bfloat16* src = m + r * cols;
  for (int i = lane; i < cols; i += 32) mx = fmaxf(mx, fabsf(__bfloat162float(src[i])));
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0) atomicMax(reinterpret_cast<int*>(out) + e, __float_as_int(mx));
}

// Calibration routing counts: acc[e] += counts[e] (collect_calibration).
__global__ void add_counts_kernel(const int32_t* __restrict__ counts, int n, long long* __restrict__ acc) {
  for (int e = threadIdx.x; e < n; e += blockDim.x) acc[e] += counts[e];
}

// Source-side calibration under expert parallelism: out[g] = max |x_j| over the tokens j routed to
// global expert g (one warp per token; atomicMax on non-negative float bit patterns).
__global__ void route_absmax_kernel(const __nv_bfloat16* __restrict__ x, int T, int d, int K,
                                    const int32_t* __restrict__ idx, float* __restrict__ out) {
  const int j = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (j >= T) return;
  float mx = 0.0f;
  const __nv_bfloat16* src = x + (size_t)j * d;
  for (int i = lane; i < d; i += 32) mx = fmaxf(mx, fabsf(__bfloat162float(src[i])));
  for (int o = 16; o; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane < K) atomicMax(reinterpret_cast<int*>(out) + idx[(size_t)j * K + lane], __float_as_int(mx));
}

// Per-column max |value| of a row-major bf16 matrix [rows][cols] into out[cols] (atomicMax on the
// bit patterns of non-negative floats). Grid (cols/256, row chunks).
__global__ void col_absmax_kernel(const __nv_bfloat16* __restrict__ m, int64_t rows, int cols, int rows_per_block,
                                  float* __restrict__ out) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  const int64_t r0 = (int64_t)blockIdx.y * rows_per_block;
  const int64_t r1 = min(rows, r0 + rows_per_block);
  float mx = 0.0f;
  for (int64_t r = r0; r < r1; ++r) mx = fmaxf(mx, fabsf(__bfloat162float(m[r * cols + c])));
  atomicMax(reinterpret_cast<int*>(out) + c, __float_as_int(mx));
}

// fold_smoothing on the packed W_in [rows][d] (K = input channel): w[.][l] *= s[l]
// (re-rounded to bf16), and W_r [d][N] fp32 rows: wr[l][.] *= s[l].
__global__ void scale_cols_bf16_kernel(__nv_bfloat16* __restrict__ m, int64_t n, int cols, const float* __restrict__ s) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    m[i] = __float2bfloat16_rn(__bfloat162float(m[i]) * s[i % cols]);
}
__global__ void scale_rows_f32_kernel(float* __restrict__ m, int rows, int cols, const float* __restrict__ s) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < rows * cols) m[i] = m[i] * s[i / cols];
}

// E4M3 quantize-dequantize of one value (SPEC.md:523-531 fp8_qdq): q = RNE_satfinite(x / s) on the
// E4M3 grid, x_hat = q * s in fp32 (the same float operations as the oracle's orc_fp8_qdq).
__device__ __forceinline__ float qdq_e4m3(float x, float s) {
  const __nv_fp8_storage_t q = __nv_cvt_float_to_fp8(__fdiv_rn(x, s), __NV_SATFINITE, __NV_E4M3);
  const __half_raw hr = __nv_cvt_fp8_to_halfraw(q, __NV_E4M3);
  return __fmul_rn(__half2float(__half(hr)), s);
}

// Router under the FP8 scheme ("all expert/router ... projection GEMMs run through
// fp8_qdq on weights (per-output-channel scale = channel absmax/448)"): the router's output
// channels are the N expert columns of W_r [d][N]. ws[c] = absmax/448 (1 for an all-zero column,
// as the expert weights), wq = qdq(W_r, ws[c]) in fp32 — the values the router's fp64 chains
// consume. One thread per column, once per quantize.
__global__ void router_qdq_w_kernel(const float* __restrict__ wr, int d, int N, float* __restrict__ wq,
                                    float* __restrict__ ws, bool given = false) {
  const int c = blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= N) return;
  float s;
  if (given) {
    s = ws[c];
  } else {
    float m = 0.0f;
    for (int l = 0; l < d; ++l) m = fmaxf(m, fabsf(wr[(size_t)l * N + c]));
    s = m > 0.0f ? __fdiv_rn(m, 448.0f) : 1.0f;
    ws[c] = s;
  }
  for (int l = 0; l < d; ++l) wq[(size_t)l * N + c] = qdq_e4m3(wr[(size_t)l * N + c], s);
}

// The router's activation operand under the FP8 scheme: the E4M3 codes of x / s_x (per-tensor
// calibration scale s_x, a device scalar); the router widens code * s_x, which is exactly
// qdq_e4m3(x, s_x). 16 values per thread per step (one 16-byte store).
template <typename XT>
__global__ void router_qdq8_kernel(const XT* __restrict__ x, int64_t n, const float* __restrict__ sx,
                                   uint8_t* __restrict__ out) {
  const float s = *sx;
  const int64_t n16 = n / 16;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n16; i += (int64_t)gridDim.x * blockDim.x) {
    float v[16];
    if constexpr (sizeof(XT) == 2) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int4 raw = reinterpret_cast<const int4*>(x + i * 16)[h];
        const __nv_bfloat16* b = reinterpret_cast<const __nv_bfloat16*>(&raw);
#pragma unroll
        for (int j = 0; j < 8; ++j) v[8 * h + j] = __bfloat162float(b[j]);
      }
    } else {
#pragma unroll
      for (int h = 0; h < 4; ++h) {
        const float4 f = reinterpret_cast<const float4*>(x + i * 16)[h];
        v[4 * h] = f.x;
        v[4 * h + 1] = f.y;
        v[4 * h + 2] = f.z;
        v[4 * h + 3] = f.w;
      }
    }
    uint32_t p[4];
#pragma unroll
    for (int w = 0; w < 4; ++w) {
      const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
          make_float2(__fdiv_rn(v[4 * w], s), __fdiv_rn(v[4 * w + 1], s)), __NV_SATFINITE, __NV_E4M3);
      const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
          make_float2(__fdiv_rn(v[4 * w + 2], s), __fdiv_rn(v[4 * w + 3], s)), __NV_SATFINITE, __NV_E4M3);
      p[w] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
    }
    reinterpret_cast<int4*>(out)[i] = make_int4((int)p[0], (int)p[1], (int)p[2], (int)p[3]);
  }
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ in, int64_t n, __nv_bfloat16* __restrict__ out) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    out[i] = __float2bfloat16_rn(in[i]);
}

__global__ void i32_to_i64_kernel(const int32_t* __restrict__ in, int n, int64_t* __restrict__ out) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}

}  // namespace cmoe
