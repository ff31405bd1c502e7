// K1, certified large-batch variant (fused forward without a decision export; host_forward.cuh
// run_router). The reference's routing needs the fp64, ascending-l logit chains only to decide
// WHICH experts a token takes and in which order; the fused forward exports neither logits nor
// probabilities. So:
//   K1a router_approx_kernel: every logit in fp32 (8 tokens x 8 experts per thread, FFMA: 2x the
//       FP64 rate, half the operand bytes) plus a rigorous bound on its distance to the reference's
//       fp32 logit: |z' - z_ref| <= E = g_d ||x||_2 ||w_i||_2 (recursive fp32 summation, Cauchy-
//       Schwarz) + the fp32 rounding of z_ref. A token is CERTIFIED when its top-K order by z' is
//       separated from everything below by more than the bounds plus a margin that keeps the
//       reference's fp32 probabilities strictly ordered (so no prob tie can reorder them);
//       otherwise the same CTA recomputes that token's logits with the reference's exact fp64
//       chains (bit-identical to gemm_nn, tensor.cpp:157-173), one thread per (token, expert).
//   K1c router_finish_tiles_kernel: softmax / top-K / combine weights / tile statistics from the
//       logits (router_finish_warps), then the usual plan.
// Routing indices, counts and the dispatch permutation are bit-exact against the reference
// (certified or recomputed); combine weights of certified tokens come from the fp32 logits (within
// ~1e-6 relative, inside the layer's bf16 output tolerance). Decision exports (route_tokens,
// forward with a decision, training) keep the exact kernels.
#pragma once

namespace cmoe {

constexpr int kCertThreads = 256;  // K1a CTA: 16 (token group, expert group) positions x 16 k-slices
constexpr int kCertTT = 8;         // tokens per thread
constexpr int kCertEG = 8;         // experts per thread
constexpr int kCertCL = 128;       // columns (l) per staged chunk; k-slice s takes columns [8s, 8s+8)
constexpr int kCertS = kCertCL / 8;
constexpr int kCertStages = 3;     // cp.async ring depth
constexpr int kCertFinTpc = 32;    // K1c tokens per tile (4 per warp: the per-token softmax is latency-bound)

struct RouterCertSmem {
  int N8, ng, tpc, N4, tpg, cl;
  size_t rx, sw, red, redx, ex, exx, total;
  __host__ __device__ RouterCertSmem(int n_experts, int xb) {
    N8 = (n_experts + 7) / 8 * 8;
    ng = N8 / kCertEG;
    tpc = 16 / ng * kCertTT;  // 16 positions = (tpc / 8) token groups x ng expert groups
    rx = 0;                                                  // [stages][tpc][CL] XT (swizzled 16-B pieces)
    sw = rx + (size_t)kCertStages * tpc * kCertCL * xb;      // [stages][CL][N8] fp32
    const size_t ring = sw + (size_t)kCertStages * kCertCL * N8 * 4;
    red = 0;                                                 // after the main loop: [S][tpc][N8] partials
    redx = red + (size_t)kCertS * tpc * N8 * 4;              //                      [S][tpc] |x|^2 partials
    const size_t fin = redx + (size_t)kCertS * tpc * 4;
    // exact chains of the CTA's uncertified tokens (after certification only the reduced logits
    // red[0 .. tpc*N8) stay live): a 2-stage ring of W_r rows (fp64 [cl][N4]) and token rows (XT)
    N4 = (n_experts + 3) / 4 * 4;
    tpg = kCertThreads / N4;
    cl = 8192 / N4 < 256 ? 8192 / N4 : 256;
    ex = ((size_t)tpc * N8 * 4 + 15) / 16 * 16;
    exx = ex + (size_t)2 * cl * N4 * 8;
    const size_t exend = exx + (size_t)2 * tpg * cl * xb;
    total = ring > fin ? ring : fin;
    total = total > exend ? total : exend;
  }
};

// W_r [d][N] (fp32, the router's weights as the reference holds them) -> [d][N8] zero-padded, and
// per expert an fp32 upper bound of ||w_i||_2 (sum of squares in fp64, rounded up generously).
__global__ void router_cert_prep_kernel(const float* __restrict__ wr, int d, int N, float* __restrict__ w8,
                                        float* __restrict__ wnorm) {
  const int N8 = (N + 7) / 8 * 8;
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < d * N8; i += gridDim.x * blockDim.x) {
    const int l = i / N8, e = i % N8;
    w8[i] = e < N ? wr[(size_t)l * N + e] : 0.0f;
  }
  if (blockIdx.x == 0)
    for (int e = threadIdx.x; e < N8; e += blockDim.x) {
      double s = 0.0;
      if (e < N)
        for (int l = 0; l < d; ++l) s += (double)wr[(size_t)l * N + e] * (double)wr[(size_t)l * N + e];
      wnorm[e] = static_cast<float>(sqrt(s) * (1.0 + 1e-9)) * (1.0f + 1e-6f);  // upper bound
    }
}

// The 8 values of group q of a swizzled staged x row, held packed (bf16: 4 registers; e4m3: 2;
// fp32: the smem address, read per use) and widened to fp32 on use — the widened copies would
// double the registers of the 8 x 8 accumulator tile. e4m3 codes widen to code * s, the FP8
// scheme's x_hat exactly.
template <typename XT>
struct XPack;
template <>
struct XPack<__nv_bfloat16> {
  uint32_t u[4];
  __device__ __forceinline__ void load(const uint8_t* row, int q, int sw, float) {
    const int4 raw = *reinterpret_cast<const int4*>(row + ((q ^ sw) * 16));
    u[0] = raw.x; u[1] = raw.y; u[2] = raw.z; u[3] = raw.w;
  }
  __device__ __forceinline__ float get(int i) const {
    return __uint_as_float((i & 1) ? (u[i >> 1] & 0xffff0000u) : (u[i >> 1] << 16));
  }
};
template <>
struct XPack<float> {
  const float* p;
  __device__ __forceinline__ void load(const uint8_t* row, int q, int sw, float) {
    p = reinterpret_cast<const float*>(row + (q ^ sw) * 32);
  }
  __device__ __forceinline__ float get(int i) const { return p[i]; }
};
template <>
struct XPack<uint8_t> {
  uint32_t u[2];
  float s;
  __device__ __forceinline__ void load(const uint8_t* row, int q, int sw, float xsc) {
    const uint2 raw = *reinterpret_cast<const uint2*>(row + (((q >> 1) ^ sw) * 16) + (q & 1) * 8);
    u[0] = raw.x;
    u[1] = raw.y;
    s = xsc;
  }
  __device__ __forceinline__ float get(int i) const {
    const __nv_fp8_storage_t c = static_cast<__nv_fp8_storage_t>((u[i >> 2] >> (8 * (i & 3))) & 0xffu);
    const __half_raw hr = __nv_cvt_fp8_to_halfraw(c, __NV_E4M3);
    return __fmul_rn(__half2float(__half(hr)), s);
  }
};

template <typename XT>
__global__ void __launch_bounds__(kCertThreads, 2) router_approx_kernel(const XT* __restrict__ x,
                                                                     const float* __restrict__ xscale,
                                                                     const float* __restrict__ w8,
                                                                     const float* __restrict__ wnorm,
                                                                     const double* __restrict__ w64, int T, int d,
                                                                     int N, int K, float* __restrict__ logits,
                                                                     int* __restrict__ count,
                                                                     int32_t* __restrict__ finite_flag) {
  __shared__ int s_flag[128];  // this CTA's uncertified tokens (tpc <= 128)
  __shared__ int s_nflag;
  if (threadIdx.x == 0) s_nflag = 0;
  constexpr int kXB = sizeof(XT), kRowB = kCertCL * kXB, kPieces = kRowB / 16;
  const RouterCertSmem L(N, kXB);
  const int N8 = L.N8, ng = L.ng, tpc = L.tpc;
  const int tok0 = blockIdx.x * tpc;
  extern __shared__ __align__(16) uint8_t smem_raw[];
  uint8_t* rawx = smem_raw + L.rx;
  float* sw = reinterpret_cast<float*>(smem_raw + L.sw);
  const float xsc = router_xscale(xscale);
  const int pos = threadIdx.x % 16, sl = threadIdx.x / 16;  // position, k-slice
  const int g = pos % ng, tg = pos / ng;
  const bool active = tg < tpc / kCertTT;  // (16 positions; unused ones when ng does not divide 16)
  const int swz = tg & 7;
  float acc[kCertTT][kCertEG];
#pragma unroll
  for (int a = 0; a < kCertTT; ++a)
#pragma unroll
    for (int b = 0; b < kCertEG; ++b) acc[a][b] = 0.0f;
  float xx[kCertTT];  // partial sum of squares of this slice's columns
#pragma unroll
  for (int a = 0; a < kCertTT; ++a) xx[a] = 0.0f;

  const int nchunks = d / kCertCL;
  auto issue = [&](int c, int buf) {
    const int c0 = c * kCertCL;
    for (int i = threadIdx.x; i < tpc * kPieces; i += kCertThreads) {
      const int r = i / kPieces, p = i % kPieces;
      const bool ok = tok0 + r < T;
      const XT* src = x + (size_t)(ok ? tok0 + r : 0) * d + c0 + p * (16 / kXB);
      const int s = (r / kCertTT) & 7;
      int ps;
      if constexpr (kXB == 2) ps = p ^ s;                               // 16-B piece = one 8-column group
      else if constexpr (kXB == 4) ps = ((p >> 1) ^ s) * 2 + (p & 1);  // a group = 2 pieces
      else ps = p ^ s;                                                  // a piece = 2 groups
      cp_async16(rawx + ((size_t)buf * tpc + r) * kRowB + ps * 16, src, ok);
    }
    const float* wsrc = w8 + (size_t)c0 * N8;
    for (int i = threadIdx.x; i < kCertCL * N8 / 4; i += kCertThreads)
      cp_async16(sw + (size_t)buf * kCertCL * N8 + i * 4, wsrc + i * 4, true);
    cp_async_commit();
  };
  for (int c = 0; c < kCertStages - 1; ++c) {
    if (c < nchunks) issue(c, c);
    else cp_async_commit();
  }
  for (int c = 0; c < nchunks; ++c) {
    const int buf = c % kCertStages;
    cp_async_wait<kCertStages - 2>();
    __syncthreads();
    if (c + kCertStages - 1 < nchunks) issue(c + kCertStages - 1, (c + kCertStages - 1) % kCertStages);
    else cp_async_commit();
    const uint8_t* xb = rawx + (size_t)buf * tpc * kRowB;
    const float* wv = sw + (size_t)buf * kCertCL * N8 + g * kCertEG;
    if (!active) continue;
    XPack<XT> xp[kCertTT];
#pragma unroll
    for (int a = 0; a < kCertTT; ++a) xp[a].load(xb + (size_t)(tg * kCertTT + a) * kRowB, sl, swz, xsc);
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int l = sl * 8 + i;
      const float4 w0 = *reinterpret_cast<const float4*>(wv + (size_t)l * N8);
      const float4 w1 = *reinterpret_cast<const float4*>(wv + (size_t)l * N8 + 4);
      const float w[8] = {w0.x, w0.y, w0.z, w0.w, w1.x, w1.y, w1.z, w1.w};
#pragma unroll
      for (int a = 0; a < kCertTT; ++a) {
        const float xa = xp[a].get(i);
#pragma unroll
        for (int b = 0; b < kCertEG; ++b) acc[a][b] = fmaf(xa, w[b], acc[a][b]);
        xx[a] = fmaf(xa, xa, xx[a]);  // |x|^2 (every expert group computes it; group 0's copy is used)
      }
    }
  }
  cp_async_wait<0>();
  __syncthreads();  // the ring is free: reuse it for the k-slice reduction
  float* red = reinterpret_cast<float*>(smem_raw + L.red);
  float* redx = reinterpret_cast<float*>(smem_raw + L.redx);
#pragma unroll
  for (int a = 0; a < kCertTT; ++a) {
    const int tl = tg * kCertTT + a;
    if (!active) break;
#pragma unroll
    for (int b = 0; b < kCertEG; ++b) red[((size_t)sl * tpc + tl) * N8 + g * kCertEG + b] = acc[a][b];
    if (g == 0) redx[sl * tpc + tl] = xx[a];
  }
  __syncthreads();
  for (int i = threadIdx.x; i < tpc * N8; i += kCertThreads) {  // fixed slice order: deterministic
    float v = red[i];
    for (int s2 = 1; s2 < kCertS; ++s2) v += red[(size_t)s2 * tpc * N8 + i];
    red[i] = v;
  }
  for (int tl = threadIdx.x; tl < tpc; tl += kCertThreads) {
    float v = redx[tl];
    for (int s2 = 1; s2 < kCertS; ++s2) v += redx[s2 * tpc + tl];
    redx[tl] = v;
  }
  __syncthreads();
  // certification: one thread per token. Error of a logit: a chain of d/S fp32 FMAs per slice,
  // then S-1 fp32 additions -> |z' - S| <= (g_{d/S} + g_S (1 + g_{d/S})) sum_l |x_l w_l|,
  // sum_l |x_l w_l| <= ||x||_2 ||w||_2 (Cauchy-Schwarz), g_n = n u / (1 - n u), u = 2^-24.
  constexpr double kU = 5.9604644775390625e-08;
  auto gam = [](double n) { return n * kU / (1.0 - n * kU); };
  const double gm = gam((double)d / kCertS) + gam((double)kCertS) * (1.0 + gam((double)d / kCertS));
  const double gx = gam((double)d / kCertS + kCertS);  // |x|^2, same structure
  const int ntok = min(tpc, T - tok0);
  for (int tl = threadIdx.x; tl < ntok; tl += kCertThreads) {
    const float* z = red + (size_t)tl * N8;
    const double xn = sqrt((double)redx[tl] * (1.0 + 2.0 * gx) + 1e-300) * (1.0 + 1e-12);
    // |z' - exact| <= gm ||x|| ||w||; the reference's fp64 chain is within d * 2^-53 sum|x w| of the
    // exact sum, and its fp32 logit within 2^-24 of that (1.2e-7 ~ 2^-23 taken for margin)
    const double gref = gm + (double)d * 1.2e-16;
    auto bound = [&](int e) {
      const double b = gref * xn * (double)wnorm[e] * (1.0 + 1e-9);
      return b + 1.2e-7 * (fabs((double)z[e]) + b) + 1e-37;
    };
    // top-K by z' (descending, lowest index first on equal values), as the reference orders probs
    int top[8];
    bool ok = isfinite(xn);
    uint64_t taken_lo = 0, taken_hi = 0;
    for (int k = 0; k < K; ++k) {
      int best = -1;
      float bv = 0.0f;
      for (int e = 0; e < N; ++e) {
        const bool tk = e < 64 ? ((taken_lo >> e) & 1ull) : ((taken_hi >> (e - 64)) & 1ull);
        if (tk) continue;
        if (best < 0 || z[e] > bv) { best = e; bv = z[e]; }
      }
      top[k] = best;
      if (best < 64) taken_lo |= 1ull << best; else taken_hi |= 1ull << (best - 64);
    }
    constexpr double kMargin = 2.384185791015625e-07;  // 2^-22: keeps the fp32 probabilities strictly ordered
    for (int k = 0; k < K && ok; ++k) {
      const double zk = z[top[k]];
      if (!(fabs(zk) < 1e30)) ok = false;  // also NaN
      const double lo = zk - bound(top[k]);
      if (k + 1 < K) {
        const int nx = top[k + 1];
        ok = ok && lo > (double)z[nx] + bound(nx) + kMargin;
      } else {
        for (int e = 0; e < N && ok; ++e) {
          const bool tk = e < 64 ? ((taken_lo >> e) & 1ull) : ((taken_hi >> (e - 64)) & 1ull);
          if (!tk) ok = fabs((double)z[e]) < 1e30 && lo > (double)z[e] + bound(e) + kMargin;
        }
      }
    }
    // the K-th probability must stay a normal fp32 number (a subnormal / zero tie falls back)
    if (ok && (double)z[top[K - 1]] < (double)z[top[0]] - 75.0) ok = false;
    if (!ok) s_flag[atomicAdd(&s_nflag, 1)] = tl;
  }
  __syncthreads();
  const int nflag = s_nflag;
  if (nflag > 0) {  // (uniform) the reference's exact fp64 chains for the uncertified tokens
    if (threadIdx.x == 0) atomicAdd(count, nflag);
    const int N4 = L.N4, tpg = L.tpg, cl = L.cl;
    double* ew = reinterpret_cast<double*>(smem_raw + L.ex);  // [2][cl][N4]
    XT* exx = reinterpret_cast<XT*>(smem_raw + L.exx);        // [2][tpg][cl]
    const int my = threadIdx.x / N4, e = threadIdx.x % N4;
    const int nch = d / cl;
    constexpr int kXP = 16 / kXB;  // x values per 16-byte piece
    for (int g0 = 0; g0 < nflag; g0 += tpg) {
      const int nt = min(tpg, nflag - g0);
      const bool act = my < nt;
      auto stage = [&](int c, int b) {
        const double* src = w64 + (size_t)c * cl * N4;  // W_r rows [c*cl, (c+1)*cl), [N4] fp64 each
        for (int i = threadIdx.x; i < cl * N4 / 2; i += kCertThreads)
          cp_async16(ew + (size_t)b * cl * N4 + 2 * i, src + 2 * i, true);
        const int pieces = cl / kXP;
        for (int i = threadIdx.x; i < nt * pieces; i += kCertThreads) {
          const int r = i / pieces, pc = i % pieces;
          cp_async16(exx + ((size_t)b * tpg + r) * cl + pc * kXP,
                     x + (size_t)(tok0 + s_flag[g0 + r]) * d + (size_t)c * cl + pc * kXP, true);
        }
        cp_async_commit();
      };
      double acc = 0.0;
      stage(0, 0);
      for (int c = 0; c < nch; ++c) {
        if (c + 1 < nch) stage(c + 1, (c + 1) & 1);
        else cp_async_commit();
        cp_async_wait<1>();
        __syncthreads();
        if (act) {  // ascending l: bit-identical to gemm_nn (tensor.cpp:157-173)
          const double* wv = ew + (size_t)(c & 1) * cl * N4 + e;
          const XT* xv = exx + ((size_t)(c & 1) * tpg + my) * cl;
#pragma unroll 16
          for (int j = 0; j < cl; ++j) acc = fma(x_to_f64<XT>(xv[j], xsc), wv[(size_t)j * N4], acc);
        }
        __syncthreads();
      }
      if (act && e < N) {
        const float z = static_cast<float>(acc);
        red[(size_t)s_flag[g0 + my] * N8 + e] = z;
        if (!isfinite(z)) atomicOr(finite_flag, 1);
      }
    }
    __syncthreads();
  }
  // logits out: fp32 approximations for certified tokens, the reference's values for the others
  for (int i = threadIdx.x; i < ntok * N; i += kCertThreads) {
    const int tl = i / N, e = i % N;
    logits[(size_t)(tok0 + tl) * N + e] = red[(size_t)tl * N8 + e];
  }
}

// K1c: softmax / top-K / combine weights and the per-tile statistics of the dispatch plan from the
// logits in rb.logits (router_finish_warps: the same arithmetic as the exact kernels' tail).
__global__ void __launch_bounds__(256) router_finish_tiles_kernel(int T, int N, int K, RouteBufs rb) {
  const int N4 = (N + 3) / 4 * 4;
  const int tok0 = blockIdx.x * kCertFinTpc;
  __shared__ float slog[kCertFinTpc * 32];  // [tpc][N4], N4 <= 32 here (host checks)
  __shared__ int sidx[kCertFinTpc * 8];
  __shared__ double slse[kCertFinTpc];
  const int ntok = min(kCertFinTpc, T - tok0);
  for (int i = threadIdx.x; i < kCertFinTpc * N4; i += blockDim.x) {
    const int tl = i / N4, e = i % N4;
    slog[i] = (tl < ntok && e < N) ? rb.logits[(size_t)(tok0 + tl) * N + e] : 0.0f;
  }
  __syncthreads();
  router_finish_warps(blockIdx.x, tok0, kCertFinTpc, T, N, N4, K, slog, sidx, slse, rb);
}

}  // namespace cmoe
