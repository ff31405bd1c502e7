// K1, certified large-batch variant (fused forward without a decision export; host_forward.cuh
// run_router). The reference's routing needs the fp64, ascending-l logit chains only to decide
// WHICH experts a token takes and in which order; the fused forward exports neither logits nor
// probabilities. One kernel per tile of tokens (router_cert_kernel):
//   1. every logit in fp32 (4 tokens x 8 experts x 8 columns per thread and chunk, 16 k-slices per
//      CTA, FFMA: 2x the FP64 rate, half the operand bytes), x rows and W_r chunks streamed by a
//      producer warp with 1-D bulk copies into a 4-stage mbarrier ring;
//   2. a rigorous bound on each logit's distance to the reference's fp32 logit:
//      |z' - z_ref| <= (g_{d/S} + g_S (1 + g_{d/S}) + d 2^-53) ||x||_2 ||w_i||_2 + fp32 rounding
//      (recursive fp32 summation per slice + slice sum; Cauchy-Schwarz). A token is CERTIFIED when its
//      top-K order by z' is separated from everything below by more than the bounds plus 2^-22, which
//      keeps the reference's fp32 probabilities strictly ordered (no prob tie can reorder them);
//   3. the uncertified tokens' logits with the reference's exact fp64 chains (bit-identical to
//      gemm_nn, tensor.cpp:157-173), one thread per (token, expert), streamed by the same producer;
//   4. softmax / top-K / combine weights / tile statistics (router_finish_warps), then the plan.
// Routing indices, counts and the dispatch permutation are bit-exact against the reference
// (certified or recomputed); combine weights of certified tokens come from the fp32 logits (within
// ~1e-6 relative, inside the layer's bf16 output tolerance). Decision exports (route_tokens,
// forward with a decision, training) keep the exact kernels.
#pragma once

namespace cmoe {

constexpr int kCertCW = 8;                       // compute warps
constexpr int kCertThreads = kCertCW * 32 + 32;  // + one producer warp
constexpr int kCertTT = 4;                       // tokens per thread
constexpr int kCertEG = 8;                       // experts per thread
constexpr int kCertCL = 128;                     // columns (l) per chunk; k-slice s takes [8s, 8s+8)
constexpr int kCertS = kCertCL / 8;              // 16 k-slices x 16 (token group, expert group) positions
constexpr int kCertStages = 4;                   // ring depth (main and exact phases)
constexpr int kCertXCL = 128;                    // exact phase: columns per chunk

__host__ __device__ inline int cert_n8(int n) {  // expert groups must divide the 16 positions
  int v = 8;
  while (v < n) v *= 2;
  return v;
}

struct RouterCertSmem {
  int N8, ng, tgc, tpc, N4, tpg, rowp, xrow;
  size_t xs, ws, stage, red, redx, sidx, slse, ex, exw, exstage, bars, total;
  __host__ __device__ RouterCertSmem(int n_experts, int xb) {
    N8 = cert_n8(n_experts);
    ng = N8 / kCertEG;
    tgc = 16 / ng;                       // token groups
    tpc = tgc * kCertTT;                 // tokens per CTA
    rowp = kCertCL * xb + 16;            // padded x row (16 B: token groups hit distinct banks)
    xs = (size_t)tpc * rowp;             // per stage: x rows, then the W_r chunk [CL][N8] fp32
    ws = (size_t)kCertCL * N8 * 4;
    stage = xs + ws;
    // after the main loop (the ring is dead): k-slice partials and the per-token tail state
    red = 0;                                            // [S][tpc][N8] fp32 partials -> logits [tpc][N8]
    redx = red + (size_t)kCertS * tpc * N8 * 4;         // [S][tpc] |x|^2 partials
    sidx = redx + (size_t)kCertS * tpc * 4;             // [tpc][8] top-K of the finish
    slse = (sidx + (size_t)tpc * 8 * 4 + 7) / 8 * 8;    // [tpc] lse^2
    // exact phase ring, after the live logits [tpc][N8] (the slice partials are dead by then; the
    // finish's sidx / slse are written only after the exact phase)
    N4 = (n_experts + 3) / 4 * 4;
    tpg = kCertCW * 32 / N4;                            // tokens per exact group
    xrow = kCertXCL * xb;
    exw = (size_t)kCertXCL * N4 * 8;                    // W_r rows [XCL][N4] fp64
    exstage = exw + (size_t)tpg * xrow;
    ex = ((size_t)tpc * N8 * 4 + 127) / 128 * 128;
    size_t end = (size_t)kCertStages * stage;
    const size_t fin = slse + (size_t)tpc * 8;
    if (fin > end) end = fin;
    const size_t exend = ex + (size_t)kCertStages * exstage;
    if (exend > end) end = exend;
    bars = (end + 15) / 16 * 16;                        // full[stages], empty[stages]
    total = bars + 2 * kCertStages * 8;
  }
};

// W_r [d][N] (fp32, the router's weights as the reference holds them) -> [d][N8] zero-padded, and
// per expert an fp32 upper bound of ||w_i||_2 (sum of squares in fp64, rounded up generously).
__global__ void router_cert_prep_kernel(const float* __restrict__ wr, int d, int N, float* __restrict__ w8,
                                        float* __restrict__ wnorm) {
  const int N8 = cert_n8(N);
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

// The 8 values of k-slice `sl` of a staged x row, held packed (bf16: 4 registers; e4m3: 2; fp32:
// the smem address, read per use) and widened to fp32 on use. e4m3 codes widen to code * s, the
// FP8 scheme's x_hat exactly.
template <typename XT>
struct XPack;
template <>
struct XPack<__nv_bfloat16> {
  uint32_t u[4];
  __device__ __forceinline__ void load(const uint8_t* row, int sl, float) {
    const int4 raw = *reinterpret_cast<const int4*>(row + sl * 16);
    u[0] = raw.x; u[1] = raw.y; u[2] = raw.z; u[3] = raw.w;
  }
  __device__ __forceinline__ float get(int i) const {
    return __uint_as_float((i & 1) ? (u[i >> 1] & 0xffff0000u) : (u[i >> 1] << 16));
  }
};
template <>
struct XPack<float> {
  const float* p;
  __device__ __forceinline__ void load(const uint8_t* row, int sl, float) {
    p = reinterpret_cast<const float*>(row + sl * 32);
  }
  __device__ __forceinline__ float get(int i) const { return p[i]; }
};
template <>
struct XPack<uint8_t> {
  uint32_t u[2];
  float s;
  __device__ __forceinline__ void load(const uint8_t* row, int sl, float xsc) {
    const uint2 raw = *reinterpret_cast<const uint2*>(row + sl * 8);
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
__global__ void __launch_bounds__(kCertThreads, 2) router_cert_kernel(const XT* __restrict__ x,
                                                                    const float* __restrict__ xscale,
                                                                    const float* __restrict__ w8,
                                                                    const float* __restrict__ wnorm,
                                                                    const double* __restrict__ w64, int T, int d,
                                                                    int N, int K, RouteBufs rb,
                                                                    int* __restrict__ count) {
  constexpr int kXB = sizeof(XT);
  const RouterCertSmem L(N, kXB);
  const int N8 = L.N8, ng = L.ng, tgc = L.tgc, tpc = L.tpc;
  const int tok0 = blockIdx.x * tpc;
  const int ntok = min(tpc, T - tok0);
  extern __shared__ __align__(128) uint8_t smem_raw[];
  uint64_t* full = reinterpret_cast<uint64_t*>(smem_raw + L.bars);
  uint64_t* empty = full + kCertStages;
  __shared__ int s_flag[64];  // this CTA's uncertified tokens (tpc <= 64)
  __shared__ int s_nflag;
  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const bool producer = warp == kCertCW;
  if (threadIdx.x == 0) {
    for (int s = 0; s < kCertStages; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCertCW);
    }
    fence_mbar_init();
    s_nflag = 0;
  }
  __syncthreads();
  const float xsc = router_xscale(xscale);
  const int nchunks = d / kCertCL;

  // ---------------- 1. fp32 logits ----------------
  const int pos = threadIdx.x % 16, sl = threadIdx.x / 16;  // (compute threads) position, k-slice
  const int g = pos % ng, tg = pos / ng;
  float acc[kCertTT][kCertEG];
  float xx[kCertTT];
#pragma unroll
  for (int a = 0; a < kCertTT; ++a) {
    xx[a] = 0.0f;
#pragma unroll
    for (int b = 0; b < kCertEG; ++b) acc[a][b] = 0.0f;
  }
  if (producer) {
    if (lane == 0) {
      const uint32_t rowb = kCertCL * kXB, wb = (uint32_t)L.ws;
      for (int c = 0; c < nchunks; ++c) {
        const int s = c % kCertStages;
        if (c >= kCertStages) mbar_wait(&empty[s], ((c / kCertStages) - 1) & 1);
        uint8_t* st = smem_raw + (size_t)s * L.stage;
        mbar_arrive_expect_tx(&full[s], ntok * rowb + wb);
        bulk_g2s(st + L.xs, w8 + (size_t)c * kCertCL * N8, wb, &full[s]);
        for (int r = 0; r < ntok; ++r)
          bulk_g2s(st + (size_t)r * L.rowp, x + (size_t)(tok0 + r) * d + (size_t)c * kCertCL, rowb, &full[s]);
      }
    }
  } else {
    for (int c = 0; c < nchunks; ++c) {
      const int s = c % kCertStages;
      mbar_wait(&full[s], (c / kCertStages) & 1);
      const uint8_t* st = smem_raw + (size_t)s * L.stage;
      const float* wv = reinterpret_cast<const float*>(st + L.xs) + g * kCertEG;
      XPack<XT> xp[kCertTT];
#pragma unroll
      for (int a = 0; a < kCertTT; ++a) xp[a].load(st + (size_t)(tg + tgc * a) * L.rowp, sl, xsc);
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
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  __syncthreads();  // every chunk consumed: the ring is dead, reuse it
  float* red = reinterpret_cast<float*>(smem_raw + L.red);
  float* redx = reinterpret_cast<float*>(smem_raw + L.redx);
  if (!producer) {
#pragma unroll
    for (int a = 0; a < kCertTT; ++a) {
      const int tl = tg + tgc * a;
#pragma unroll
      for (int b = 0; b < kCertEG; ++b) red[((size_t)sl * tpc + tl) * N8 + g * kCertEG + b] = acc[a][b];
      if (g == 0) redx[sl * tpc + tl] = xx[a];
    }
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

  // ---------------- 2. certification: one thread per token ----------------
  constexpr double kU = 5.9604644775390625e-08;  // 2^-24
  auto gam = [](double n) { return n * kU / (1.0 - n * kU); };
  const double gm = gam((double)d / kCertS) + gam((double)kCertS) * (1.0 + gam((double)d / kCertS));
  const double gx = gam((double)d / kCertS + kCertS);  // |x|^2, same structure
  const double gref = gm + (double)d * 1.2e-16;         // + the reference's fp64 chain vs the exact sum
  for (int tl = threadIdx.x; tl < ntok; tl += kCertThreads) {
    const float* z = red + (size_t)tl * N8;
    const double xn = sqrt((double)redx[tl] * (1.0 + 2.0 * gx) + 1e-300) * (1.0 + 1e-12);
    auto bound = [&](int e) {  // + the fp32 rounding of the reference logit (1.2e-7 ~ 2^-23 for margin)
      const double b = gref * xn * (double)wnorm[e] * (1.0 + 1e-9);
      return b + 1.2e-7 * (fabs((double)z[e]) + b) + 1e-37;
    };
    int top[8];
    bool ok = isfinite(xn);
    uint64_t taken_lo = 0, taken_hi = 0;
    for (int k = 0; k < K; ++k) {  // top-K by z' (descending, lowest index first on equal values)
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

  // ---------------- 3. the reference's exact chains for the uncertified tokens ----------------
  const int nflag = s_nflag;
  if (nflag > 0) {  // (uniform)
    if (threadIdx.x == 0) atomicAdd(count, nflag);
    const int N4 = L.N4, tpg = L.tpg;
    const int nxc = d / kCertXCL;
    const int my = threadIdx.x / N4, e = threadIdx.x % N4;
    int it = nchunks;  // ring index continues from the main loop (barrier phases)
    for (int g0 = 0; g0 < nflag; g0 += tpg) {
      const int nt = min(tpg, nflag - g0);
      if (producer) {
        if (lane == 0) {
          const uint32_t xrow = (uint32_t)L.xrow, wbytes = (uint32_t)L.exw;
          for (int c = 0; c < nxc; ++c) {
            const int i = it + c, s = i % kCertStages;
            if (i >= kCertStages) mbar_wait(&empty[s], ((i / kCertStages) - 1) & 1);
            uint8_t* st = smem_raw + L.ex + (size_t)s * L.exstage;
            mbar_arrive_expect_tx(&full[s], wbytes + nt * xrow);
            bulk_g2s(st, w64 + (size_t)c * kCertXCL * N4, wbytes, &full[s]);
            for (int r = 0; r < nt; ++r)
              bulk_g2s(st + L.exw + (size_t)r * xrow, x + (size_t)(tok0 + s_flag[g0 + r]) * d + (size_t)c * kCertXCL,
                       xrow, &full[s]);
          }
        }
      } else {
        const bool act = my < nt;
        double dacc = 0.0;
        for (int c = 0; c < nxc; ++c) {
          const int i = it + c, s = i % kCertStages;
          mbar_wait(&full[s], (i / kCertStages) & 1);
          if (act) {  // ascending l: bit-identical to gemm_nn (tensor.cpp:157-173)
            const uint8_t* st = smem_raw + L.ex + (size_t)s * L.exstage;
            const double* wv = reinterpret_cast<const double*>(st) + e;
            const XT* xv = reinterpret_cast<const XT*>(st + L.exw + (size_t)my * L.xrow);
#pragma unroll 16
            for (int j = 0; j < kCertXCL; ++j) dacc = fma(x_to_f64<XT>(xv[j], xsc), wv[(size_t)j * N4], dacc);
          }
          __syncwarp();
          if (lane == 0) mbar_arrive(&empty[s]);
        }
        if (act && e < N) {
          const float zz = static_cast<float>(dacc);
          red[(size_t)s_flag[g0 + my] * N8 + e] = zz;
          if (!isfinite(zz)) atomicOr(rb.finite_flag, 1);
        }
      }
      it += nxc;
      __syncthreads();
    }
  }

  // ---------------- 4. softmax / top-K / combine weights / tile statistics ----------------
  router_finish_warps(blockIdx.x, tok0, tpc, T, N, N8, K, red, reinterpret_cast<int*>(smem_raw + L.sidx),
                      reinterpret_cast<double*>(smem_raw + L.slse), rb);
}

}  // namespace cmoe
