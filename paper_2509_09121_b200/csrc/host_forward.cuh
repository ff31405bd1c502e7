// Single-GPU forward orchestration: router, plan, dispatch, grouped-GEMM launches, combine.
// Host side of libcompass_moe.so, included once, in order, by capi.cu (a single translation
// unit; the helpers live in an anonymous namespace).
#pragma once

namespace {

// m-tiles per L2-resident group for a row-grouped GEMM whose A rows are k_bytes long (decode_tile).
int64_t l2_group_budget() {
  static const int64_t budget = [] {
    const char* e = std::getenv("CL_MOE_L2_GROUP_MB");
    return (int64_t)(e ? std::atoi(e) : 32) << 20;
  }();
  return budget;
}
// Integer tuning knob from the environment (read once by the callers' statics).
int gemm_env(const char* name, int dflt) {
  const char* e = std::getenv(name);
  return e ? std::atoi(e) : dflt;
}
int m_group_for(int64_t k_bytes, int bm) {
  const int64_t budget = l2_group_budget();
  if (budget <= 0) return 0;
  return static_cast<int>(std::max<int64_t>(1, budget / (k_bytes * bm)));
}

template <int G, int EPI, bool F8, bool OF8, bool WG = false, int CM = 1>
void launch_gemm(cl_moe* h, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args_in, cudaStream_t st,
                 int grid_sms = 0) {
  if (!h->tile_counter) h->tile_counter = dalloc<int>(1);
  GemmArgs args = args_in;
  args.tile_counter = h->tile_counter;
  // Smallest m-group of the tile orders (row-grouped and weight-gradient). When an expert's A
  // slabs are too long for the L2 budget (dgrad2's K = 2f, the weight gradients of a hot expert),
  // the budget alone gives groups of 1-2 m-tiles; with the dynamic scheduler the running tiles'
  // start times spread over one tile duration, so an L2 line is reused only by tiles claimed
  // within a few dozen of each other, and the slabs such a window touches (gm A + window/gm B) are
  // fewest at a few m-tiles per group. Measured on C5 (tools/gemm_dram_sweep.sh, floors 1-16):
  // dgrad2 DRAM reads 76 -> 55 GB at 4, dW_in 97 -> 41 GB and dW_out 35 -> 24 GB at 6, C5 step
  // -5 %; a row-grouped floor of 6 slowed C2's GEMM2 (budget 4) by 1 %, so it stays at 4.
  static const int gm_min = gemm_env("CL_MOE_GEMM_GROUP_MIN", 4), wg_gm_min = gemm_env("CL_MOE_WGRAD_GROUP_MIN", 6);
  if (!WG && args.m_group == 0) {
    const int g = m_group_for((int64_t)args.num_kb * kBKBytes, 128 * G);
    args.m_group = g > 0 ? std::max(1, std::max(g, gm_min) / CM) : 0;
  }
  if (WG && args.group_bytes == 0) args.group_bytes = l2_group_budget();
  if (WG) args.m_group = wg_gm_min;
  // (measurement knobs: L2 hints of the operand loads, 0 = default / 1 normal / 2 last / 3 first)
  static const uint64_t hints[4] = {0, kEvictNormal, kEvictLast, kEvictFirst};
  static const int a_hint = gemm_env("CL_MOE_GEMM_A_HINT", 0) & 3, b_hint = gemm_env("CL_MOE_GEMM_B_HINT", 0) & 3;
  if (!args.a_hint) args.a_hint = hints[a_hint];
  if (!args.b_hint) args.b_hint = hints[b_hint];
  static const int pf_kb = gemm_env("CL_MOE_GEMM_PREFETCH_KB", 0), pf_lead = gemm_env("CL_MOE_GEMM_PREFETCH_LEAD", 12);
  if (!WG) {
    args.prefetch_kb = pf_kb;
    args.prefetch_lead = pf_lead;
  }
  CK(cudaMemsetAsync(h->tile_counter, 0, sizeof(int), st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(((grid_sms > 0 ? std::min(grid_sms, h->num_sms) : h->num_sms) / (G * CM)) * (G * CM));
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = GemmCfg<G>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G * CM;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<G, EPI, F8, OF8, WG, CM>, a, b, args));
}

// K1 launch for router input type XT (bf16 storage, or the caller's fp32 tensor): the variant and
// tile geometry were chosen by run_router (tpc does not depend on XT).
template <typename XT>
void launch_router(cl_moe* h, const XT* x, const double* w64, int64_t T, int N, int n_tiles, int variant, int ws_cons,
                   int big_tok, int lat_chunk, int* tail, float* rwd, int32_t* invd, cudaStream_t st,
                   const float* xs = nullptr) {
  constexpr int xb = sizeof(XT);
  const int d = (int)h->d, K = (int)h->K;
  switch (variant) {
    case 5: {  // dmma (fp64 tensor cores): ws_cons carries the warps per CTA (2 or 4; 8 tokens
               // each); w64 points at the [d][N4] layout, the fragments follow. Then the finish.
      const double* wf = w64 + router_wfrag_offset(d, N);
      const size_t smem = RouterDmmaSmem(N, ws_cons, xb).total;
      const int nt = dmma_n8(N) / 8;
#define CL_MOE_DMMA_LAUNCH(NT, W) \
  router_dmma_kernel<NT, W, XT><<<dm_tiles, W * 32, smem, st>>>(x, wf, (int)T, d, N, h->rb, xs)
      const int dm_tiles = static_cast<int>((T + ws_cons * 8 - 1) / (ws_cons * 8));
      if (ws_cons == 4) {
        if (nt == 1) CL_MOE_DMMA_LAUNCH(1, 4);
        else if (nt == 2) CL_MOE_DMMA_LAUNCH(2, 4);
        else CL_MOE_DMMA_LAUNCH(4, 4);
      } else {
        if (nt == 1) CL_MOE_DMMA_LAUNCH(1, 2);
        else if (nt == 2) CL_MOE_DMMA_LAUNCH(2, 2);
        else CL_MOE_DMMA_LAUNCH(4, 2);
      }
#undef CL_MOE_DMMA_LAUNCH
      CK(cudaGetLastError());
      router_finish_kernel<<<n_tiles, router_finish_threads(N), router_finish_smem(N, router_finish_tpc(N)), st>>>(
          (int)T, N, K, router_finish_tpc(N), h->rb);
      break;
    }
    case 4:  // ws
      if (ws_cons == 32)
        router_ws_kernel<32, XT><<<n_tiles, 32 + 64, RouterWsSmem(N, 32, xb).total, st>>>(x, w64, (int)T, d, N, K,
                                                                                          h->rb, tail, rwd, invd, xs);
      else if (ws_cons == 64)
        router_ws_kernel<64, XT><<<n_tiles, 64 + 64, RouterWsSmem(N, 64, xb).total, st>>>(x, w64, (int)T, d, N, K,
                                                                                          h->rb, tail, rwd, invd, xs);
      else
        router_ws_kernel<128, XT><<<n_tiles, 128 + 64, RouterWsSmem(N, 128, xb).total, st>>>(x, w64, (int)T, d, N,
                                                                                             K, h->rb, tail, rwd, invd, xs);
      break;
    case 3:  // lat (bf16 only: the A/B variant kept from round 1)
      if constexpr (xb == 2) {
        if (lat_chunk == 256)
          router_lat_kernel<3, 256><<<n_tiles, 128, RouterLatSmem<3, 256>(N).total, st>>>(x, w64, (int)T, d, N, K, h->rb);
        else if (lat_chunk == 128)
          router_lat_kernel<3, 128><<<n_tiles, 128, RouterLatSmem<3, 128>(N).total, st>>>(x, w64, (int)T, d, N, K, h->rb);
        else
          router_lat_kernel<3, 64><<<n_tiles, 128, RouterLatSmem<3, 64>(N).total, st>>>(x, w64, (int)T, d, N, K, h->rb);
      }
      break;
    case 2:  // big
      if (big_tok == 2)
        router_big_kernel<32, 3, 2, XT><<<n_tiles, 32, RouterBigSmem(N, 32, 3, 2, xb).total, st>>>(x, w64, (int)T, d,
                                                                                                  N, K, h->rb, xs);
      else
        router_big_kernel<32, 3, 4, XT><<<n_tiles, 32, RouterBigSmem(N, 32, 3, 4, xb).total, st>>>(x, w64, (int)T, d,
                                                                                                  N, K, h->rb, xs);
      break;
    case 1:  // small
      router_kernel<32, 8, XT><<<n_tiles, 32, router_smem_bytes(N, 32, 8, xb), st>>>(x, w64, (int)T, d, N, K, h->rb, xs);
      break;
    default:
      router_kernel<128, 3, XT><<<n_tiles, 128, router_smem_bytes(N, 128, 3, xb), st>>>(x, w64, (int)T, d, N, K,
                                                                                       h->rb, xs);
  }
}

// Certified large-batch K1 (router_cert.cuh): approximate fp32 logits + bound, exact fp64 chains for
// the tokens whose decision is not certified, then softmax / top-K / tile statistics. Fused forward
// without a decision export only (h->need_exact false). Opt-in (CL_MOE_ROUTER_CERT=1, read per call):
// on this B200 it did not beat the exact large-batch kernel (DESIGN.md §4 K1).
bool cert_enabled() {
  const char* e = std::getenv("CL_MOE_ROUTER_CERT");
  return e && e[0] == '1';
}

// Allocates the certified router's buffers and rebuilds its fp32 W_r copy when the weights changed
// (also called before a CUDA-graph capture: no allocation while capturing).
void cert_prepare(cl_moe* h, bool fp8, cudaStream_t st) {
  const int N = static_cast<int>(h->N), d = static_cast<int>(h->d), N8 = cert_n8(N);
  if (!h->cert_count) h->cert_count = dalloc<int>(1);
  float*& w8 = fp8 ? h->cert_w8q : h->cert_w8;
  float*& wn = fp8 ? h->cert_wnq : h->cert_wn;
  int64_t& ver = fp8 ? h->cert_verq : h->cert_ver;
  const int64_t cur = fp8 ? h->wrq_ver : h->wr_ver;
  if (!w8) {
    w8 = dalloc<float>((size_t)d * N8);
    wn = dalloc<float>(N8);
  }
  if (ver != cur) {
    router_cert_prep_kernel<<<grid_for((int64_t)d * 8), 256, 0, st>>>(fp8 ? h->wrq : h->wr, d, N, w8, wn);
    CK(cudaGetLastError());
    ver = cur;
  }
}

int cert_tpc(int N, int xb) { return RouterCertSmem(N, xb).tpc; }

template <typename XT>
void launch_router_cert(cl_moe* h, const XT* x, const float* xs, bool fp8, int64_t T, cudaStream_t st) {
  const int N = static_cast<int>(h->N), d = static_cast<int>(h->d);
  cert_prepare(h, fp8, st);
  CK(cudaMemsetAsync(h->cert_count, 0, sizeof(int), st));
  const RouterCertSmem L(N, sizeof(XT));
  router_cert_kernel<XT><<<(int)((T + L.tpc - 1) / L.tpc), kCertThreads, L.total, st>>>(
      x, xs, fp8 ? h->cert_w8q : h->cert_w8, fp8 ? h->cert_wnq : h->cert_wn, fp8 ? h->wr64q : h->wr64, (int)T, d, N,
      (int)h->K, h->rb, h->cert_count);
  CK(cudaGetLastError());
  ++h->cert_calls;
}

// route_tokens on device: K1 + K2. `xf32`: x is the caller's fp32 tensor (routing on the
// reference's own values), else bf16.
// dense = true (dense decode): the 128-thread warp-specialised router with the plan and the dense
// row weights fused into its last CTA, when that variant applies (returns whether it did).
bool run_router(cl_moe* h, const void* x, int64_t T, cudaStream_t st, bool own_prof = true, bool dense = false,
                bool xf32 = false) {
  if (T < 1) throw RunErr("route_tokens: B must be >= 1");
  if (T > h->cap) throw ConfigErr(fmt("T=%lld exceeds max_tokens=%lld", (long long)T, (long long)h->cap));
  const int N = static_cast<int>(h->N);
  // FP8 scheme: the router consumes qdq(x) as fp32 (see below), so size the variants for fp32
  const bool rq = h->precision == CL_MOE_FP8_E4M3 && h->router_fp8;
  const int xb = rq ? 1 : xf32 ? 4 : 2;  // router input bytes per value (FP8 scheme: E4M3 codes)
  // small batches: 1 token x 4 experts per thread, 32-thread CTAs, 8-deep prefetch ring (latency);
  // large batches: 4 tokens x 4 experts per thread (shared-memory traffic per DFMA / 3).
  // decode-size batches: one thread per (token, expert) chain (latency-bound: parallelism first).
  static const int force = [] {
    const char* e = std::getenv("CL_MOE_ROUTER");  // test override: "ws", "lat", "small", "big" or "dmma"
    return e ? (e[0] == 'b' ? 2 : e[0] == 's' ? 1 : e[0] == 'l' ? 3 : e[0] == 'w' ? 4 : e[0] == 'd' ? 5 : 0) : 0;
  }();
  // large batches: 4 tokens x 4 experts per thread when that still gives >= 3 CTAs per SM, else
  // 2 x 4 (2x the CTAs, e.g. C3's 8192 tokens); CL_MOE_BIG_TOK=2|4 pins the choice (benchmarks)
  static const int big_tok_env = [] {
    const char* e = std::getenv("CL_MOE_BIG_TOK");
    return e ? std::atoi(e) : 0;
  }();
  const int tiles4 = (int)((T + RouterBigSmem(N, 32, 3, 4).tpc - 1) / RouterBigSmem(N, 32, 3, 4).tpc);
  const int big_tok = big_tok_env == 2 || big_tok_env == 4 ? big_tok_env : (tiles4 >= 3 * h->num_sms ? 4 : 2);
  const int tpc_big = RouterBigSmem(N, 32, 3, big_tok).tpc;
  const bool big_ok = RouterBigSmem(N, 32, 3, big_tok, xb).total <= 220 * 1024;
  const bool big = big_ok && (force == 2 || (force == 0 && (T + tpc_big - 1) / tpc_big >= h->num_sms));
  // latency variant: chunk length by expert count (shared-memory budget), ring depth 3
  const int N4r = (N + 3) / 4 * 4;
  const int lat_chunk = N4r <= 16 ? 256 : N4r <= 32 ? 128 : 64;
  const int tpc_lat = RouterLatSmem<3, 64>(N).tpc;
  const bool lat_size = (T + tpc_lat - 1) / tpc_lat <= h->num_sms;
  // decode-size batches: the warp-specialised chain kernel (ws), on the smallest CTA (32 / 64 / 128
  // chain threads) that still gives every CTA its own SM; CL_MOE_ROUTER=lat keeps the older variant
  // (bf16 input only; fp32 input takes ws)
  const bool ws = !big && (force == 4 || (force == 0 && lat_size) || (force == 3 && xb != 2));
  const bool lat = !big && !ws && (force == 3 || (force == 0 && lat_size));
  int ws_cons = 128;
  for (int c : {32, 64}) {
    const int tp = RouterWsSmem(N, c, xb).tpc;
    if (ws_cons == 128 && tp >= 1 && (T + tp - 1) / tp <= h->num_sms) ws_cons = c;
  }
  if (dense) ws_cons = 128;  // dense decode: fewest CTAs (the router runs beside GEMM1)
  const bool fuse = dense && ws && RouterWsSmem(N, 128, xb).tpc >= 1 && h->route_ctr;  // (ensure_dense allocates)
  int* tail = fuse ? h->route_ctr : nullptr;
  float* rwd = fuse ? h->rwd : nullptr;
  int32_t* invd = fuse ? h->invd : nullptr;
  const bool small = !big && !lat && !ws && router_smem_bytes(N, 32, 8, xb) <= 220 * 1024;
  // batches beyond the decode sizes: the fp64 tensor-core router (router_dmma_kernel), when the
  // device check passed and the experts fit its instantiations (N <= 32)
  const int nt8 = dmma_n8(N) / 8;
  // 4 warps (32 tokens) per CTA when that still leaves >= 2 CTAs per SM, else 2 (16 tokens)
  const int dmma_w = (T + 31) / 32 >= 2 * h->num_sms ? 4 : 2;
  const bool dmma_fit = h->dmma_ok && (nt8 == 1 || nt8 == 2 || nt8 == 4) &&
                        RouterDmmaSmem(N, dmma_w, xb).total <= 220 * 1024;
  // (the opt-in certified router takes precedence when enabled)
  const bool cert = big && !h->need_exact && !dense && N <= 32 && cert_enabled() && force == 0;
  const bool dmma = dmma_fit && !cert && (force == 5 || (force == 0 && !lat_size && !dense));
  const int tpc = dmma ? router_finish_tpc(N) : big ? tpc_big : ws ? RouterWsSmem(N, ws_cons, xb).tpc : lat ? tpc_lat
                                 : router_tokens_per_cta(N, small ? 32 : 128);
  const int variant = dmma ? 5 : ws ? 4 : lat ? 3 : big ? 2 : small ? 1 : 0;
  const int tpc_eff = cert ? cert_tpc(N, xb) : tpc;
  h->tpc_cur = tpc_eff;
  h->last_router_variant = cert ? 6 : variant;
  h->last_tokens = T;
  const int n_tiles = static_cast<int>((T + tpc_eff - 1) / tpc_eff);
  if (own_prof) prof_begin(h, st);
  if (rq) {
    // router GEMM under the FP8 scheme: x_hat = qdq(x, s_x) per tensor (E4M3 codes,
    // widened as code * s_x inside K1), W_r_hat per expert column (quantize time)
    const int64_t n = T * h->d;
    if (xf32)
      router_qdq8_kernel<float><<<grid_for(n / 16), 256, 0, st>>>(static_cast<const float*>(x), n, h->sxr_dev, h->xq8);
    else
      router_qdq8_kernel<__nv_bfloat16><<<grid_for(n / 16), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), n,
                                                                           h->sxr_dev, h->xq8);
    CK(cudaGetLastError());
    if (cert)
      launch_router_cert<uint8_t>(h, h->xq8, h->sxr_dev, true, T, st);
    else
      launch_router<uint8_t>(h, h->xq8, h->wr64q, T, N, n_tiles, variant, dmma ? dmma_w : ws_cons, big_tok, lat_chunk, tail, rwd, invd,
                             st, h->sxr_dev);
  } else if (cert && xf32) {
    launch_router_cert<float>(h, static_cast<const float*>(x), nullptr, false, T, st);
  } else if (cert) {
    launch_router_cert<__nv_bfloat16>(h, static_cast<const __nv_bfloat16*>(x), nullptr, false, T, st);
  } else if (xf32)
    launch_router<float>(h, static_cast<const float*>(x), h->wr64, T, N, n_tiles, variant, dmma ? dmma_w : ws_cons, big_tok, lat_chunk, tail,
                         rwd, invd, st);
  else
    launch_router<__nv_bfloat16>(h, static_cast<const __nv_bfloat16*>(x), h->wr64, T, N, n_tiles, variant, dmma ? dmma_w : ws_cons, big_tok,
                                 lat_chunk, tail, rwd, invd, st);
  CK(cudaGetLastError());
  prof_mark(h, 0, st);
  if (!fuse) launch_plan(n_tiles, (int)T, N, (int)h->K, h->rb, st);
  CK(cudaGetLastError());
  prof_mark(h, 1, st);
  return fuse;
}

void plan_from_decision(cl_moe* h, const int32_t* idx, const float* w, int64_t T, cudaStream_t st) {
  if (T < 1) throw RunErr("moe_forward: B must be >= 1");
  if (T > h->cap) throw ConfigErr(fmt("T=%lld exceeds max_tokens=%lld", (long long)T, (long long)h->cap));
  const int N = static_cast<int>(h->N);
  const int tpc = router_tokens_per_cta(N, 128);
  h->tpc_cur = tpc;
  h->last_tokens = T;
  const int n_tiles = static_cast<int>((T + tpc - 1) / tpc);
  CK(cudaMemcpyAsync(h->rb.topk_idx, idx, sizeof(int32_t) * T * h->K, cudaMemcpyDeviceToDevice, st));
  CK(cudaMemcpyAsync(h->rb.combine_w, w, sizeof(float) * T * h->K, cudaMemcpyDeviceToDevice, st));
  prof_begin(h, st);
  decision_tiles_kernel<<<n_tiles, 128, 0, st>>>(h->rb.topk_idx, (int)T, N, (int)h->K, tpc, h->rb);
  CK(cudaGetLastError());
  prof_mark(h, 0, st);
  launch_plan(n_tiles, (int)T, N, (int)h->K, h->rb, st);
  CK(cudaGetLastError());
  prof_mark(h, 1, st);
}

// GEMM1 (+SwiGLU) and GEMM2 (+optional row weight) over the local expert segments `offsets`.
void run_gemms(cl_moe* h, const int32_t* offsets, void* act, __nv_bfloat16* y, const float* row_w,
               const CUtensorMap* mA1, const CUtensorMap* mA2, const CUtensorMap* mA1q, const CUtensorMap* mA2q,
               cudaStream_t st, __nv_bfloat16* h_save = nullptr, void* const* row_ptr = nullptr,
               cudaEvent_t g2_wait = nullptr, const uint32_t* g1_arrive = nullptr,
               const uint32_t* g1_arrive_tgt = nullptr, const int32_t* a1_poff = nullptr,
               const CUtensorMap* mA2_padded = nullptr) {
  const bool fp8 = h->precision == CL_MOE_FP8_E4M3;
  GemmArgs g1{};
  g1.offsets = offsets;
  if (h->gemm_auto) {
    // M=256 CTA-pair tiles pay off only when experts have enough rows; small batches (decode)
    // stream weights and are better served by M=128 tiles (less A over-fetch per B byte).
    const int64_t rows_per_expert = h->last_tokens * h->K * (h->cfg.ep_size > 1 ? h->cfg.ep_size : 1) / h->n_local;
    h->gemm_ctas = rows_per_expert >= 1024 ? 2 : 1;
  }
  g1.n_experts = h->n_local;
  g1.arrive = g1_arrive;  // EP dispatch overlap: wait for the peers' rows per expert
  g1.arrive_tgt = g1_arrive_tgt;
  g1.err_flag = h->rb.finite_flag;
  g1.n_tiles_n = static_cast<int>(2 * h->f / kBN);
  g1.num_kb = static_cast<int>(h->d * (fp8 ? 1 : 2) / kBKBytes);
  g1.b_rows_per_expert = static_cast<int>(2 * h->f);
  g1.out = act;
  g1.ldo = static_cast<int>(h->f);
  g1.a_poff = a1_poff;  // single-GPU training: the dispatched rows sit in the padded layout
  if (mA2_padded) g1.out = nullptr;  // ... and A is written only there (aux_t), GEMM2 reads it there
  g1.act_scale = h->sx_in;
  g1.w_scale = h->ws_in;
  g1.out_scale = h->sx_mid;
  g1.aux = h_save;
  g1.ffn = static_cast<int>(h->f);
  if (h_save) {  // training: also write A^T into the padded K-major buffer of the dW_out GEMM
    g1.aux_t = h->AT;
    g1.rp = h->rp_cap;
    g1.poff = h->poff;
  }
  GemmArgs g2{};
  g2.offsets = offsets;
  g2.n_experts = h->n_local;
  g2.n_tiles_n = static_cast<int>(h->d / kBN);
  g2.num_kb = static_cast<int>(h->f * (fp8 ? 1 : 2) / kBKBytes);
  g2.b_rows_per_expert = static_cast<int>(h->d);
  g2.out = y;
  g2.ldo = static_cast<int>(h->d);
  g2.row_scale = row_w;
  g2.row_ptr = row_ptr;
  g1.half_tail = g2.half_tail = 1;  // 2-CTA: tail m-tiles of <= 128 rows as M=128 pair MMAs
  g2.act_scale = h->sx_mid;
  g2.w_scale = h->ws_out;
  if (mA2_padded) {
    g2.a_poff = h->poff;
    mA2 = mA2_padded;
  }
  const int v = h->gemm_ctas == 2 ? 1 : 0;
  // clusters of two CTA pairs sharing the B tile by TMA multicast (CL_MOE_GEMM_MC=1)
  static const bool mc_env = [] {
    const char* e = std::getenv("CL_MOE_GEMM_MC");
    return e && e[0] == '1';
  }();
  const bool mc = mc_env && v && !h_save && h->g1_grid == 0 && h->num_sms % 4 == 0;
  if (mc && !fp8) {
    launch_gemm<2, EPI_SWIGLU, false, false, false, 2>(h, mA1[v], h->mB1m, g1, st);
    prof_mark(h, 3, st);
    if (g2_wait) CK(cudaStreamWaitEvent(st, g2_wait, 0));
    launch_gemm<2, EPI_ROWSCALE, false, false, false, 2>(h, mA2[v], h->mB2m, g2, st);
  } else if (mc) {
    launch_gemm<2, EPI_SWIGLU, true, true, false, 2>(h, mA1q[v], h->mB1qm, g1, st);
    prof_mark(h, 3, st);
    if (g2_wait) CK(cudaStreamWaitEvent(st, g2_wait, 0));
    launch_gemm<2, EPI_ROWSCALE, true, false, false, 2>(h, mA2q[v], h->mB2qm, g2, st);
  } else if (!fp8) {
    if (v) {
      launch_gemm<2, EPI_SWIGLU, false, false>(h, mA1[v], h->mB1[v], g1, st, h->g1_grid);
      prof_mark(h, 3, st);
      if (g2_wait) CK(cudaStreamWaitEvent(st, g2_wait, 0));
      launch_gemm<2, EPI_ROWSCALE, false, false>(h, mA2[v], h->mB2[v], g2, st);
    } else {
      launch_gemm<1, EPI_SWIGLU, false, false>(h, mA1[v], h->mB1[v], g1, st, h->g1_grid);
      prof_mark(h, 3, st);
      if (g2_wait) CK(cudaStreamWaitEvent(st, g2_wait, 0));
      launch_gemm<1, EPI_ROWSCALE, false, false>(h, mA2[v], h->mB2[v], g2, st);
    }
  } else {
    if (v) {
      launch_gemm<2, EPI_SWIGLU, true, true>(h, mA1q[v], h->mB1q[v], g1, st, h->g1_grid);
      prof_mark(h, 3, st);
      if (g2_wait) CK(cudaStreamWaitEvent(st, g2_wait, 0));
      launch_gemm<2, EPI_ROWSCALE, true, false>(h, mA2q[v], h->mB2q[v], g2, st);
    } else {
      launch_gemm<1, EPI_SWIGLU, true, true>(h, mA1q[v], h->mB1q[v], g1, st, h->g1_grid);
      prof_mark(h, 3, st);
      if (g2_wait) CK(cudaStreamWaitEvent(st, g2_wait, 0));
      launch_gemm<1, EPI_ROWSCALE, true, false>(h, mA2q[v], h->mB2q[v], g2, st);
    }
  }
}

// dispatch + expert FFN + combine (local experts; ep_size == 1).
void run_ep(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st, bool train = false);

void run_experts(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st) {
  if (h->comm) {  // expert parallel (one rank: loopback through the same exchange code)
    run_ep(h, x, T, out, out_f32, st);
    return;
  }
  if (!h->ep_abort_reason.empty()) throw RunErr(h->ep_abort_reason);  // communicator aborted (host_ep.cuh ep_wait)
  if (h->cfg.ep_size > 1) throw ConfigErr("ep_size > 1 needs cl_moe_ep_init (or cl_moe_ep_group_forward)");
  const int N = static_cast<int>(h->N);
  const int tpc = h->tpc_cur;
  const bool fp8 = h->precision == CL_MOE_FP8_E4M3;
  const int blocks = static_cast<int>((T + 7) / 8);
  if (fp8)
    dispatch_kernel<true><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N, (int)h->K,
                                                  tpc, h->rb, h->rb.topk_idx, h->rb.combine_w, h->xperm, h->perm,
                                                  h->inv, h->row_w, h->sx_in);
  else
    dispatch_kernel<false><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N,
                                                   (int)h->K, tpc, h->rb, h->rb.topk_idx, h->rb.combine_w, h->xperm,
                                                   h->perm, h->inv, h->row_w, nullptr);
  CK(cudaGetLastError());
  prof_mark(h, 2, st);

  run_gemms(h, h->rb.offsets, h->act, h->y, h->row_w, h->mA1, h->mA2, h->mA1q, h->mA2q, st);
  prof_mark(h, 4, st);
  if (out_f32)
    launch_combine<float>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<float*>(out), h->rb.finite_flag, st);
  else
    launch_combine<__nv_bfloat16>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<__nv_bfloat16*>(out),
                                  h->rb.finite_flag, st);
  CK(cudaGetLastError());
  prof_mark(h, 5, st);
  h->cur_ev = nullptr;
  h->last_rows = T * h->K;
  h->last_dense = false;
  h->last_xperm_padded = false;
}

// ---------------------------------------------------------------------------------------
// Dense decode. At T <= kDenseMaxT tokens an M=128 GEMM tile holds every token, so running each
// expert on all T tokens costs no extra tensor work while the weights stream from HBM anyway;
// what it buys is independence from routing: GEMM1 (the longest stage) starts at once and the
// router + plan run beside it on a high-priority stream (launched first, so their CTAs hold SMs
// while GEMM1's persistent CTAs take the rest). GEMM2 waits for the routing decision: its row
// weight is the combine weight of (t, e) for routed pairs and 0 otherwise, and the combine reads
// the routed rows only. Every routed row sees exactly the sparse path's arithmetic, so outputs are
// bit-identical to it (tests/test_gpu_dense_decode.py). The plan and the dense row weights run in
// the router's last CTA, so nothing on the routing side has to find an SM while GEMM1's persistent
// CTAs hold them. CL_MOE_DENSE_DECODE=0 disables the dense path.
constexpr int kDenseMaxT = 128;

bool dense_ok(const cl_moe* h, int64_t T) {
  if (h->comm || h->cfg.ep_size > 1 || T < 1 || T > kDenseMaxT) return false;
  const char* e = std::getenv("CL_MOE_DENSE_DECODE");
  return !(e && e[0] == '0');
}

void ensure_dense(cl_moe* h) {
  if (h->xd) return;
  const uint64_t rows = static_cast<uint64_t>(h->N) * kDenseMaxT;
  h->xd = dalloc<__nv_bfloat16>(rows * h->d);
  h->actd = dalloc<__nv_bfloat16>(rows * h->f);
  h->yd = dalloc<__nv_bfloat16>(rows * h->d);
  h->rwd = dalloc<float>(rows);
  h->invd = dalloc<int32_t>((size_t)kDenseMaxT * h->K);
  h->offd = dalloc<int32_t>(h->N + 1);
  for (int v = 0; v < 2; ++v) {
    h->mA1d[v] = make_map(h->xd, false, h->d, rows, 128);
    h->mA2d[v] = make_map(h->actd, false, h->f, rows, 128);
    h->mA1dq[v] = make_map(h->xd, true, h->d, rows, 128);
    h->mA2dq[v] = make_map(h->actd, true, h->f, rows, 128);
  }
  int lo = 0, hi = 0;
  CK(cudaDeviceGetStreamPriorityRange(&lo, &hi));
  CK(cudaStreamCreateWithPriority(&h->s_route, cudaStreamNonBlocking, hi));
  CK(cudaEventCreateWithFlags(&h->ev_fork, cudaEventDisableTiming));
  CK(cudaEventCreateWithFlags(&h->ev_join, cudaEventDisableTiming));
  h->route_ctr = dalloc<int>(1);
  CK(cudaMemset(h->route_ctr, 0, sizeof(int)));
}

// route_tokens + moe_forward of the single-GPU layer: dense decode when eligible, else the
// sparse path (router, plan, dispatch, grouped GEMMs, combine).
// xr (nullable): the router's input when it differs from the GEMM operand x — the caller's fp32
// tensor (xr_f32), routed on its own values while the experts take its bf16 rounding.
void run_forward(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st,
                 const void* xr = nullptr, bool xr_f32 = false) {
  if (!xr) xr = x;
  if (!dense_ok(h, T)) {
    run_router(h, xr, T, st, true, false, xr_f32);
    run_experts(h, x, T, out, out_f32, st);
    return;
  }
  ensure_dense(h);
  const int N = static_cast<int>(h->N), K = static_cast<int>(h->K);
  const bool fp8 = h->precision == CL_MOE_FP8_E4M3;
  prof_begin(h, st, 2);
  CK(cudaEventRecord(h->ev_fork, st));
  CK(cudaStreamWaitEvent(h->s_route, h->ev_fork, 0));
  if (!run_router(h, xr, T, h->s_route, false, true, xr_f32)) {  // plan + row weights not fused (other variant)
    dense_weights_kernel<<<(int)((N * T + 255) / 256), 256, 0, h->s_route>>>(h->rb.topk_idx, h->rb.combine_w, (int)T,
                                                                             N, K, h->rwd, h->invd);
    CK(cudaGetLastError());
    prof_mark(h, 1, h->s_route);
  }
  CK(cudaEventRecord(h->ev_join, h->s_route));
  const int rb8 = static_cast<int>((N * T + 7) / 8);
  const dim3 blocks(rb8, std::max(1, std::min(8, (8 * h->num_sms + rb8 - 1) / rb8)));  // ~8 CTAs per SM
  if (fp8)
    dense_dispatch_kernel<true><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N,
                                                        h->xd, h->sx_in, h->offd);
  else
    dense_dispatch_kernel<false><<<blocks, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N,
                                                         h->xd, nullptr, h->offd);
  CK(cudaGetLastError());
  prof_mark(h, 2, st);
  run_gemms(h, h->offd, h->actd, h->yd, h->rwd, h->mA1d, h->mA2d, h->mA1dq, h->mA2dq, st, nullptr, nullptr, h->ev_join);
  prof_mark(h, 4, st);
  if (out_f32)
    launch_combine<float>(h->yd, h->invd, (int)T, (int)h->d, K, static_cast<float*>(out), h->rb.finite_flag, st);
  else
    launch_combine<__nv_bfloat16>(h->yd, h->invd, (int)T, (int)h->d, K, static_cast<__nv_bfloat16*>(out),
                                  h->rb.finite_flag, st);
  CK(cudaGetLastError());
  prof_mark(h, 5, st);
  h->cur_ev = nullptr;
  h->last_rows = N * T;  // dense layout: row e*T + t = token t for expert e
  h->last_dense = true;
  h->last_xperm_padded = false;
}

void export_decision(cl_moe* h, int64_t T, const cl_moe_decision* o, cudaStream_t st) {
  if (!o) return;
  const int64_t N = h->N, K = h->K;
  if (o->logits) CK(cudaMemcpyAsync(o->logits, h->rb.logits, sizeof(float) * T * N, cudaMemcpyDeviceToDevice, st));
  if (o->probs) CK(cudaMemcpyAsync(o->probs, h->rb.probs, sizeof(float) * T * N, cudaMemcpyDeviceToDevice, st));
  if (o->topk_idx) CK(cudaMemcpyAsync(o->topk_idx, h->rb.topk_idx, sizeof(int32_t) * T * K, cudaMemcpyDeviceToDevice, st));
  if (o->combine_weights)
    CK(cudaMemcpyAsync(o->combine_weights, h->rb.combine_w, sizeof(float) * T * K, cudaMemcpyDeviceToDevice, st));
  if (o->counts) {
    i32_to_i64_kernel<<<(int)((N + 127) / 128), 128, 0, st>>>(h->rb.counts, (int)N, o->counts);
    CK(cudaGetLastError());
  }
  if (o->agg_prob) CK(cudaMemcpyAsync(o->agg_prob, h->rb.agg_prob, sizeof(float) * N, cudaMemcpyDeviceToDevice, st));
  if (o->aux_loss) CK(cudaMemcpyAsync(o->aux_loss, h->rb.losses, sizeof(float), cudaMemcpyDeviceToDevice, st));
  if (o->z_loss) CK(cudaMemcpyAsync(o->z_loss, h->rb.losses + 1, sizeof(float), cudaMemcpyDeviceToDevice, st));
}

void ensure_fp8_storage(cl_moe* h) {
  if (!h->xq8) {  // router under the FP8 scheme
    h->sxr_dev = dalloc<float>(1);
    h->wrq = dalloc<float>(h->d * h->N);
    h->wsr = dalloc<float>(h->N);
    h->wr64q = dalloc<double>(router_w64_size((int)h->d, (int)h->N));
    h->xq8 = dalloc<uint8_t>(h->cap * h->d);
  }
  if (h->win8) return;
  h->win8 = dalloc<uint8_t>((size_t)h->n_local * 2 * h->f * h->d);
  h->wout8 = dalloc<uint8_t>((size_t)h->n_local * h->d * h->f);
  h->ws_in = dalloc<float>((size_t)h->n_local * 2 * h->f);
  h->ws_out = dalloc<float>((size_t)h->n_local * h->d);
  build_maps(h, true);
}

}  // namespace
