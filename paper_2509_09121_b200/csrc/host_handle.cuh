// Handle state (struct cl_moe), error mapping, TMA descriptors, device allocation, stage timing.
// Host side of libcompass_moe.so, included once, in order, by capi.cu (a single translation
// unit; the helpers live in an anonymous namespace).
#pragma once

namespace {

struct ConfigErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct RunErr : std::runtime_error {
  using std::runtime_error::runtime_error;
};

std::string fmt(const char* f, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, f);
  vsnprintf(buf, sizeof(buf), f, ap);
  va_end(ap);
  return buf;
}

#define CK(x)                                                                                \
  do {                                                                                       \
    cudaError_t e_ = (x);                                                                    \
    if (e_ != cudaSuccess) throw RunErr(fmt("%s failed: %s", #x, cudaGetErrorString(e_)));  \
  } while (0)

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                              const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (q != cudaDriverEntryPointSuccess || !p) throw RunErr("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

// 2D row-major tensor [rows][inner] with a 128-byte-swizzled box of [box_rows][128 bytes].
CUtensorMap make_map(const void* base, bool fp8, uint64_t inner, uint64_t rows, uint32_t box_rows) {
  CUtensorMap m;
  const uint32_t esz = fp8 ? 1 : 2;
  cuuint64_t dims[2] = {inner, rows};
  cuuint64_t strides[1] = {inner * esz};
  cuuint32_t box[2] = {128u / esz, box_rows};
  cuuint32_t es[2] = {1, 1};
  CUresult r = encode_fn()(&m, fp8 ? CU_TENSOR_MAP_DATA_TYPE_UINT8 : CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                           const_cast<void*>(base), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                           CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                           CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw RunErr(fmt("cuTensorMapEncodeTiled failed (%d)", (int)r));
  return m;
}

template <typename T>
T* dalloc(size_t n) {
  void* p = nullptr;
  if (n == 0) n = 1;
  CK(cudaMalloc(&p, n * sizeof(T)));
  return static_cast<T*>(p);
}

int grid_for(int64_t n, int threads = 256) {
  return static_cast<int>(std::min<int64_t>((n + threads - 1) / threads, 148 * 32));
}

}  // namespace

struct cl_moe {
  cl_moe_config cfg{};
  int64_t d = 0, N = 0, K = 0, f = 0, cap = 0;
  int n_local = 0, e0 = 0;
  int gemm_ctas = 2;
  bool gemm_auto = true;               // pick cta_group per call from the rows per expert
  int num_sms = 148;
  int precision = CL_MOE_BF16;
  std::string last_error;

  // weights
  float* wr = nullptr;                 // [d][N] fp32
  double* wr64 = nullptr;              // [d][N4] fp64 copy streamed by the router, then [N4][d]
  __nv_bfloat16* win = nullptr;        // [n_local][2f][d] packed
  __nv_bfloat16* wout = nullptr;       // [n_local][d][f] packed
  uint8_t* win8 = nullptr;             // e4m3 copies
  uint8_t* wout8 = nullptr;
  float* ws_in = nullptr;              // [n_local][2f]
  float* ws_out = nullptr;             // [n_local][d]
  float* sx_in = nullptr;              // [n_local]
  float* sx_in_all = nullptr;          // [N] GEMM1-input scales of every expert (EP: the source
                                       //     quantizes a row with its owner's scale)
  float* calib_all = nullptr;          // [N] EP calibration: source-side max |x| per global expert
  float* sx_mid = nullptr;             // [n_local]
  float* calib = nullptr;              // [2][n_local] running maxima
  float* calib_ch = nullptr;           // [d] per-channel max |hidden| over calibration tokens
  long long* calib_counts = nullptr;   // [N] routing counts over calibration tokens
  float* smooth = nullptr;             // [d] scratch for fold_smoothing
  bool fp8_ready = false;
  // router under the FP8 scheme: qdq'd W_r and the per-tensor activation scale
  int router_fp8 = 1;                  // 1: router GEMM through fp8_qdq in FP8 mode; 0: fp32 gating
  float sxr = 0.0f;                    // router activation scale (host copy; 0 = from calibration)
  bool sxr_explicit = false;
  float* sxr_dev = nullptr;            // [1]
  float* wrq = nullptr;                // [d][N] qdq(W_r) fp32
  float* wsr = nullptr;                // [N] router weight scales (per expert column)
  double* wr64q = nullptr;             // widened qdq(W_r), same layout as wr64
  uint8_t* xq8 = nullptr;              // [cap][d] E4M3 codes of x / s_x (router operand, FP8 scheme)
  // certified large-batch router (router_cert.cuh): fp32 padded W_r copies [d][N8] + ||w_i|| bounds
  // of the plain and of the FP8-scheme router, rebuilt when the weights change (version counters)
  float* cert_w8 = nullptr;
  float* cert_wn = nullptr;
  float* cert_w8q = nullptr;
  float* cert_wnq = nullptr;
  int* cert_count = nullptr;           // [1] tokens recomputed exactly by the last certified call
  int64_t wr_ver = 0, wrq_ver = 0, cert_ver = -1, cert_verq = -1;
  bool need_exact = false;             // the current call exports the decision (or trains): exact K1 only
  int64_t cert_calls = 0;
  // QuantScheme bookkeeping (scheme file)
  std::vector<float> smooth_applied;   // product of the folded smoothing vectors (empty: none)
  double alpha_smooth = NAN;           // alpha of the last compute_smoothing
  int64_t tau = -1;                    // tau of the last balance_calibration

  // workspaces
  RouteBufs rb{};
  int n_tiles_cap = 0;
  void* xperm = nullptr;               // [cap*K][d] (bf16 or e4m3)
  void* act = nullptr;                 // [cap*K][f]
  __nv_bfloat16* y = nullptr;          // [cap*K][d]
  int32_t* perm = nullptr;
  int32_t* inv = nullptr;
  float* row_w = nullptr;
  // host-buffer entry points: two pipeline slots so the H2D of call i+1 and the D2H of call i-1
  // overlap the layer compute of call i (separate copy streams, event-ordered).
  struct HostSlot {
    void* x = nullptr;       // bf16 [cap][d]
    float* xf = nullptr;     // fp32 staging [cap][d] (fp32 io only)
    void* out = nullptr;     // [cap][d] bf16 or fp32
    cudaEvent_t h2d = nullptr, done = nullptr, d2h = nullptr;
    bool used = false;
  } slot[2];
  int next_slot = 0;
  void* io_out = nullptr;              // calibration output scratch
  __nv_bfloat16* x16 = nullptr;        // [cap][d] bf16 GEMM operand of a device fp32 forward
  cudaStream_t own_stream = nullptr;   // compute stream of the host-buffer path
  // captured forwards (cl_moe_forward_graph), keyed by buffers, T and precision
  struct GraphEntry {
    const void* x;
    void* out;
    int64_t T;
    int precision;
    cudaGraphExec_t exec;
  };
  std::vector<GraphEntry> graphs;
  cudaStream_t cap_stream = nullptr;
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  int64_t last_rows = 0;
  bool last_dense = false;  // the last forward took the dense-decode path (stage view = dense buffers)
  int tpc_cur = 32;                    // router tile (tokens) of the last routing call
  bool dmma_ok = false;                // the fp64 tensor-core router passed its device check (init)
  int last_router_variant = -1;        // K1 kernel of the last routing call (cl_moe_router_variant)
  int64_t last_tokens = 0;             // T of the current call

  // per-stage CUDA-event timing (cl_moe_profile): one event set per profiled call
  bool prof = false;
  std::vector<std::vector<cudaEvent_t>> prof_sets;
  std::vector<int> prof_kind;          // 0 forward (6 stages), 1 backward (7 stages)
  size_t prof_used = 0;
  std::vector<cudaEvent_t>* cur_ev = nullptr;
  uint64_t nvtx_id = 0;                // open NVTX stage range (nvtxRangeStartA)
  int nvtx_kind = 0;

  // expert parallelism (ep.cuh)
  NcclApi::Comm comm = nullptr;
  std::string ep_abort_reason;          // set when a failed / stalled exchange aborted the communicator
  int64_t recv_cap = 0;                 // receive-buffer rows (worst case: every rank's every slot)
  __nv_bfloat16* x_recv = nullptr;      // [recv_cap][d]
  __nv_bfloat16* act_recv = nullptr;    // [recv_cap][f]
  __nv_bfloat16* y_recv = nullptr;      // [recv_cap][d]
  int32_t* ep_counts_dev = nullptr;     // [R][N] all-gathered counts
  int32_t* ep_off_dev = nullptr;        // [NL+1] local expert offsets in the receive buffer
  int32_t* ep_counts_host = nullptr;    // pinned mirrors
  int32_t* ep_off_host = nullptr;
  std::vector<int64_t> ep_C, ep_piece, ep_myoff;  // exchange layout of the last EP forward
  __nv_bfloat16* dYsrc = nullptr;       // EP training: source-order dY [cap*K][d]
  __nv_bfloat16* dXsrc = nullptr;       // EP training: source-order dX [cap*K][d]
  CUtensorMap mA1e[2], mA2e[2];
  CUtensorMap mA1eq[2], mA2eq[2];       // e4m3 views of x_recv / act_recv
  bool maps_eq = false;
  // peer-memory (NVLink) transport (ep.cuh): 0 = NCCL send/recv, 1 = direct peer stores
  int ep_transport = 0;
  char** peer_x_dev = nullptr;          // [R] every rank's x_recv, as mapped in this process
  char** peer_y_dev = nullptr;          // [R] every rank's y (source-order return buffer)
  float** peer_w_dev = nullptr;         // [R] every rank's w_recv
  float* w_recv = nullptr;              // [recv_cap] combine weight of each received row
  void** expert_dst = nullptr;          // [N] dispatch destinations of this rank's pieces
  float** expert_dst_w = nullptr;       // [N] ... of their combine weights
  void** row_ptr = nullptr;             // [recv_cap] return address of every received row
  char** peer_dy_dev = nullptr;         // [R] every rank's dYbuf (training: dY rows to the owners)
  char** peer_dx_dev = nullptr;         // [R] every rank's dXsrc (training: dX rows back)
  // dispatch overlapped with GEMM1 (CL_MOE_EP_OVERLAP=1): arrival counters of this rank's experts
  // (mapped by the peers), the running targets, every rank's counter array, per global expert the
  // owner's counter
  uint32_t* arrive = nullptr;           // [n_local]
  uint32_t* arrive_tgt = nullptr;       // [n_local]
  char** peer_a_dev = nullptr;          // [R]
  uint32_t** expert_arrive = nullptr;   // [N]
  void** expert_dst_dy = nullptr;       // [N] this rank's dY pieces in the owners' dYbuf
  void** row_ptr_dx = nullptr;          // [recv_cap] source address of every received row's dX
  bool ep_group = false;                // member of a single-process EP group (cl_moe_ep_group_*)
  float* bar_buf = nullptr;             // [1] payload of the exchange barriers
  std::vector<void*> ipc_opened;        // peers' buffers mapped through CUDA IPC

  // training (expert-FFN backward)
  bool train_ready = false;
  int64_t train_T = 0;                  // T of the last cl_moe_forward_train
  const void* cur_x = nullptr;          // hidden of the last cl_moe_forward_train (caller-owned)
  int64_t rp_cap = 0;                   // padded-row capacity of the transposes
  __nv_bfloat16* win_ref = nullptr;     // [NL][d][2f] reference layout (dgrad-2 B operand)
  __nv_bfloat16* wout_ref = nullptr;    // [NL][f][d]  reference layout (dgrad-1 B operand)
  __nv_bfloat16* Hbuf = nullptr;        // [cap*K][2f] pre-activations [G | U]
  __nv_bfloat16* dYbuf = nullptr;       // [cap*K][d]
  __nv_bfloat16* dXbuf = nullptr;       // [cap*K][d]
  // weight-gradient operands in the padded row layout [rp_cap][C] (expert e's rows from poff[e],
  // zero padding rows): X, A (= SwiGLU output), dY, dH
  __nv_bfloat16 *XT = nullptr, *AT = nullptr, *dYT = nullptr, *dHT = nullptr;
  int32_t* poff = nullptr;              // [NL+1]
  int* tile_counter = nullptr;          // grouped-GEMM dynamic tile scheduler
  float* rdz = nullptr;                 // router backward: dz [cap][N] fp32
  float* rpart = nullptr;               // dW_r partials [chunks][d][N]
  float* dcw_scratch = nullptr;         // d(combine weights) [cap][K] when the caller does not want them
  int32_t* kb_off = nullptr;            // [NL+1]
  CUtensorMap mAdg1[2], mBdg1[2], mBdg2[2], mAwo[2], mBwo[2], mAwi[2], mBwi[2];
  CUtensorMap mAdg2T[2];  // dgrad-2's A = dH in the padded row layout (GemmArgs::a_poff)
  CUtensorMap mA1T[2], mAdg1T[2];  // single-GPU training: GEMM1's A = X, dgrad-1's A = dY, padded
  CUtensorMap mA2T[2];             // single-GPU training: GEMM2's A = SwiGLU output, padded
  bool last_xperm_padded = false;  // the last call (single-GPU forward_train) left x_perm padded
  bool mAdg1_ready = false;        // dgrad-1's receive-layout dY map exists (expert parallel)

  CUtensorMap mA1[2], mB1[2], mA2[2], mB2[2];      // [variant: 0 = 1-CTA, 1 = 2-CTA]
  CUtensorMap mA1q[2], mB1q[2], mA2q[2], mB2q[2];  // e4m3 maps
  CUtensorMap mB1m, mB2m, mB1qm, mB2qm;            // 64-row B boxes (multicast clusters, kCM == 2)
  bool maps_q = false;

  // dense decode (host_forward.cuh run_forward): every expert runs all T <= kDenseMaxT tokens so
  // the expert GEMMs start before routing is known; the router runs beside them on s_route
  __nv_bfloat16 *xd = nullptr, *actd = nullptr, *yd = nullptr;  // [N * kDenseMaxT] rows
  float* rwd = nullptr;                                          // [N * kDenseMaxT] row weights (0 = unrouted)
  int32_t *invd = nullptr, *offd = nullptr;                      // [kDenseMaxT * K], [N + 1]
  CUtensorMap mA1d[2], mA2d[2], mA1dq[2], mA2dq[2];
  cudaStream_t s_route = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  int g1_grid = 0;  // > 0: GEMM1 grid limit
  int* route_ctr = nullptr;  // router_ws_kernel tail counter (dense decode)

  ~cl_moe() {
    void* ptrs[] = {sx_in_all, calib_all, calib_counts, calib_ch, smooth, wr64,   wr,     win,     wout,    win8,      wout8,        ws_in,        ws_out,
                    sx_in,  sx_mid,  calib,   xperm,     act,          y,            perm,
                    inv,    row_w,   slot[0].x, slot[0].xf, slot[0].out, slot[1].x, slot[1].xf, slot[1].out,
                    io_out, rb.logits,    rb.probs,
                    rb.topk_idx, rb.combine_w, rb.local_rank, rb.tile_cnt, rb.tile_psum, rb.tile_lse2,
                    rb.counts, rb.offsets, rb.agg_prob, rb.losses, rb.finite_flag};
    for (void* p : ptrs)
      if (p) cudaFree(p);
    for (void* p : {(void*)x_recv, (void*)act_recv, (void*)y_recv, (void*)ep_counts_dev, (void*)ep_off_dev,
                    (void*)win_ref, (void*)wout_ref, (void*)Hbuf, (void*)dYbuf, (void*)dXbuf, (void*)XT,
                    (void*)AT, (void*)dYT, (void*)dHT, (void*)poff, (void*)kb_off, (void*)rdz, (void*)rpart,
                    (void*)dcw_scratch, (void*)dYsrc, (void*)dXsrc, (void*)tile_counter, (void*)peer_x_dev,
                    (void*)peer_y_dev, (void*)peer_w_dev, (void*)w_recv, (void*)expert_dst, (void*)expert_dst_w,
                    (void*)row_ptr, (void*)bar_buf, (void*)peer_dy_dev, (void*)peer_dx_dev, (void*)expert_dst_dy,
                    (void*)row_ptr_dx, (void*)arrive, (void*)arrive_tgt, (void*)peer_a_dev, (void*)expert_arrive, (void*)xd, (void*)actd, (void*)yd, (void*)rwd, (void*)invd, (void*)offd, (void*)route_ctr, (void*)x16, (void*)sxr_dev, (void*)wrq,
                    (void*)wsr, (void*)wr64q, (void*)xq8, (void*)cert_w8, (void*)cert_wn,
                    (void*)cert_w8q, (void*)cert_wnq, (void*)cert_count})
      if (p) cudaFree(p);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (ep_counts_host) cudaFreeHost(ep_counts_host);
    if (ep_off_host) cudaFreeHost(ep_off_host);
    if (comm) NcclApi::get().CommDestroy(comm);
    for (auto& g : graphs) cudaGraphExecDestroy(g.exec);
    if (cap_stream) cudaStreamDestroy(cap_stream);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    if (s_route) cudaStreamDestroy(s_route);
    if (ev_fork) cudaEventDestroy(ev_fork);
    if (ev_join) cudaEventDestroy(ev_join);
    for (auto& sl : slot)
      for (cudaEvent_t e : {sl.h2d, sl.done, sl.d2h})
        if (e) cudaEventDestroy(e);
    for (auto& v : prof_sets)
      for (auto e : v) cudaEventDestroy(e);
  }
};

namespace {

// The call exports the routing decision (or trains on it): K1 must produce the reference's exact
// logits / probabilities, not only a certified decision (router_cert.cuh).
struct ExactRoute {
  cl_moe* h;
  bool prev;
  ExactRoute(cl_moe* hh, bool on) : h(hh), prev(hh ? hh->need_exact : false) {
    if (h) h->need_exact = prev || on;
  }
  ~ExactRoute() {
    if (h) h->need_exact = prev;
  }
};

template <typename Fn>
cl_status guarded(cl_moe* h, Fn fn) {
  if (!h) return CL_ERR_CONFIG;
  try {
    h->last_error.clear();
    fn();
    return CL_OK;
  } catch (const ConfigErr& e) {
    h->last_error = e.what();
    return CL_ERR_CONFIG;
  } catch (const std::exception& e) {
    h->last_error = e.what();
    return CL_ERR_RUN;
  }
}

constexpr int kStages = 6;     // forward: router, plan, dispatch, gemm1, gemm2, combine
constexpr int kBwdStages = 7;  // backward: combine-bwd, dgrad1, dgrad2, dispatch-bwd, transposes, wgrad-out, wgrad-in

// NVTX: one range per stage of every call (host timeline of the launches; cheap without a tool),
// named like the profile stages so an Nsight timeline reads like profile_read.
const char* nvtx_stage_name(int kind, int stage) {
  static const char* fwd[kStages] = {"moe.router", "moe.plan", "moe.dispatch", "moe.gemm1_swiglu", "moe.gemm2_weight",
                                     "moe.combine"};
  static const char* bwd[kBwdStages] = {"moe.bwd.combine", "moe.bwd.dgrad1_swiglu", "moe.bwd.dgrad2",
                                        "moe.bwd.dispatch", "moe.bwd.transposes", "moe.bwd.wgrad_out",
                                        "moe.bwd.wgrad_in"};
  return kind == 1 ? bwd[stage] : fwd[stage];
}
void nvtx_next(cl_moe* h, int stage) {  // ends the open range; opens `stage`'s (if any)
  if (h->nvtx_id) nvtxRangeEnd(h->nvtx_id);
  h->nvtx_id = 0;
  if (stage >= 0 && stage < (h->nvtx_kind == 1 ? kBwdStages : kStages))
    h->nvtx_id = nvtxRangeStartA(nvtx_stage_name(h->nvtx_kind, stage));
}

void prof_begin(cl_moe* h, cudaStream_t st, int kind = 0) {
  h->cur_ev = nullptr;
  h->nvtx_kind = kind;
  nvtx_next(h, 0);
  if (!h->prof) return;
  if (h->prof_used == h->prof_sets.size()) {
    std::vector<cudaEvent_t> v(kBwdStages + 1);
    for (auto& e : v) CK(cudaEventCreate(&e));
    h->prof_sets.push_back(v);
    h->prof_kind.push_back(0);
  }
  h->prof_kind[h->prof_used] = kind;
  h->cur_ev = &h->prof_sets[h->prof_used++];
  CK(cudaEventRecord((*h->cur_ev)[0], st));
}
void prof_mark(cl_moe* h, int stage, cudaStream_t st) {
  nvtx_next(h, stage + 1);
  if (h->cur_ev) CK(cudaEventRecord((*h->cur_ev)[stage + 1], st));
}

void validate(const cl_moe_config* c) {
  if (!c) throw ConfigErr("config is null");
  if (c->d_model <= 0 || c->d_model % 256) throw ConfigErr(fmt("d_model=%lld must be a positive multiple of 256", (long long)c->d_model));
  if (c->d_ff <= 0 || c->d_ff % 128) throw ConfigErr(fmt("d_ff=%lld must be a positive multiple of 128", (long long)c->d_ff));
  if (c->n_experts < 1 || c->n_experts > 128) throw ConfigErr(fmt("n_experts=%lld outside [1, 128]", (long long)c->n_experts));
  if (c->top_k < 1 || c->top_k > c->n_experts || c->top_k > 8)
    throw ConfigErr(fmt("top_k=%lld outside [1, min(N, 8)]", (long long)c->top_k));
  if (c->max_tokens < 1 || c->max_tokens * c->top_k > (int64_t(1) << 30)) throw ConfigErr("max_tokens out of range");
  const int ep = c->ep_size <= 0 ? 1 : c->ep_size;
  if (c->n_experts % ep) throw ConfigErr("n_experts must be divisible by ep_size");
  if (c->ep_rank < 0 || c->ep_rank >= ep) throw ConfigErr("ep_rank out of range");
  if (c->max_tokens * c->top_k * ep > (int64_t(1) << 30))  // receive rows are int32-indexed
    throw ConfigErr("max_tokens x top_k x ep_size out of range");
  if (c->gemm_ctas < 0 || c->gemm_ctas > 2) throw ConfigErr("gemm_ctas must be 0, 1 or 2");
}

void build_maps(cl_moe* h, bool fp8) {
  const uint64_t rows = static_cast<uint64_t>(h->cap * h->K);
  for (int v = 0; v < 2; ++v) {
    const uint32_t brow = v == 0 ? 256 : 128;
    if (!fp8) {
      h->mA1[v] = make_map(h->xperm, false, h->d, rows, 128);
      h->mB1[v] = make_map(h->win, false, h->d, (uint64_t)h->n_local * 2 * h->f, brow);
      h->mA2[v] = make_map(h->act, false, h->f, rows, 128);
      h->mB2[v] = make_map(h->wout, false, h->f, (uint64_t)h->n_local * h->d, brow);
    } else {
      h->mA1q[v] = make_map(h->xperm, true, h->d, rows, 128);
      h->mB1q[v] = make_map(h->win8, true, h->d, (uint64_t)h->n_local * 2 * h->f, brow);
      h->mA2q[v] = make_map(h->act, true, h->f, rows, 128);
      h->mB2q[v] = make_map(h->wout8, true, h->f, (uint64_t)h->n_local * h->d, brow);
    }
  }
  if (!fp8) {
    h->mB1m = make_map(h->win, false, h->d, (uint64_t)h->n_local * 2 * h->f, 64);
    h->mB2m = make_map(h->wout, false, h->f, (uint64_t)h->n_local * h->d, 64);
  } else {
    h->mB1qm = make_map(h->win8, true, h->d, (uint64_t)h->n_local * 2 * h->f, 64);
    h->mB2qm = make_map(h->wout8, true, h->f, (uint64_t)h->n_local * h->d, 64);
  }
}

void init_handle(cl_moe* h, const cl_moe_config* c) {
  validate(c);
  h->cfg = *c;
  h->d = c->d_model;
  h->N = c->n_experts;
  h->K = c->top_k;
  h->f = c->d_ff;
  h->cap = c->max_tokens;
  const int ep = c->ep_size <= 0 ? 1 : c->ep_size;
  h->n_local = static_cast<int>(h->N / ep);
  h->e0 = c->ep_rank * h->n_local;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) throw RunErr("no CUDA device available (the MoE path has no CPU fallback)");
  CK(cudaSetDevice(c->device));
  cudaDeviceProp prop;
  CK(cudaGetDeviceProperties(&prop, c->device));
  if (prop.major != 10) throw RunErr(fmt("device %d is sm_%d%d; this library is built for sm_100a only", c->device, prop.major, prop.minor));
  h->num_sms = prop.multiProcessorCount;
  h->gemm_auto = c->gemm_ctas == 0;
  h->gemm_ctas = c->gemm_ctas == 0 ? 2 : c->gemm_ctas;
  CK(cudaStreamCreateWithFlags(&h->own_stream, cudaStreamNonBlocking));
  h->tile_counter = dalloc<int>(1);  // (allocated up front: no cudaMalloc inside a graph capture)
  CK(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
  for (auto& sl : h->slot) {
    CK(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl.d2h, cudaEventDisableTiming));
  }

  const int64_t rows = h->cap * h->K;
  const int tpc = std::min({router_tokens_per_cta(static_cast<int>(h->N), 32),
                            RouterBigSmem(static_cast<int>(h->N), 32, 3, 2).tpc,
                            RouterLatSmem<3, 64>(static_cast<int>(h->N)).tpc,
                            std::max(1, RouterWsSmem(static_cast<int>(h->N), 32).tpc)});  // smallest tile of any variant
  h->n_tiles_cap = static_cast<int>((h->cap + tpc - 1) / tpc);
  RouteBufs& rb = h->rb;
  rb.logits = dalloc<float>(h->cap * h->N);
  rb.probs = dalloc<float>(h->cap * h->N);
  rb.topk_idx = dalloc<int32_t>(rows);
  rb.combine_w = dalloc<float>(rows);
  rb.local_rank = dalloc<int32_t>(rows);
  rb.tile_cnt = dalloc<int32_t>((size_t)h->n_tiles_cap * h->N);
  rb.tile_psum = dalloc<double>((size_t)h->n_tiles_cap * h->N);
  rb.tile_lse2 = dalloc<double>(h->n_tiles_cap);
  rb.counts = dalloc<int32_t>(h->N);
  rb.offsets = dalloc<int32_t>(h->N + 1);
  rb.agg_prob = dalloc<float>(h->N);
  rb.losses = dalloc<float>(2);
  rb.finite_flag = dalloc<int32_t>(1);
  CK(cudaMemset(rb.finite_flag, 0, sizeof(int32_t)));
  CK(cudaMemset(rb.offsets, 0, sizeof(int32_t) * (h->N + 1)));

  h->xperm = dalloc<__nv_bfloat16>(rows * h->d);
  h->act = dalloc<__nv_bfloat16>(rows * h->f);
  h->y = dalloc<__nv_bfloat16>(rows * h->d);
  h->perm = dalloc<int32_t>(rows);
  h->inv = dalloc<int32_t>(rows);
  h->row_w = dalloc<float>(rows);

  h->wr = dalloc<float>(h->d * h->N);
  // [d][N4], the router_ws layout, the router_dmma fragment layout (widen_router_kernel)
  h->wr64 = dalloc<double>(router_w64_size((int)h->d, (int)h->N));
  for (const void* fn : {(const void*)router_dmma_kernel<1, 2>, (const void*)router_dmma_kernel<2, 2>,
                         (const void*)router_dmma_kernel<4, 2>, (const void*)router_dmma_kernel<1, 4>,
                         (const void*)router_dmma_kernel<2, 4>, (const void*)router_dmma_kernel<4, 4>,
                         (const void*)router_dmma_kernel<1, 2, float>, (const void*)router_dmma_kernel<2, 2, float>,
                         (const void*)router_dmma_kernel<4, 2, float>, (const void*)router_dmma_kernel<1, 4, float>,
                         (const void*)router_dmma_kernel<2, 4, float>, (const void*)router_dmma_kernel<4, 4, float>,
                         (const void*)router_dmma_kernel<1, 2, uint8_t>, (const void*)router_dmma_kernel<2, 2, uint8_t>,
                         (const void*)router_dmma_kernel<4, 2, uint8_t>, (const void*)router_dmma_kernel<1, 4, uint8_t>,
                         (const void*)router_dmma_kernel<2, 4, uint8_t>, (const void*)router_dmma_kernel<4, 4, uint8_t>})
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  {  // the DMMA router is used only if the instruction accumulates as the sequential chain here
    unsigned long long* bad = dalloc<unsigned long long>(1);
    CK(cudaMemset(bad, 0, sizeof(unsigned long long)));
    dmma_selftest_kernel<<<h->num_sms, 256>>>(64, bad);
    CK(cudaGetLastError());
    unsigned long long nb = 1;
    CK(cudaMemcpy(&nb, bad, sizeof(nb), cudaMemcpyDeviceToHost));
    CK(cudaFree(bad));
    const char* e = std::getenv("CL_MOE_ROUTER_DMMA");  // "0": keep the DFMA variants (A/B)
    h->dmma_ok = nb == 0 && !(e && e[0] == '0');
  }
  CK(cudaFuncSetAttribute(router_kernel<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_kernel<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_lat_kernel<3, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_lat_kernel<3, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_lat_kernel<3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  // fp32-input instantiations (routing on the caller's fp32 tensor)
  CK(cudaFuncSetAttribute(router_kernel<128, 3, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_kernel<32, 8, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3, 4, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3, 2, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<32, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<64, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<128, float>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  for (const void* fn : {(const void*)router_cert_kernel<__nv_bfloat16>, (const void*)router_cert_kernel<float>,
                         (const void*)router_cert_kernel<uint8_t>})
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  // E4M3-code instantiations (the router under the FP8 scheme)
  CK(cudaFuncSetAttribute(router_kernel<128, 3, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_kernel<32, 8, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3, 4, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3, 2, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<32, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<64, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_ws_kernel<128, uint8_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  h->win = dalloc<__nv_bfloat16>((size_t)h->n_local * 2 * h->f * h->d);
  h->wout = dalloc<__nv_bfloat16>((size_t)h->n_local * h->d * h->f);
  h->sx_in = dalloc<float>(h->n_local);
  h->sx_in_all = dalloc<float>(h->N);
  h->calib_all = dalloc<float>(h->N);
  CK(cudaMemset(h->calib_all, 0, sizeof(float) * h->N));
  h->sx_mid = dalloc<float>(h->n_local);
  h->calib = dalloc<float>(2 * h->n_local);
  CK(cudaMemset(h->calib, 0, sizeof(float) * 2 * h->n_local));
  h->calib_ch = dalloc<float>(h->d);
  CK(cudaMemset(h->calib_ch, 0, sizeof(float) * h->d));
  h->calib_counts = dalloc<long long>(h->N);
  CK(cudaMemset(h->calib_counts, 0, sizeof(long long) * h->N));
  h->smooth = dalloc<float>(h->d);

  using namespace cmoe;
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<1, EPI_SWIGLU, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<1, EPI_ROWSCALE, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<2, EPI_SWIGLU, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<2, EPI_ROWSCALE, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<1, EPI_SWIGLU_BWD, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<2, EPI_SWIGLU_BWD, false, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<1, EPI_WGRAD, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<2, EPI_WGRAD, false, false, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<1, EPI_SWIGLU, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<1, EPI_ROWSCALE, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<1>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<2, EPI_SWIGLU, true, true>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
  CK(cudaFuncSetAttribute(grouped_gemm_kernel<2, EPI_ROWSCALE, true, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
  // clusters of two CTA pairs sharing B by multicast (GemmArgs / kCM == 2)
  for (const void* fn : {(const void*)grouped_gemm_kernel<2, EPI_SWIGLU, false, false, false, 2>,
                         (const void*)grouped_gemm_kernel<2, EPI_ROWSCALE, false, false, false, 2>,
                         (const void*)grouped_gemm_kernel<2, EPI_SWIGLU, true, true, false, 2>,
                         (const void*)grouped_gemm_kernel<2, EPI_ROWSCALE, true, false, false, 2>}) {
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, GemmCfg<2>::kSmem));
    CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
  }
}

}  // namespace
