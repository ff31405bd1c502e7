// Host orchestration of the MoE layer behind the C ABI of include/compass_moe.h.
//
// Error convention follows the reference C API (proj/src/capi.cpp:44-68): configuration errors
// -> CL_ERR_CONFIG, anything else (CUDA error, non-finite output, invalid runtime input)
// -> CL_ERR_RUN, message kept on the handle. No CPU fallback exists: without a usable sm_100
// device every entry point fails with CL_ERR_RUN.
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <vector>

#include "compass_moe.h"
#include "grouped_gemm.cuh"
#include "moe_kernels.cuh"
#include "synth_pack.cuh"
#include "ep.cuh"
#include "bwd_kernels.cuh"
#include "ckpt.hpp"

using namespace cmoe;

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
  double* wr64 = nullptr;              // [d][N4] fp64 copy streamed by the router
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
  cudaStream_t own_stream = nullptr;   // compute stream of the host-buffer path
  cudaStream_t s_h2d = nullptr, s_d2h = nullptr;
  int64_t last_rows = 0;
  int tpc_cur = 32;                    // router tile (tokens) of the last routing call
  int64_t last_tokens = 0;             // T of the current call

  // per-stage CUDA-event timing (cl_moe_profile): one event set per profiled call
  bool prof = false;
  std::vector<std::vector<cudaEvent_t>> prof_sets;
  std::vector<int> prof_kind;          // 0 forward (6 stages), 1 backward (7 stages)
  size_t prof_used = 0;
  std::vector<cudaEvent_t>* cur_ev = nullptr;

  // expert parallelism (ep.cuh)
  NcclApi::Comm comm = nullptr;
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
  __nv_bfloat16* dHbuf = nullptr;       // [cap*K][2f]
  __nv_bfloat16* dXbuf = nullptr;       // [cap*K][d]
  __nv_bfloat16 *XT = nullptr, *AT = nullptr, *dYT = nullptr, *dHT = nullptr;  // [C][rp_cap]
  int32_t* poff = nullptr;              // [NL+1]
  int* tile_counter = nullptr;          // grouped-GEMM dynamic tile scheduler
  float* rdz = nullptr;                 // router backward: dz [cap][N] fp32
  float* rpart = nullptr;               // dW_r partials [chunks][d][N]
  float* dcw_scratch = nullptr;         // d(combine weights) [cap][K] when the caller does not want them
  int32_t* kb_off = nullptr;            // [NL+1]
  CUtensorMap mAdg1[2], mBdg1[2], mAdg2[2], mBdg2[2], mAwo[2], mBwo[2], mAwi[2], mBwi[2];

  CUtensorMap mA1[2], mB1[2], mA2[2], mB2[2];      // [variant: 0 = 1-CTA, 1 = 2-CTA]
  CUtensorMap mA1q[2], mB1q[2], mA2q[2], mB2q[2];  // e4m3 maps
  bool maps_q = false;

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
                    (void*)win_ref, (void*)wout_ref, (void*)Hbuf, (void*)dYbuf, (void*)dHbuf, (void*)dXbuf, (void*)XT,
                    (void*)AT, (void*)dYT, (void*)dHT, (void*)poff, (void*)kb_off, (void*)rdz, (void*)rpart,
                    (void*)dcw_scratch, (void*)dYsrc, (void*)dXsrc, (void*)tile_counter, (void*)peer_x_dev,
                    (void*)peer_y_dev, (void*)peer_w_dev, (void*)w_recv, (void*)expert_dst, (void*)expert_dst_w,
                    (void*)row_ptr, (void*)bar_buf, (void*)peer_dy_dev, (void*)peer_dx_dev, (void*)expert_dst_dy,
                    (void*)row_ptr_dx})
      if (p) cudaFree(p);
    for (void* p : ipc_opened) cudaIpcCloseMemHandle(p);
    if (ep_counts_host) cudaFreeHost(ep_counts_host);
    if (ep_off_host) cudaFreeHost(ep_off_host);
    if (comm) NcclApi::get().CommDestroy(comm);
    if (own_stream) cudaStreamDestroy(own_stream);
    if (s_h2d) cudaStreamDestroy(s_h2d);
    if (s_d2h) cudaStreamDestroy(s_d2h);
    for (auto& sl : slot)
      for (cudaEvent_t e : {sl.h2d, sl.done, sl.d2h})
        if (e) cudaEventDestroy(e);
    for (auto& v : prof_sets)
      for (auto e : v) cudaEventDestroy(e);
  }
};

namespace {

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

void prof_begin(cl_moe* h, cudaStream_t st, int kind = 0) {
  h->cur_ev = nullptr;
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
  CK(cudaStreamCreateWithFlags(&h->s_h2d, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&h->s_d2h, cudaStreamNonBlocking));
  for (auto& sl : h->slot) {
    CK(cudaEventCreateWithFlags(&sl.h2d, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl.done, cudaEventDisableTiming));
    CK(cudaEventCreateWithFlags(&sl.d2h, cudaEventDisableTiming));
  }

  const int64_t rows = h->cap * h->K;
  const int tpc = std::min({router_tokens_per_cta(static_cast<int>(h->N), 32),
                            RouterBigSmem(static_cast<int>(h->N), 32, 3).tpc,
                            RouterLatSmem<3, 64>(static_cast<int>(h->N)).tpc});  // smallest tile of any variant
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
  h->wr64 = dalloc<double>(h->d * ((h->N + 3) / 4 * 4));
  CK(cudaFuncSetAttribute(router_kernel<128, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_kernel<32, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_big_kernel<32, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_lat_kernel<3, 256>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_lat_kernel<3, 128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
  CK(cudaFuncSetAttribute(router_lat_kernel<3, 64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 220 * 1024));
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
}

// m-tiles per L2-resident group for a row-grouped GEMM whose A rows are k_bytes long (decode_tile).
int64_t l2_group_budget() {
  static const int64_t budget = [] {
    const char* e = std::getenv("CL_MOE_L2_GROUP_MB");
    return (int64_t)(e ? std::atoi(e) : 32) << 20;
  }();
  return budget;
}
int m_group_for(int64_t k_bytes, int bm) {
  const int64_t budget = l2_group_budget();
  if (budget <= 0) return 0;
  return static_cast<int>(std::max<int64_t>(1, budget / (k_bytes * bm)));
}

template <int G, int EPI, bool F8, bool OF8, bool WG = false>
void launch_gemm(cl_moe* h, const CUtensorMap& a, const CUtensorMap& b, const GemmArgs& args_in, cudaStream_t st) {
  if (!h->tile_counter) h->tile_counter = dalloc<int>(1);
  GemmArgs args = args_in;
  args.tile_counter = h->tile_counter;
  if (!WG && args.m_group == 0) args.m_group = m_group_for((int64_t)args.num_kb * kBKBytes, 128 * G);
  if (WG && args.group_bytes == 0) args.group_bytes = l2_group_budget();
  CK(cudaMemsetAsync(h->tile_counter, 0, sizeof(int), st));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3((h->num_sms / G) * G);
  cfg.blockDim = dim3(kGemmThreads);
  cfg.dynamicSmemBytes = GemmCfg<G>::kSmem;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = G;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, grouped_gemm_kernel<G, EPI, F8, OF8, WG>, a, b, args));
}

// route_tokens on device: K1 + K2.
void run_router(cl_moe* h, const void* x, int64_t T, cudaStream_t st) {
  if (T < 1) throw RunErr("route_tokens: B must be >= 1");
  if (T > h->cap) throw ConfigErr(fmt("T=%lld exceeds max_tokens=%lld", (long long)T, (long long)h->cap));
  const int N = static_cast<int>(h->N);
  // small batches: 1 token x 4 experts per thread, 32-thread CTAs, 8-deep prefetch ring (latency);
  // large batches: 4 tokens x 4 experts per thread (shared-memory traffic per DFMA / 3).
  // decode-size batches: one thread per (token, expert) chain (latency-bound: parallelism first).
  static const int force = [] {
    const char* e = std::getenv("CL_MOE_ROUTER");  // bring-up / test override: "lat", "small" or "big"
    return e ? (e[0] == 'b' ? 2 : e[0] == 's' ? 1 : e[0] == 'l' ? 3 : 0) : 0;
  }();
  const int tpc_big = RouterBigSmem(N, 32, 3).tpc;
  const bool big_ok = RouterBigSmem(N, 32, 3).total <= 220 * 1024;
  const bool big = big_ok && (force == 2 || (force == 0 && (T + tpc_big - 1) / tpc_big >= h->num_sms));
  // latency variant: chunk length by expert count (shared-memory budget), ring depth 3
  const int N4r = (N + 3) / 4 * 4;
  const int lat_chunk = N4r <= 16 ? 256 : N4r <= 32 ? 128 : 64;
  const int tpc_lat = RouterLatSmem<3, 64>(N).tpc;
  const bool lat = !big && (force == 3 || (force == 0 && (T + tpc_lat - 1) / tpc_lat <= h->num_sms));
  const bool small = !big && !lat && router_smem_bytes(N, 32, 8) <= 220 * 1024;
  const int tpc = big ? tpc_big : lat ? tpc_lat : router_tokens_per_cta(N, small ? 32 : 128);
  h->tpc_cur = tpc;
  h->last_tokens = T;
  const int n_tiles = static_cast<int>((T + tpc - 1) / tpc);
  prof_begin(h, st);
  if (lat && lat_chunk == 256)
    router_lat_kernel<3, 256><<<n_tiles, 128, RouterLatSmem<3, 256>(N).total, st>>>(
        static_cast<const __nv_bfloat16*>(x), h->wr64, (int)T, (int)h->d, N, (int)h->K, h->rb);
  else if (lat && lat_chunk == 128)
    router_lat_kernel<3, 128><<<n_tiles, 128, RouterLatSmem<3, 128>(N).total, st>>>(
        static_cast<const __nv_bfloat16*>(x), h->wr64, (int)T, (int)h->d, N, (int)h->K, h->rb);
  else if (lat)
    router_lat_kernel<3, 64><<<n_tiles, 128, RouterLatSmem<3, 64>(N).total, st>>>(
        static_cast<const __nv_bfloat16*>(x), h->wr64, (int)T, (int)h->d, N, (int)h->K, h->rb);
  else if (big)
    router_big_kernel<32, 3><<<n_tiles, 32, RouterBigSmem(N, 32, 3).total, st>>>(
        static_cast<const __nv_bfloat16*>(x), h->wr64, (int)T, (int)h->d, N, (int)h->K, h->rb);
  else if (small)
    router_kernel<32, 8><<<n_tiles, 32, router_smem_bytes(N, 32, 8), st>>>(
        static_cast<const __nv_bfloat16*>(x), h->wr64, (int)T, (int)h->d, N, (int)h->K, h->rb);
  else
    router_kernel<128, 3><<<n_tiles, 128, router_smem_bytes(N, 128, 3), st>>>(
        static_cast<const __nv_bfloat16*>(x), h->wr64, (int)T, (int)h->d, N, (int)h->K, h->rb);
  CK(cudaGetLastError());
  prof_mark(h, 0, st);
  plan_kernel<<<1, kPlanThreads, 0, st>>>(n_tiles, (int)T, N, (int)h->K, h->rb);
  CK(cudaGetLastError());
  prof_mark(h, 1, st);
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
  plan_kernel<<<1, kPlanThreads, 0, st>>>(n_tiles, (int)T, N, (int)h->K, h->rb);
  CK(cudaGetLastError());
  prof_mark(h, 1, st);
}

// GEMM1 (+SwiGLU) and GEMM2 (+optional row weight) over the local expert segments `offsets`.
void run_gemms(cl_moe* h, const int32_t* offsets, void* act, __nv_bfloat16* y, const float* row_w,
               const CUtensorMap* mA1, const CUtensorMap* mA2, const CUtensorMap* mA1q, const CUtensorMap* mA2q,
               cudaStream_t st, __nv_bfloat16* h_save = nullptr, void* const* row_ptr = nullptr) {
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
  g1.n_tiles_n = static_cast<int>(2 * h->f / kBN);
  g1.num_kb = static_cast<int>(h->d * (fp8 ? 1 : 2) / kBKBytes);
  g1.b_rows_per_expert = static_cast<int>(2 * h->f);
  g1.out = act;
  g1.ldo = static_cast<int>(h->f);
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
  const int v = h->gemm_ctas == 2 ? 1 : 0;
  if (!fp8) {
    if (v) {
      launch_gemm<2, EPI_SWIGLU, false, false>(h, mA1[v], h->mB1[v], g1, st);
      prof_mark(h, 3, st);
      launch_gemm<2, EPI_ROWSCALE, false, false>(h, mA2[v], h->mB2[v], g2, st);
    } else {
      launch_gemm<1, EPI_SWIGLU, false, false>(h, mA1[v], h->mB1[v], g1, st);
      prof_mark(h, 3, st);
      launch_gemm<1, EPI_ROWSCALE, false, false>(h, mA2[v], h->mB2[v], g2, st);
    }
  } else {
    if (v) {
      launch_gemm<2, EPI_SWIGLU, true, true>(h, mA1q[v], h->mB1q[v], g1, st);
      prof_mark(h, 3, st);
      launch_gemm<2, EPI_ROWSCALE, true, false>(h, mA2q[v], h->mB2q[v], g2, st);
    } else {
      launch_gemm<1, EPI_SWIGLU, true, true>(h, mA1q[v], h->mB1q[v], g1, st);
      prof_mark(h, 3, st);
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
  if (h->win8) return;
  h->win8 = dalloc<uint8_t>((size_t)h->n_local * 2 * h->f * h->d);
  h->wout8 = dalloc<uint8_t>((size_t)h->n_local * h->d * h->f);
  h->ws_in = dalloc<float>((size_t)h->n_local * 2 * h->f);
  h->ws_out = dalloc<float>((size_t)h->n_local * h->d);
  build_maps(h, true);
}

void ep_fp8_maps(cl_moe* h) {
  if (h->maps_eq) return;
  for (int v = 0; v < 2; ++v) {
    h->mA1eq[v] = make_map(h->x_recv, true, h->d, h->recv_cap, 128);
    h->mA2eq[v] = make_map(h->act_recv, true, h->f, h->recv_cap, 128);
  }
  h->maps_eq = true;
}

void ep_alloc(cl_moe* h) {
  if (h->x_recv) return;
  const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
  h->recv_cap = h->cap * h->K * R;
  h->x_recv = dalloc<__nv_bfloat16>(h->recv_cap * h->d);
  h->act_recv = dalloc<__nv_bfloat16>(h->recv_cap * h->f);
  h->y_recv = dalloc<__nv_bfloat16>(h->recv_cap * h->d);
  h->ep_counts_dev = dalloc<int32_t>((size_t)R * h->N);
  h->ep_off_dev = dalloc<int32_t>(h->n_local + 1);
  CK(cudaMallocHost(&h->ep_counts_host, sizeof(int32_t) * R * h->N));
  CK(cudaMallocHost(&h->ep_off_host, sizeof(int32_t) * (h->n_local + 1)));
  for (int v = 0; v < 2; ++v) {
    h->mA1e[v] = make_map(h->x_recv, false, h->d, h->recv_cap, 128);
    h->mA2e[v] = make_map(h->act_recv, false, h->f, h->recv_cap, 128);
  }
}

#define NCK(x)                                                                               \
  do {                                                                                       \
    int r_ = (x);                                                                            \
    if (r_ != 0) throw RunErr(fmt("%s failed: %s", #x, NcclApi::get().GetErrorString(r_))); \
  } while (0)

// One direction of the expert-parallel row exchange (layout of the last EP forward).
// to_experts: rows of this rank's source permutation `src` (piece g at my_off[g]) go to the
// owner of expert g, landing at its (local expert, source) slot of `dst`; otherwise the reverse.
void ep_exchange(cl_moe* h, const void* src, void* dst, bool to_experts, cudaStream_t st, size_t row_b = 0) {
  NcclApi& nc = NcclApi::get();
  const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
  const int rank = h->cfg.ep_rank;
  const int N = static_cast<int>(h->N), NL = h->n_local;
  if (row_b == 0) row_b = static_cast<size_t>(h->d) * 2;
  const auto& C = h->ep_C;
  const auto& piece = h->ep_piece;
  const auto& my_off = h->ep_myoff;
  const uint8_t* s8 = static_cast<const uint8_t*>(src);
  uint8_t* d8 = static_cast<uint8_t*>(dst);
  NCK(nc.GroupStart());
  if (to_experts) {
    for (int r = 0; r < R; ++r)
      for (int e = 0; e < NL; ++e) {
        const int g = r * NL + e;
        const int64_t n = C[(size_t)rank * N + g];
        if (n) NCK(nc.Send(s8 + my_off[g] * row_b, n * row_b, NcclApi::kUint8, r, h->comm, st));
      }
    for (int e = 0; e < NL; ++e)
      for (int sr = 0; sr < R; ++sr) {
        const int64_t n = C[(size_t)sr * N + rank * NL + e];
        if (n) NCK(nc.Recv(d8 + piece[(size_t)e * R + sr] * row_b, n * row_b, NcclApi::kUint8, sr, h->comm, st));
      }
  } else {
    for (int e = 0; e < NL; ++e)
      for (int sr = 0; sr < R; ++sr) {
        const int64_t n = C[(size_t)sr * N + rank * NL + e];
        if (n) NCK(nc.Send(s8 + piece[(size_t)e * R + sr] * row_b, n * row_b, NcclApi::kUint8, sr, h->comm, st));
      }
    for (int r = 0; r < R; ++r)
      for (int e = 0; e < NL; ++e) {
        const int g = r * NL + e;
        const int64_t n = C[(size_t)rank * N + g];
        if (n) NCK(nc.Recv(d8 + my_off[g] * row_b, n * row_b, NcclApi::kUint8, r, h->comm, st));
      }
  }
  NCK(nc.GroupEnd());
}

// Expert-parallel forward (ep.cuh): route + plan + dispatch over all N experts, counts
// all-gather, (expert, source)-piece exchange, local grouped GEMMs, reverse exchange, weighted
// combine. Requires cl_moe_ep_init. bf16 only in this round. `train` keeps H / A^T on the expert
// side for cl_moe_backward.
void run_ep_peer(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st, bool train);

void run_ep(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st, bool train) {
  if (!h->comm) throw ConfigErr("expert parallelism needs cl_moe_ep_init first");
  const bool fp8 = h->precision == CL_MOE_FP8_E4M3;
  if (fp8 && train) throw ConfigErr("training runs in bf16 (set_precision(BF16) first)");
  if (fp8) ep_fp8_maps(h);
  if (h->ep_transport == 1) {
    run_ep_peer(h, x, T, out, out_f32, st, train);
    return;
  }
  NcclApi& nc = NcclApi::get();
  const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
  const int rank = h->cfg.ep_rank;
  const int N = static_cast<int>(h->N), NL = h->n_local;
  const int tpc = h->tpc_cur;
  const int blocks = static_cast<int>((T + 7) / 8);
  if (fp8)  // rows quantized with their owner's GEMM1-input scale (global table)
    dispatch_kernel<true><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N,
                                                  (int)h->K, tpc, h->rb, h->rb.topk_idx, h->rb.combine_w, h->xperm,
                                                  h->perm, h->inv, h->row_w, h->sx_in_all);
  else
    dispatch_kernel<false><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N,
                                                   (int)h->K, tpc, h->rb, h->rb.topk_idx, h->rb.combine_w, h->xperm,
                                                   h->perm, h->inv, h->row_w, nullptr);
  CK(cudaGetLastError());
  prof_mark(h, 2, st);
  // ---- counts exchange ----
  NCK(nc.AllGather(h->rb.counts, h->ep_counts_dev, (size_t)N, NcclApi::kInt32, h->comm, st));
  CK(cudaMemcpyAsync(h->ep_counts_host, h->ep_counts_dev, sizeof(int32_t) * R * N, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  h->ep_C.assign((size_t)R * N, 0);
  h->ep_piece.assign((size_t)NL * R, 0);
  h->ep_myoff.assign((size_t)N + 1, 0);
  std::vector<int64_t> loc(NL + 1);
  for (size_t i = 0; i < h->ep_C.size(); ++i) h->ep_C[i] = h->ep_counts_host[i];
  const int64_t total = ep_layout(h->ep_C.data(), R, N, rank, loc.data(), h->ep_piece.data());
  if (total > h->recv_cap) throw RunErr("expert-parallel receive buffer overflow");
  for (int g = 0; g < N; ++g) h->ep_myoff[g + 1] = h->ep_myoff[g] + h->ep_C[(size_t)rank * N + g];
  for (int e = 0; e <= NL; ++e) h->ep_off_host[e] = static_cast<int32_t>(loc[e]);
  CK(cudaMemcpyAsync(h->ep_off_dev, h->ep_off_host, sizeof(int32_t) * (NL + 1), cudaMemcpyHostToDevice, st));
  // ---- dispatch exchange: piece (dest r, expert g) -> r's (local expert, source) slot ----
  ep_exchange(h, h->xperm, h->x_recv, true, st, (size_t)h->d * (fp8 ? 1 : 2));
  // ---- local experts ----
  if (train) {
    pad_plan_kernel<<<1, 32, 0, st>>>(h->ep_off_dev, NL, h->poff, h->kb_off);
    CK(cudaGetLastError());
  }
  run_gemms(h, h->ep_off_dev, h->act_recv, h->y_recv, nullptr, h->mA1e, h->mA2e, h->mA1eq, h->mA2eq, st,
            train ? h->Hbuf : nullptr);
  prof_mark(h, 4, st);
  // ---- reverse exchange into this rank's permutation slots ----
  ep_exchange(h, h->y_recv, h->y, false, st);
  if (out_f32)
    launch_combine<float>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<float*>(out), h->rb.finite_flag, st,
                          h->rb.combine_w);
  else
    launch_combine<__nv_bfloat16>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<__nv_bfloat16*>(out),
                                  h->rb.finite_flag, st, h->rb.combine_w);
  CK(cudaGetLastError());
  prof_mark(h, 5, st);
  h->cur_ev = nullptr;
  h->last_rows = T * h->K;
  if (train) {
    h->train_T = T;
    h->cur_x = x;
  }
}

// ---- peer-memory transport (ep.cuh): phases shared by the multi-process path and the
// single-process emulation group ----
void ep_peer_alloc(cl_moe* h) {
  if (h->row_ptr) return;
  const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
  h->peer_x_dev = dalloc<char*>(R);
  h->peer_y_dev = dalloc<char*>(R);
  h->peer_w_dev = dalloc<float*>(R);
  h->w_recv = dalloc<float>(h->recv_cap);
  h->expert_dst = dalloc<void*>(h->N);
  h->expert_dst_w = dalloc<float*>(h->N);
  h->row_ptr = dalloc<void*>(h->recv_cap);
  h->peer_dy_dev = dalloc<char*>(R);
  h->peer_dx_dev = dalloc<char*>(R);
  h->expert_dst_dy = dalloc<void*>(h->N);
  h->row_ptr_dx = dalloc<void*>(h->recv_cap);
  if (h->f % 256 == 0) {  // training-capable: the two backward exchange targets, mapped by peers
    if (!h->dYbuf) h->dYbuf = dalloc<__nv_bfloat16>(h->recv_cap * h->d);
    if (!h->dXsrc) h->dXsrc = dalloc<__nv_bfloat16>(h->cap * h->K * h->d);
  }
  h->bar_buf = dalloc<float>(1);
  CK(cudaMemset(h->bar_buf, 0, sizeof(float)));
}

void ep_peer_layout(cl_moe* h, cudaStream_t st) {
  const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
  const int64_t xrb = h->d * (h->precision == CL_MOE_FP8_E4M3 ? 1 : 2);
  ep_peer_layout_kernel<<<h->n_local * R + 1, 256, 0, st>>>(h->ep_counts_dev, R, (int)h->N, h->cfg.ep_rank, h->recv_cap,
                                                             xrb, h->d * 2, h->peer_x_dev, h->peer_y_dev, h->peer_w_dev,
                                                             h->expert_dst, h->expert_dst_w, h->ep_off_dev, h->row_ptr,
                                                             h->rb.finite_flag, h->peer_dy_dev, h->peer_dx_dev,
                                                             h->expert_dst_dy, h->row_ptr_dx);
  CK(cudaGetLastError());
}

void ep_peer_dispatch(cl_moe* h, const void* x, int64_t T, cudaStream_t st) {
  const int blocks = static_cast<int>((T + 7) / 8);
  if (h->precision == CL_MOE_FP8_E4M3)
    dispatch_kernel<true><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, (int)h->N,
                                                  (int)h->K, h->tpc_cur, h->rb, h->rb.topk_idx, h->rb.combine_w,
                                                  h->xperm, h->perm, h->inv, h->row_w, h->sx_in_all, h->expert_dst,
                                                  h->expert_dst_w);
  else
    dispatch_kernel<false><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, (int)h->N,
                                                   (int)h->K, h->tpc_cur, h->rb, h->rb.topk_idx, h->rb.combine_w,
                                                   h->xperm, h->perm, h->inv, h->row_w, nullptr, h->expert_dst,
                                                   h->expert_dst_w);
  CK(cudaGetLastError());
  prof_mark(h, 2, st);
}

void ep_peer_experts(cl_moe* h, cudaStream_t st, bool train = false) {
  if (h->precision == CL_MOE_FP8_E4M3) ep_fp8_maps(h);
  if (train) {  // padded row plan of the receive layout for the weight-gradient GEMMs
    pad_plan_kernel<<<1, 32, 0, st>>>(h->ep_off_dev, h->n_local, h->poff, h->kb_off);
    CK(cudaGetLastError());
  }
  // inference: rows return weighted (as on one GPU); training keeps Y unweighted for the backward
  run_gemms(h, h->ep_off_dev, h->act_recv, h->y_recv, train ? nullptr : h->w_recv, h->mA1e, h->mA2e, h->mA1eq,
            h->mA2eq, st, train ? h->Hbuf : nullptr, h->row_ptr);
  prof_mark(h, 4, st);
}

void ep_peer_combine(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st,
                     bool train = false) {
  // inference: rows arrive already scaled by their combine weight (GEMM2 epilogue), as on one GPU
  const float* w = train ? h->rb.combine_w : nullptr;
  if (out_f32)
    launch_combine<float>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<float*>(out), h->rb.finite_flag, st,
                          w);
  else
    launch_combine<__nv_bfloat16>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<__nv_bfloat16*>(out),
                                  h->rb.finite_flag, st, w);
  if (train) {
    h->train_T = T;
    h->cur_x = x;
  }
  CK(cudaGetLastError());
  prof_mark(h, 5, st);
  h->cur_ev = nullptr;
  h->last_rows = T * h->K;
}

// Multi-process forward over NVLink peer memory. NCCL carries only the R x N counts and two
// one-float barriers; the rows move as direct stores of the dispatch kernel and of the GEMM2
// epilogue. No host synchronisation: the layout is computed on the device.
//   all-gather(counts) -> layout -> dispatch (stores into owners' x_recv) -> barrier
//   -> GEMM1 -> GEMM2 (epilogue stores into sources' y) -> barrier -> combine
// The first all-gather also orders this forward after every rank's previous use of x_recv / y.
void run_ep_peer(cl_moe* h, const void* x, int64_t T, void* out, bool out_f32, cudaStream_t st, bool train) {
  NcclApi& nc = NcclApi::get();
  NCK(nc.AllGather(h->rb.counts, h->ep_counts_dev, (size_t)h->N, NcclApi::kInt32, h->comm, st));
  ep_peer_layout(h, st);
  ep_peer_dispatch(h, x, T, st);
  NCK(nc.AllReduce(h->bar_buf, h->bar_buf, 1, NcclApi::kFloat32, NcclApi::kSum, h->comm, st));
  ep_peer_experts(h, st, train);
  NCK(nc.AllReduce(h->bar_buf, h->bar_buf, 1, NcclApi::kFloat32, NcclApi::kSum, h->comm, st));
  ep_peer_combine(h, x, T, out, out_f32, st, train);
}

void ensure_training(cl_moe* h) {
  if (h->train_ready) return;
  if (h->f % 256) throw ConfigErr("training needs d_ff to be a multiple of 256");
  if (h->cfg.ep_size > 1 && !h->comm && !h->ep_group)
    throw ConfigErr("expert-parallel training needs cl_moe_ep_init first");
  const bool ep = h->comm != nullptr || h->ep_group;
  // expert-side rows: the receive buffer under expert parallelism
  const int64_t rows = ep ? h->recv_cap : h->cap * h->K, d = h->d, f = h->f, NL = h->n_local;
  if (!h->win_ref) {  // buffers and descriptors: once per handle
    if (ep) {
      h->dYsrc = dalloc<__nv_bfloat16>(h->cap * h->K * d);
      if (!h->dXsrc) h->dXsrc = dalloc<__nv_bfloat16>(h->cap * h->K * d);
    }
    h->rp_cap = (rows + 63) / 64 * 64 + 64 * NL;  // 64-aligned: TMA row strides must be 16-byte multiples
    h->win_ref = dalloc<__nv_bfloat16>((size_t)NL * d * 2 * f);
    h->wout_ref = dalloc<__nv_bfloat16>((size_t)NL * f * d);
    h->Hbuf = dalloc<__nv_bfloat16>(rows * 2 * f);
    if (!h->dYbuf) h->dYbuf = dalloc<__nv_bfloat16>(rows * d);
    h->dHbuf = dalloc<__nv_bfloat16>(rows * 2 * f);
    h->dXbuf = dalloc<__nv_bfloat16>(rows * d);
    h->XT = dalloc<__nv_bfloat16>(d * h->rp_cap);
    h->AT = dalloc<__nv_bfloat16>(f * h->rp_cap);
    h->dYT = dalloc<__nv_bfloat16>(d * h->rp_cap);
    h->dHT = dalloc<__nv_bfloat16>(2 * f * h->rp_cap);
    h->poff = dalloc<int32_t>(NL + 1);
    h->kb_off = dalloc<int32_t>(NL + 1);
    for (int v = 0; v < 2; ++v) {
      const uint32_t brow = v == 0 ? 256 : 128;
      h->mAdg1[v] = make_map(h->dYbuf, false, d, rows, 128);
      h->mBdg1[v] = make_map(h->wout_ref, false, d, (uint64_t)NL * f, brow);
      h->mAdg2[v] = make_map(h->dHbuf, false, 2 * f, rows, 128);
      h->mBdg2[v] = make_map(h->win_ref, false, 2 * f, (uint64_t)NL * d, brow);
      h->mAwo[v] = make_map(h->AT, false, h->rp_cap, f, 128);
      h->mBwo[v] = make_map(h->dYT, false, h->rp_cap, d, brow);
      h->mAwi[v] = make_map(h->XT, false, h->rp_cap, d, 128);
      h->mBwi[v] = make_map(h->dHT, false, h->rp_cap, 2 * f, brow);
    }
  }
  // reference-layout weight copies (re-derived whenever the packed weights change)
  for (int e = 0; e < NL; ++e) {
    transpose_weight_kernel<true><<<dim3((unsigned)(2 * f / 32), (unsigned)(d / 32)), 256>>>(
        h->win + (size_t)e * 2 * f * d, (int)(2 * f), (int)d, (int)f, h->win_ref + (size_t)e * d * 2 * f);
    transpose_weight_kernel<false><<<dim3((unsigned)(d / 32), (unsigned)(f / 32)), 256>>>(
        h->wout + (size_t)e * d * f, (int)d, (int)f, (int)f, h->wout_ref + (size_t)e * f * d);
  }
  CK(cudaGetLastError());
  CK(cudaDeviceSynchronize());
  h->train_ready = true;
}

// Training-mode forward: H = [G | U] kept, Y kept unweighted, combine weights applied in the
// combine (fp32) so the backward can form d(combine_w) = <dOut, Y>.
void run_forward_train(cl_moe* h, const void* x, int64_t T, void* out, cudaStream_t st) {
  if (h->precision != CL_MOE_BF16) throw ConfigErr("training runs in bf16");
  if (h->cfg.ep_size > 1 && !h->comm)
    throw ConfigErr("ep_size > 1 needs cl_moe_ep_init (or cl_moe_ep_group_train_step)");
  ensure_training(h);
  if (h->comm) {
    run_ep(h, x, T, out, false, st, true);
    return;
  }
  const int N = static_cast<int>(h->N);
  const int tpc = h->tpc_cur;
  const int blocks = static_cast<int>((T + 7) / 8);
  dispatch_kernel<false><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N, (int)h->K,
                                                 tpc, h->rb, h->rb.topk_idx, h->rb.combine_w, h->xperm, h->perm,
                                                 h->inv, h->row_w, nullptr);
  pad_plan_kernel<<<1, 32, 0, st>>>(h->rb.offsets, h->n_local, h->poff, h->kb_off);
  CK(cudaGetLastError());
  prof_mark(h, 2, st);
  run_gemms(h, h->rb.offsets, h->act, h->y, nullptr, h->mA1, h->mA2, h->mA1q, h->mA2q, st, h->Hbuf);
  prof_mark(h, 4, st);
  launch_combine<__nv_bfloat16>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<__nv_bfloat16*>(out),
                                h->rb.finite_flag, st, h->rb.combine_w);
  CK(cudaGetLastError());
  prof_mark(h, 5, st);
  h->cur_ev = nullptr;
  h->last_rows = T * h->K;
  h->train_T = T;
  h->cur_x = x;
}

// Expert-FFN backward of the last training forward.
// Backward phases (shared by the single-handle call and the single-process EP group):
//   A  combine backward (+ dY rows to the experts' owners)
//   B  dgrad GEMMs on the expert side (+ dX rows back to their sources)
//   C  dispatch backward (+ router backward)
//   D  transposes and weight-gradient GEMMs
// Under the peer transport, A's kernel stores dY rows straight into the owners' dYbuf and B's
// dgrad-2 epilogue stores dX rows straight into the sources' dXsrc; the caller puts a barrier
// between A/B and B/C (NCCL all-reduce of one float, or phase order in the group).
struct BwdArgs {
  const void* d_out;
  void* d_hidden;
  float* d_cw;
  float* dw_in;
  float* dw_out;
  float* dw_router;
  float g_aux, g_z;
};

bool ep_mode(const cl_moe* h) { return h->comm != nullptr || h->ep_group; }
bool ep_peer_mode(const cl_moe* h) { return h->ep_group || (h->comm && h->ep_transport == 1); }

void bwd_check(cl_moe* h) {
  if (!h->train_ready || h->train_T == 0) throw ConfigErr("backward needs a preceding cl_moe_forward_train");
}

void bwd_phase_a(cl_moe* h, const BwdArgs& a, cudaStream_t st) {
  const int64_t T = h->train_T, rows = T * h->K, d = h->d;
  const bool ep = ep_mode(h), peer = ep_peer_mode(h);
  __nv_bfloat16* dY_src = ep ? h->dYsrc : h->dYbuf;
  prof_begin(h, st, 1);
  // 1. combine backward: dY = w * dOut[token], d_combine_w = <dOut[token], Y>
  combine_bwd_kernel<<<(int)((rows + 7) / 8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a.d_out), h->y, h->perm,
                                                           h->rb.combine_w, (int)rows, (int)d, (int)h->K, dY_src,
                                                           a.d_cw, peer ? h->expert_dst_dy : nullptr, h->rb.topk_idx,
                                                           h->rb.offsets);
  CK(cudaGetLastError());
  if (ep && !peer) ep_exchange(h, dY_src, h->dYbuf, true, st);  // dY rows to the experts' owners
  prof_mark(h, 0, st);
}

void bwd_phase_b(cl_moe* h, const BwdArgs& a, cudaStream_t st) {
  const int64_t d = h->d, f = h->f;
  const int NL = h->n_local;
  const bool ep = ep_mode(h), peer = ep_peer_mode(h);
  const int32_t* es_off = ep ? h->ep_off_dev : h->rb.offsets;
  __nv_bfloat16* dX_src = ep ? h->dXsrc : h->dXbuf;
  const int v = h->gemm_ctas == 2 ? 1 : 0;  // same variant the training forward chose
  // 2. dA = dY W_out^T fused with the SwiGLU backward -> dH
  GemmArgs a1{};
  a1.offsets = es_off;
  a1.n_experts = NL;
  a1.n_tiles_n = static_cast<int>(f / kBN);
  a1.num_kb = static_cast<int>(d * 2 / kBKBytes);
  a1.b_rows_per_expert = static_cast<int>(f);
  a1.out = h->dHbuf;
  a1.aux = h->Hbuf;
  a1.ffn = static_cast<int>(f);
  a1.aux_t = h->dHT;  // dH^T straight from the epilogue (dW_in GEMM operand)
  a1.rp = h->rp_cap;
  a1.poff = h->poff;
  // 3. dX = dH W_in^T (peer transport: each row straight back into its source's dXsrc)
  GemmArgs a2{};
  a2.offsets = es_off;
  a2.n_experts = NL;
  a2.n_tiles_n = static_cast<int>(d / kBN);
  a2.num_kb = static_cast<int>(2 * f * 2 / kBKBytes);
  a2.b_rows_per_expert = static_cast<int>(d);
  a2.out = h->dXbuf;
  a2.ldo = static_cast<int>(d);
  a2.row_ptr = peer ? h->row_ptr_dx : nullptr;
  if (v) {
    launch_gemm<2, EPI_SWIGLU_BWD, false, false>(h, h->mAdg1[v], h->mBdg1[v], a1, st);
    prof_mark(h, 1, st);
    launch_gemm<2, EPI_ROWSCALE, false, false>(h, h->mAdg2[v], h->mBdg2[v], a2, st);
  } else {
    launch_gemm<1, EPI_SWIGLU_BWD, false, false>(h, h->mAdg1[v], h->mBdg1[v], a1, st);
    prof_mark(h, 1, st);
    launch_gemm<1, EPI_ROWSCALE, false, false>(h, h->mAdg2[v], h->mBdg2[v], a2, st);
  }
  if (ep && !peer) ep_exchange(h, h->dXbuf, dX_src, false, st);  // dX rows back to their tokens' ranks
  prof_mark(h, 2, st);
}

void bwd_phase_c(cl_moe* h, const BwdArgs& a, cudaStream_t st) {
  const int64_t T = h->train_T, d = h->d;
  const bool ep = ep_mode(h);
  __nv_bfloat16* dX_src = ep ? h->dXsrc : h->dXbuf;
  // 4. dispatch backward (gather_rows bwd): d_hidden[j] = sum_k dX[inv[j,k]]  (+ router term)
  if (a.dw_router) {
    const int N = static_cast<int>(h->N);
    if (!h->rdz) {
      h->rdz = dalloc<float>(h->cap * h->N);
      h->rpart = dalloc<float>(((h->cap + kRwTokens - 1) / kRwTokens) * h->d * h->N);
    }
    router_bwd_dz_kernel<<<(int)((T + 127) / 128), 128, 0, st>>>(h->rb.probs, h->rb.logits, h->rb.topk_idx, a.d_cw,
                                                                h->rb.counts, (int)T, N, (int)h->K, a.g_aux, a.g_z,
                                                                h->rdz);
    const int chunks = static_cast<int>((T + kRwTokens - 1) / kRwTokens);
    router_wgrad_partial_kernel<<<dim3((unsigned)(d / 64), (unsigned)chunks, (unsigned)((N + 15) / 16)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(h->cur_x), h->rdz, (int)T, (int)d, N, h->rpart);
    router_wgrad_reduce_kernel<<<(int)((d * N + 255) / 256), 256, 0, st>>>(h->rpart, chunks, (int)(d * N), a.dw_router);
    // the router is replicated: its gradient is the sum over the data-parallel ranks
    if (h->comm) NCK(NcclApi::get().AllReduce(a.dw_router, a.dw_router, (size_t)(d * N), NcclApi::kFloat32,
                                              NcclApi::kSum, h->comm, st));
    const int blocks = static_cast<int>((T + 7) / 8);
    switch (h->K) {
      case 1: dispatch_bwd_router_kernel<1><<<blocks, 256, 0, st>>>(dX_src, h->inv, (int)T, (int)d, h->rdz, h->wr, N, static_cast<__nv_bfloat16*>(a.d_hidden)); break;
      case 2: dispatch_bwd_router_kernel<2><<<blocks, 256, 0, st>>>(dX_src, h->inv, (int)T, (int)d, h->rdz, h->wr, N, static_cast<__nv_bfloat16*>(a.d_hidden)); break;
      case 4: dispatch_bwd_router_kernel<4><<<blocks, 256, 0, st>>>(dX_src, h->inv, (int)T, (int)d, h->rdz, h->wr, N, static_cast<__nv_bfloat16*>(a.d_hidden)); break;
      default: throw ConfigErr("router backward supports top_k in {1, 2, 4}");
    }
  } else {
    launch_combine<__nv_bfloat16>(dX_src, h->inv, (int)T, (int)d, (int)h->K, static_cast<__nv_bfloat16*>(a.d_hidden),
                                  h->rb.finite_flag, st);
  }
  CK(cudaGetLastError());
  prof_mark(h, 3, st);
}

void bwd_phase_d(cl_moe* h, const BwdArgs& a, cudaStream_t st) {
  const int64_t d = h->d, f = h->f;
  const int NL = h->n_local;
  const bool ep = ep_mode(h);
  const int32_t* es_off = ep ? h->ep_off_dev : h->rb.offsets;
  const void* es_x = ep ? static_cast<const void*>(h->x_recv) : h->xperm;
  // 5. weight gradients over each expert's rows (variable K): padded K-major transposes, then
  //    dW_out[e] = A_e^T dY_e ([f x d]) and dW_in[e] = X_e^T dH_e ([d x 2f]), fp32.
  //    (A^T and dH^T were written by the GEMM1 / dgrad-1 epilogues; only their padding columns
  //    need zeroing. X^T and dY^T go through the transpose kernel.)
  const unsigned pb = static_cast<unsigned>(h->rp_cap / 64);
  transpose_pad_kernel<<<dim3((unsigned)(d / 64), pb), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(es_x), (int)d,
                                                                     es_off, h->poff, NL, h->XT, h->rp_cap);
  transpose_pad_kernel<<<dim3((unsigned)(d / 64), pb), 256, 0, st>>>(h->dYbuf, (int)d, es_off, h->poff, NL, h->dYT,
                                                                     h->rp_cap);
  zero_pad_cols_kernel<<<dim3((unsigned)((f + 7) / 8), (unsigned)NL), 256, 0, st>>>(h->AT, (int)f, h->rp_cap, es_off,
                                                                                    h->poff);
  zero_pad_cols_kernel<<<dim3((unsigned)((2 * f + 7) / 8), (unsigned)NL), 256, 0, st>>>(h->dHT, (int)(2 * f),
                                                                                        h->rp_cap, es_off, h->poff);
  CK(cudaGetLastError());
  prof_mark(h, 4, st);
  const int gw = (f % 256 == 0) ? 2 : 1;
  GemmArgs wo{};
  wo.n_experts = NL;
  wo.kb_off = h->kb_off;
  wo.m_tiles = static_cast<int>(f / (128 * gw));
  wo.n_tiles_n = static_cast<int>(d / kBN);
  wo.out = a.dw_out;
  wo.ldo = static_cast<int>(d);
  wo.out_estride = f * d;
  GemmArgs wi{};
  wi.n_experts = NL;
  wi.kb_off = h->kb_off;
  wi.m_tiles = static_cast<int>(d / (128 * gw));
  wi.n_tiles_n = static_cast<int>(2 * f / kBN);
  wi.out = a.dw_in;
  wi.ldo = static_cast<int>(2 * f);
  wi.out_estride = d * 2 * f;
  if (gw == 2) {
    launch_gemm<2, EPI_WGRAD, false, false, true>(h, h->mAwo[1], h->mBwo[1], wo, st);
    prof_mark(h, 5, st);
    launch_gemm<2, EPI_WGRAD, false, false, true>(h, h->mAwi[1], h->mBwi[1], wi, st);
  } else {
    launch_gemm<1, EPI_WGRAD, false, false, true>(h, h->mAwo[0], h->mBwo[0], wo, st);
    prof_mark(h, 5, st);
    launch_gemm<1, EPI_WGRAD, false, false, true>(h, h->mAwi[0], h->mBwi[0], wi, st);
  }
  prof_mark(h, 6, st);
  h->cur_ev = nullptr;
}

// One float all-reduce on the communicator: orders every rank's preceding peer stores before
// anything this rank issues next (the stores were fenced with __threadfence_system).
void ep_barrier(cl_moe* h, cudaStream_t st) {
  NCK(NcclApi::get().AllReduce(h->bar_buf, h->bar_buf, 1, NcclApi::kFloat32, NcclApi::kSum, h->comm, st));
}

void run_backward(cl_moe* h, const void* d_out, void* d_hidden, float* d_cw, float* dw_in, float* dw_out,
                  cudaStream_t st, float* dw_router = nullptr, float g_aux = 0.0f, float g_z = 0.0f) {
  bwd_check(h);
  const BwdArgs a{d_out, d_hidden, d_cw, dw_in, dw_out, dw_router, g_aux, g_z};
  const bool peer = h->comm && h->ep_transport == 1;
  bwd_phase_a(h, a, st);
  if (peer) ep_barrier(h, st);
  bwd_phase_b(h, a, st);
  if (peer) ep_barrier(h, st);
  bwd_phase_c(h, a, st);
  bwd_phase_d(h, a, st);
}

}  // namespace

extern "C" {

cl_status cl_moe_ep_unique_id(uint8_t* id_out) {
  if (!id_out) return CL_ERR_CONFIG;
  try {
    NcclApi::UniqueId id;
    if (NcclApi::get().GetUniqueId(&id) != 0) return CL_ERR_RUN;
    std::memcpy(id_out, id.internal, 128);
    return CL_OK;
  } catch (const std::exception& e) {
    std::fprintf(stderr, "cl_moe_ep_unique_id: %s\n", e.what());
    return CL_ERR_RUN;
  }
}

cl_status cl_moe_ep_init(cl_moe* h, const uint8_t* id) {
  return guarded(h, [&] {
    if (!id) throw ConfigErr("id is null");
    CK(cudaSetDevice(h->cfg.device));
    const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
    NcclApi::UniqueId uid;
    std::memcpy(uid.internal, id, 128);
    if (h->comm) {
      NcclApi::get().CommDestroy(h->comm);
      h->comm = nullptr;
    }
    NCK(NcclApi::get().CommInitRank(&h->comm, R, uid, h->cfg.ep_rank));
    ep_alloc(h);
  });
}

cl_status cl_moe_ep_peer_init(cl_moe* h) {
  return guarded(h, [&] {
    if (!h->comm) throw ConfigErr("cl_moe_ep_peer_init needs cl_moe_ep_init first");
    CK(cudaSetDevice(h->cfg.device));
    const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size, rank = h->cfg.ep_rank;
    ep_peer_alloc(h);
    // exchange the IPC handles of x_recv and y over the communicator
    constexpr size_t kH = sizeof(cudaIpcMemHandle_t);
    constexpr int kB = 5;  // x_recv, y, w_recv, and for training dYbuf, dXsrc
    void* const own[kB] = {h->x_recv, h->y, h->w_recv, h->dYbuf, h->dXsrc};
    std::vector<uint8_t> mine(kB * kH, 0), all(kB * kH * R);
    for (int b = 0; b < kB; ++b) {
      if (!own[b]) continue;  // not training-capable (d_ff % 256): an all-zero handle
      cudaIpcMemHandle_t hb;
      CK(cudaIpcGetMemHandle(&hb, own[b]));
      std::memcpy(mine.data() + b * kH, &hb, kH);
    }
    uint8_t* dbuf = dalloc<uint8_t>(kB * kH * (R + 1));
    cudaStream_t st = nullptr;
    CK(cudaMemcpy(dbuf, mine.data(), kB * kH, cudaMemcpyHostToDevice));
    NCK(NcclApi::get().AllGather(dbuf, dbuf + kB * kH, kB * kH, NcclApi::kUint8, h->comm, st));
    CK(cudaStreamSynchronize(st));
    CK(cudaMemcpy(all.data(), dbuf + kB * kH, kB * kH * R, cudaMemcpyDeviceToHost));
    cudaFree(dbuf);
    std::vector<void*> peer[kB];
    for (int b = 0; b < kB; ++b) peer[b].assign(R, nullptr);
    std::string why;
    for (int s = 0; s < R && why.empty(); ++s)
      for (int b = 0; b < kB && why.empty(); ++b) {
        if (s == rank) {
          peer[b][s] = own[b];
          continue;
        }
        if (!own[b]) continue;  // same on every rank (same configuration)
        cudaIpcMemHandle_t hd;
        std::memcpy(&hd, all.data() + ((size_t)s * kB + b) * kH, kH);
        void* p = nullptr;
        const cudaError_t e = cudaIpcOpenMemHandle(&p, hd, cudaIpcMemLazyEnablePeerAccess);
        if (e != cudaSuccess) {
          cudaGetLastError();
          why = fmt("rank %d cannot map rank %d's buffers: %s", rank, s, cudaGetErrorString(e));
          break;
        }
        h->ipc_opened.push_back(p);
        peer[b][s] = p;
      }
    // all ranks switch together or not at all
    float* okf = dalloc<float>(1);
    const float bad = why.empty() ? 0.f : 1.f;
    CK(cudaMemcpy(okf, &bad, sizeof(float), cudaMemcpyHostToDevice));
    NCK(NcclApi::get().AllReduce(okf, okf, 1, NcclApi::kFloat32, NcclApi::kSum, h->comm, st));
    CK(cudaStreamSynchronize(st));
    float nbad = 0.f;
    CK(cudaMemcpy(&nbad, okf, sizeof(float), cudaMemcpyDeviceToHost));
    cudaFree(okf);
    if (nbad > 0.f) {
      for (void* p : h->ipc_opened) cudaIpcCloseMemHandle(p);
      h->ipc_opened.clear();
      throw RunErr(why.empty() ? fmt("peer transport unavailable on %d rank(s); keeping NCCL", (int)nbad) : why);
    }
    CK(cudaMemcpy(h->peer_x_dev, peer[0].data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->peer_y_dev, peer[1].data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->peer_w_dev, peer[2].data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->peer_dy_dev, peer[3].data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->peer_dx_dev, peer[4].data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
    h->ep_transport = 1;
  });
}

// Single-process emulation of R expert-parallel ranks on one device (test and bring-up path):
// the same layout / dispatch / GEMM / combine kernels with "peer" addresses that are the other
// handles' buffers. Every phase runs for all ranks before the next one starts, in stream order,
// so no kernel ever waits on another; the count all-gather becomes R x R device copies.
static void group_check(cl_moe* const* hs, int R) {
  cl_moe* h0 = hs[0];
  for (int r = 0; r < R; ++r) {
    cl_moe* h = hs[r];
    if (h->cfg.ep_size != R || h->cfg.ep_rank != r || h->N != h0->N || h->d != h0->d || h->f != h0->f ||
        h->K != h0->K || h->cfg.device != h0->cfg.device)
      throw ConfigErr(fmt("handle %d is not rank %d of a matching %d-rank group", r, r, R));
    if (h->precision != h0->precision) throw ConfigErr("all ranks of a group need the same precision");
    if (h->comm) throw ConfigErr("group handles must not have a communicator");
  }
}

// Forward of every rank, phase by phase (see cl_moe_ep_group_forward).
static void group_forward(cl_moe* const* hs, int R, const void* const* hidden, const int64_t* T, void* const* out,
                          cudaStream_t st, bool train) {
  const int N = static_cast<int>(hs[0]->N);
  std::vector<char*> px(R), py(R), pdy(R), pdx(R);
  std::vector<float*> pw(R);
  for (int r = 0; r < R; ++r) {
    cl_moe* h = hs[r];
    h->ep_group = true;
    ep_alloc(h);
    ep_peer_alloc(h);
    if (train) ensure_training(h);
    px[r] = reinterpret_cast<char*>(h->x_recv);
    py[r] = reinterpret_cast<char*>(h->y);
    pw[r] = h->w_recv;
    pdy[r] = reinterpret_cast<char*>(h->dYbuf);
    pdx[r] = reinterpret_cast<char*>(h->dXsrc);
  }
  for (int r = 0; r < R; ++r) {
    CK(cudaMemcpyAsync(hs[r]->peer_x_dev, px.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_y_dev, py.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_w_dev, pw.data(), sizeof(float*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_dy_dev, pdy.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_dx_dev, pdx.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
  }
  for (int r = 0; r < R; ++r) run_router(hs[r], hidden[r], T[r], st);
  for (int r = 0; r < R; ++r)
    for (int s = 0; s < R; ++s)
      CK(cudaMemcpyAsync(hs[r]->ep_counts_dev + (size_t)s * N, hs[s]->rb.counts, sizeof(int32_t) * N,
                         cudaMemcpyDeviceToDevice, st));
  for (int r = 0; r < R; ++r) ep_peer_layout(hs[r], st);
  for (int r = 0; r < R; ++r) ep_peer_dispatch(hs[r], hidden[r], T[r], st);
  for (int r = 0; r < R; ++r) ep_peer_experts(hs[r], st, train);
  for (int r = 0; r < R; ++r) ep_peer_combine(hs[r], hidden[r], T[r], out[r], false, st, train);
  CK(cudaStreamSynchronize(st));  // the host pointer tables above must outlive their copies
}

// Single-process emulation of R expert-parallel ranks on one device (test and bring-up path):
// the same layout / dispatch / GEMM / combine kernels with "peer" addresses that are the other
// handles' buffers. Every phase runs for all ranks before the next one starts, in stream order,
// so no kernel ever waits on another; the count all-gather becomes R x R device copies.
cl_status cl_moe_ep_group_forward(cl_moe* const* hs, int32_t R, const void* const* hidden, const int64_t* T,
                                  void* const* out, void* stream) {
  if (!hs || R < 1 || !hidden || !T || !out) return CL_ERR_CONFIG;
  for (int r = 0; r < R; ++r)
    if (!hs[r]) return CL_ERR_CONFIG;
  return guarded(hs[0], [&] {
    group_check(hs, R);
    for (int r = 0; r < R; ++r)
      if (!hidden[r] || !out[r]) throw ConfigErr("null argument");
    CK(cudaSetDevice(hs[0]->cfg.device));
    group_forward(hs, R, hidden, T, out, (cudaStream_t)stream, false);
  });
}

// Training step of an emulated group: forward_train + expert-FFN backward of every rank, with
// the backward's two row exchanges as peer stores (combine-backward kernel -> owners' dYbuf,
// dgrad-2 epilogue -> sources' dXsrc), phase by phase.
cl_status cl_moe_ep_group_train_step(cl_moe* const* hs, int32_t R, const void* const* hidden, const int64_t* T,
                                     void* const* out, const void* const* d_out, void* const* d_hidden,
                                     float* const* d_combine_w, float* const* dw_in, float* const* dw_out,
                                     void* stream) {
  if (!hs || R < 1 || !hidden || !T || !out || !d_out || !d_hidden || !d_combine_w || !dw_in || !dw_out)
    return CL_ERR_CONFIG;
  for (int r = 0; r < R; ++r)
    if (!hs[r]) return CL_ERR_CONFIG;
  return guarded(hs[0], [&] {
    group_check(hs, R);
    for (int r = 0; r < R; ++r) {
      if (!hidden[r] || !out[r] || !d_out[r] || !d_hidden[r] || !d_combine_w[r] || !dw_in[r] || !dw_out[r])
        throw ConfigErr("null argument");
      if (hs[r]->precision != CL_MOE_BF16) throw ConfigErr("training runs in bf16");
    }
    CK(cudaSetDevice(hs[0]->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    group_forward(hs, R, hidden, T, out, st, true);
    std::vector<BwdArgs> a(R);
    for (int r = 0; r < R; ++r) {
      bwd_check(hs[r]);
      a[r] = BwdArgs{d_out[r], d_hidden[r], d_combine_w[r], dw_in[r], dw_out[r], nullptr, 0.0f, 0.0f};
    }
    for (int r = 0; r < R; ++r) bwd_phase_a(hs[r], a[r], st);
    for (int r = 0; r < R; ++r) bwd_phase_b(hs[r], a[r], st);
    for (int r = 0; r < R; ++r) bwd_phase_c(hs[r], a[r], st);
    for (int r = 0; r < R; ++r) bwd_phase_d(hs[r], a[r], st);
  });
}

cl_status cl_moe_ep_peer_layout(const int64_t* counts, int32_t R, int32_t N, int32_t rank, int64_t* dispatch_row,
                                int64_t* return_row, int64_t* local_offsets) {
  if (!counts || !dispatch_row || !return_row || !local_offsets || R < 1 || N < R || N % R || rank < 0 || rank >= R)
    return CL_ERR_CONFIG;
  const int NL = N / R;
  for (int g = 0; g < N; ++g) dispatch_row[g] = ep_piece_row(counts, R, N, g / NL, g % NL, rank);
  for (int e = 0; e < NL; ++e)
    for (int s = 0; s < R; ++s) return_row[e * R + s] = ep_src_row(counts, N, s, rank * NL + e);
  for (int e = 0; e <= NL; ++e) local_offsets[e] = ep_piece_row(counts, R, N, rank, e, 0);
  return CL_OK;
}

cl_status cl_moe_ep_forward(cl_moe* h, const void* hidden, int64_t T, void* out, const cl_moe_decision* decision,
                            void* stream) {
  return guarded(h, [&] {
    if (!hidden || !out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    run_router(h, hidden, T, (cudaStream_t)stream);
    run_ep(h, hidden, T, out, false, (cudaStream_t)stream);
    export_decision(h, T, decision, (cudaStream_t)stream);
  });
}

cl_status cl_moe_forward_train(cl_moe* h, const void* hidden, int64_t T, void* out, const cl_moe_decision* decision,
                               void* stream) {
  return guarded(h, [&] {
    if (!hidden || !out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    ensure_training(h);
    run_router(h, hidden, T, (cudaStream_t)stream);
    run_forward_train(h, hidden, T, out, (cudaStream_t)stream);
    export_decision(h, T, decision, (cudaStream_t)stream);
  });
}

cl_status cl_moe_backward(cl_moe* h, const void* d_out, void* d_hidden, float* d_combine_w, float* dw_in, float* dw_out,
                          void* stream) {
  return guarded(h, [&] {
    if (!d_out || !d_hidden || !d_combine_w || !dw_in || !dw_out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    run_backward(h, d_out, d_hidden, d_combine_w, dw_in, dw_out, (cudaStream_t)stream);
  });
}

cl_status cl_moe_backward_full(cl_moe* h, const void* d_out, float g_aux, float g_z, void* d_hidden, float* dw_router,
                               float* dw_in, float* dw_out, float* d_combine_w, void* stream) {
  return guarded(h, [&] {
    if (!d_out || !d_hidden || !dw_router || !dw_in || !dw_out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    float* dcw = d_combine_w;
    if (!dcw) {
      if (!h->dcw_scratch) h->dcw_scratch = dalloc<float>(h->cap * h->K);
      dcw = h->dcw_scratch;
    }
    run_backward(h, d_out, d_hidden, dcw, dw_in, dw_out, (cudaStream_t)stream, dw_router, g_aux, g_z);
  });
}

// ---- reference checkpoint format (CLCKPT1, proj/include/compasslab/checkpoint.hpp:4-9) ----
// Failures of the create entries (no handle exists yet) are kept per thread.
static thread_local std::string g_create_error;

cl_status cl_moe_create_from_checkpoint(const cl_moe_config* cfg, const char* path, const char* prefix, cl_moe** out) {
  if (!out || !cfg) return CL_ERR_CONFIG;
  *out = nullptr;
  try {
    if (!path) return CL_ERR_CONFIG;
    const std::string pre = prefix ? prefix : "";
    const Checkpoint c = Checkpoint::load(path);
    const int ep = cfg->ep_size <= 0 ? 1 : cfg->ep_size;
    if (cfg->n_experts < 1 || cfg->n_experts % ep) {
      g_create_error = "n_experts must be a positive multiple of ep_size";
      return CL_ERR_CONFIG;
    }
    const int64_t d = cfg->d_model, N = cfg->n_experts, f = cfg->d_ff, NL = N / ep, e0 = cfg->ep_rank * NL;
    const std::vector<float> wr = c.get(pre + "router", {d, N});
    std::vector<float> w_in((size_t)NL * d * 2 * f), w_out((size_t)NL * f * d);
    for (int64_t e = 0; e < NL; ++e) {
      const std::string ex = pre + "experts." + std::to_string(e0 + e) + ".";
      std::memcpy(w_in.data() + e * d * 2 * f, c.get(ex + "w_in", {d, 2 * f}).data(), sizeof(float) * d * 2 * f);
      std::memcpy(w_out.data() + e * f * d, c.get(ex + "w_out", {f, d}).data(), sizeof(float) * f * d);
    }
    return cl_moe_create(cfg, wr.data(), w_in.data(), w_out.data(), out);
  } catch (const std::exception& e) {
    g_create_error = std::string("cl_moe_create_from_checkpoint: ") + e.what();
    return CL_ERR_RUN;
  }
}

cl_status cl_moe_save_checkpoint(cl_moe* h, const char* path, const char* prefix) {
  return guarded(h, [&] {
    if (!path) throw ConfigErr("path is null");
    CK(cudaSetDevice(h->cfg.device));
    const std::string pre = prefix ? prefix : "";
    const int64_t d = h->d, N = h->N, f = h->f, NL = h->n_local;
    std::vector<float> wr(d * N), win((size_t)NL * d * 2 * f), wout((size_t)NL * f * d);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(wr.data(), h->wr, sizeof(float) * d * N, cudaMemcpyDeviceToHost));
    // packed bf16 -> reference layouts on device, then widen on the host
    __nv_bfloat16* tmp = dalloc<__nv_bfloat16>((size_t)d * 2 * f);
    std::vector<uint16_t> hb((size_t)d * 2 * f);
    auto widen = [&](const std::vector<uint16_t>& src, float* dst, size_t n) {
      for (size_t i = 0; i < n; ++i) {
        const uint32_t u = static_cast<uint32_t>(src[i]) << 16;
        std::memcpy(dst + i, &u, 4);
      }
    };
    for (int64_t e = 0; e < NL; ++e) {
      transpose_weight_kernel<true><<<dim3((unsigned)(2 * f / 32), (unsigned)(d / 32)), 256>>>(
          h->win + (size_t)e * 2 * f * d, (int)(2 * f), (int)d, (int)f, tmp);
      CK(cudaGetLastError());
      CK(cudaMemcpy(hb.data(), tmp, sizeof(uint16_t) * d * 2 * f, cudaMemcpyDeviceToHost));
      widen(hb, win.data() + e * d * 2 * f, (size_t)d * 2 * f);
      transpose_weight_kernel<false><<<dim3((unsigned)(d / 32), (unsigned)(f / 32)), 256>>>(
          h->wout + (size_t)e * d * f, (int)d, (int)f, (int)f, tmp);
      CK(cudaGetLastError());
      CK(cudaMemcpy(hb.data(), tmp, sizeof(uint16_t) * f * d, cudaMemcpyDeviceToHost));
      widen(hb, wout.data() + e * f * d, (size_t)f * d);
    }
    cudaFree(tmp);
    std::map<std::string, std::pair<std::vector<int64_t>, const float*>> ts;
    ts[pre + "router"] = {{d, N}, wr.data()};
    for (int64_t e = 0; e < NL; ++e) {
      const std::string ex = pre + "experts." + std::to_string(h->e0 + e) + ".";
      ts[ex + "w_in"] = {{d, 2 * f}, win.data() + e * d * 2 * f};
      ts[ex + "w_out"] = {{f, d}, wout.data() + e * f * d};
    }
    Checkpoint::save(path, ts);
  });
}

// ---- balance_calibration ----
cl_status cl_moe_balance_calibration(cl_moe* h, const void* base, int64_t T_base, const void* pool, int64_t P,
                                     int64_t tau, int64_t* selected, int64_t* n_selected, int64_t* final_counts,
                                     void* stream) {
  return guarded(h, [&] {
    if (tau < 1) throw ConfigErr("balance_calibration: tau must be >= 1");
    if (!selected || !n_selected || !final_counts || (P > 0 && !pool)) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    const int64_t N = h->N, K = h->K, d = h->d;
    std::vector<int64_t> cnt(N, 0);
    std::vector<int32_t> c32(N);
    if (base && T_base > 0) {
      for (int64_t t0 = 0; t0 < T_base; t0 += h->cap) {
        const int64_t t = std::min<int64_t>(h->cap, T_base - t0);
        run_router(h, static_cast<const __nv_bfloat16*>(base) + t0 * d, t, st);
        CK(cudaMemcpyAsync(c32.data(), h->rb.counts, sizeof(int32_t) * N, cudaMemcpyDeviceToHost, st));
        CK(cudaStreamSynchronize(st));
        for (int64_t e = 0; e < N; ++e) cnt[e] += c32[e];
      }
    }
    // pre-route the pool (router only) and greedily take tokens routed to a deficit expert
    std::vector<int32_t> idx;
    int64_t ns = 0;
    auto deficit = [&]() {
      for (int64_t e = 0; e < N; ++e)
        if (cnt[e] < tau) return true;
      return false;
    };
    for (int64_t t0 = 0; t0 < P && deficit(); t0 += h->cap) {
      const int64_t t = std::min<int64_t>(h->cap, P - t0);
      run_router(h, static_cast<const __nv_bfloat16*>(pool) + t0 * d, t, st);
      idx.resize(t * K);
      CK(cudaMemcpyAsync(idx.data(), h->rb.topk_idx, sizeof(int32_t) * t * K, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
      for (int64_t j = 0; j < t && deficit(); ++j) {
        bool useful = false;
        for (int64_t k = 0; k < K; ++k) useful |= cnt[idx[j * K + k]] < tau;
        if (!useful) continue;
        for (int64_t k = 0; k < K; ++k) cnt[idx[j * K + k]] += 1;
        selected[ns++] = t0 + j;
      }
    }
    *n_selected = ns;
    for (int64_t e = 0; e < N; ++e) final_counts[e] = cnt[e];
    for (int64_t e = 0; e < N; ++e)
      if (cnt[e] < tau)
        throw RunErr(fmt("balance_calibration: token pool exhausted with expert %lld at %lld < tau=%lld", (long long)e,
                         (long long)cnt[e], (long long)tau));
  });
}

cl_status cl_moe_ep_layout(const int64_t* counts, int32_t R, int32_t N, int32_t rank, int64_t* local_offsets,
                           int64_t* recv_piece, int64_t* recv_total) {
  if (!counts || !local_offsets || !recv_piece || R < 1 || N < R || N % R || rank < 0 || rank >= R)
    return CL_ERR_CONFIG;
  const int64_t t = ep_layout(counts, R, N, rank, local_offsets, recv_piece);
  if (recv_total) *recv_total = t;
  return CL_OK;
}


const char* cl_moe_version(void) { return "0.1.0-sm100a"; }

const char* cl_moe_last_error(const cl_moe* h) { return h == nullptr ? g_create_error.c_str() : h->last_error.c_str(); }

static cl_status create_common(const cl_moe_config* cfg, cl_moe** out, const float* w_router, const float* w_in,
                               const float* w_out, bool synthetic, uint64_t seed) {
  if (out == nullptr) return CL_ERR_CONFIG;
  *out = nullptr;
  cl_moe* h = new cl_moe();
  const cl_status st = guarded(h, [&] {
    init_handle(h, cfg);
    const int64_t d = h->d, f = h->f, N = h->N;
    const float sd = static_cast<float>(1.0 / std::sqrt(static_cast<double>(d)));
    const float sf = static_cast<float>(1.0 / std::sqrt(static_cast<double>(f)));
    if (synthetic) {
      synth_f32_kernel<<<grid_for(d * N), 256>>>(split_seed(seed, 2), d * N, sd, h->wr);
      for (int el = 0; el < h->n_local; ++el) {
        const int e = h->e0 + el;
        synth_pack_win_kernel<<<grid_for(2 * f * d), 256>>>(split_seed(seed, 16 + e), (int)d, (int)f, sd,
                                                            h->win + (size_t)el * 2 * f * d);
        synth_pack_wout_kernel<<<grid_for(d * f), 256>>>(split_seed(seed, 16 + N + e), (int)d, (int)f, sf,
                                                         h->wout + (size_t)el * d * f);
      }
      CK(cudaGetLastError());
    } else {
      if (!w_router || !w_in || !w_out) throw ConfigErr("weights are null");
      CK(cudaMemcpy(h->wr, w_router, sizeof(float) * d * N, cudaMemcpyHostToDevice));
      float* tmp = dalloc<float>(2 * f * d);
      for (int el = 0; el < h->n_local; ++el) {
        CK(cudaMemcpy(tmp, w_in + (size_t)el * d * 2 * f, sizeof(float) * d * 2 * f, cudaMemcpyHostToDevice));
        pack_transpose_kernel<true><<<dim3((unsigned)(2 * f / 32), (unsigned)((d + 31) / 32)), dim3(32, 8)>>>(
            tmp, (int)d, (int)(2 * f), (int)f, h->win + (size_t)el * 2 * f * d);
        CK(cudaGetLastError());
        CK(cudaMemcpy(tmp, w_out + (size_t)el * f * d, sizeof(float) * f * d, cudaMemcpyHostToDevice));
        pack_transpose_kernel<false><<<dim3((unsigned)(d / 32), (unsigned)((f + 31) / 32)), dim3(32, 8)>>>(
            tmp, (int)f, (int)d, (int)f, h->wout + (size_t)el * d * f);
        CK(cudaGetLastError());
      }
      CK(cudaDeviceSynchronize());
      cudaFree(tmp);
    }
    widen_router_kernel<<<grid_for(d * N), 256>>>(h->wr, (int)d, (int)N, h->wr64);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    build_maps(h, false);
  });
  if (st != CL_OK) {
    g_create_error = h->last_error;
    delete h;
    return st;
  }
  *out = h;
  return CL_OK;
}

cl_status cl_moe_create(const cl_moe_config* cfg, const float* w_router, const float* w_in, const float* w_out,
                        cl_moe** out) {
  return create_common(cfg, out, w_router, w_in, w_out, false, 0);
}

cl_status cl_moe_create_synthetic(const cl_moe_config* cfg, uint64_t seed, cl_moe** out) {
  return create_common(cfg, out, nullptr, nullptr, nullptr, true, seed);
}

void cl_moe_destroy(cl_moe* h) {
  if (h) {
    cudaSetDevice(h->cfg.device);
    cudaDeviceSynchronize();
  }
  delete h;
}

cl_status cl_moe_synthetic_tokens_shifted(cl_moe* h, uint64_t seed, int64_t T, float shift, void* x, void* stream) {
  return guarded(h, [&] {
    if (!x || T < 1) throw ConfigErr("bad arguments");
    CK(cudaSetDevice(h->cfg.device));
    synth_bf16_kernel<<<grid_for(T * h->d), 256, 0, (cudaStream_t)stream>>>(split_seed(seed, 1), T * h->d, 1.0f,
                                                                             static_cast<__nv_bfloat16*>(x), shift);
    CK(cudaGetLastError());
  });
}

cl_status cl_moe_synthetic_tokens(cl_moe* h, uint64_t seed, int64_t T, void* x, void* stream) {
  return cl_moe_synthetic_tokens_shifted(h, seed, T, 0.0f, x, stream);
}

cl_status cl_moe_synthetic_skew(cl_moe* h, double gamma) {
  return guarded(h, [&] {
    CK(cudaSetDevice(h->cfg.device));
    const int64_t d = h->d, N = h->N;
    std::vector<float> wr(d * N), add(N);
    for (int64_t i = 0; i < N; ++i)
      add[i] = static_cast<float>(gamma * std::log(1.0 / std::pow(static_cast<double>(i + 1), 1.2)) /
                                  static_cast<double>(d));
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(wr.data(), h->wr, sizeof(float) * d * N, cudaMemcpyDeviceToHost));
    for (int64_t l = 0; l < d; ++l)
      for (int64_t i = 0; i < N; ++i) wr[l * N + i] = wr[l * N + i] + add[i];
    CK(cudaMemcpy(h->wr, wr.data(), sizeof(float) * d * N, cudaMemcpyHostToDevice));
    widen_router_kernel<<<grid_for(d * N), 256>>>(h->wr, (int)d, (int)N, h->wr64);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
  });
}

cl_status cl_moe_route_tokens(cl_moe* h, const void* hidden, int64_t T, const cl_moe_decision* out, void* stream) {
  return guarded(h, [&] {
    if (!hidden) throw ConfigErr("hidden is null");
    CK(cudaSetDevice(h->cfg.device));
    run_router(h, hidden, T, (cudaStream_t)stream);
    export_decision(h, T, out, (cudaStream_t)stream);
  });
}

cl_status cl_moe_moe_forward(cl_moe* h, const void* hidden, int64_t T, const int32_t* topk_idx,
                             const float* combine_weights, void* out, void* stream) {
  return guarded(h, [&] {
    if (!hidden || !topk_idx || !combine_weights || !out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    plan_from_decision(h, topk_idx, combine_weights, T, (cudaStream_t)stream);
    run_experts(h, hidden, T, out, false, (cudaStream_t)stream);
  });
}

cl_status cl_moe_forward(cl_moe* h, const void* hidden, int64_t T, void* out, const cl_moe_decision* decision,
                         void* stream) {
  return guarded(h, [&] {
    if (!hidden || !out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    run_router(h, hidden, T, (cudaStream_t)stream);
    run_experts(h, hidden, T, out, false, (cudaStream_t)stream);
    export_decision(h, T, decision, (cudaStream_t)stream);
  });
}

static void host_enqueue(cl_moe* h, const void* hidden_host, int64_t T, void* out_host, int32_t io_dtype) {
  if (!hidden_host || !out_host) throw ConfigErr("null argument");
  if (io_dtype != CL_MOE_IO_BF16 && io_dtype != CL_MOE_IO_F32) throw ConfigErr("io_dtype must be BF16 or F32");
  if (T < 1) throw RunErr("moe_forward: B must be >= 1");
  if (T > h->cap) throw ConfigErr("T exceeds max_tokens");
  CK(cudaSetDevice(h->cfg.device));
  auto& sl = h->slot[h->next_slot];
  h->next_slot ^= 1;
  const bool f32 = io_dtype == CL_MOE_IO_F32;
  if (!sl.x) {
    sl.x = dalloc<__nv_bfloat16>(h->cap * h->d);
    sl.out = dalloc<float>(h->cap * h->d);
  }
  if (f32 && !sl.xf) sl.xf = dalloc<float>(h->cap * h->d);
  const int64_t n = T * h->d;
  cudaStream_t st = h->own_stream;
  // H2D may overwrite the slot's input once the compute of its previous use has consumed it
  if (sl.used) CK(cudaStreamWaitEvent(h->s_h2d, sl.done, 0));
  if (f32) CK(cudaMemcpyAsync(sl.xf, hidden_host, n * 4, cudaMemcpyHostToDevice, h->s_h2d));
  else CK(cudaMemcpyAsync(sl.x, hidden_host, n * 2, cudaMemcpyHostToDevice, h->s_h2d));
  CK(cudaEventRecord(sl.h2d, h->s_h2d));
  // compute: after this slot's H2D, and after the D2H of the slot's previous output
  CK(cudaStreamWaitEvent(st, sl.h2d, 0));
  if (sl.used) CK(cudaStreamWaitEvent(st, sl.d2h, 0));
  if (f32) {
    f32_to_bf16_kernel<<<grid_for(n), 256, 0, st>>>(sl.xf, n, static_cast<__nv_bfloat16*>(sl.x));
    CK(cudaGetLastError());
  }
  run_router(h, sl.x, T, st);
  run_experts(h, sl.x, T, sl.out, f32, st);
  CK(cudaEventRecord(sl.done, st));
  CK(cudaStreamWaitEvent(h->s_d2h, sl.done, 0));
  CK(cudaMemcpyAsync(out_host, sl.out, n * (f32 ? 4 : 2), cudaMemcpyDeviceToHost, h->s_d2h));
  CK(cudaEventRecord(sl.d2h, h->s_d2h));
  sl.used = true;
}

static void host_wait(cl_moe* h) {
  CK(cudaSetDevice(h->cfg.device));
  CK(cudaStreamSynchronize(h->s_d2h));
  CK(cudaStreamSynchronize(h->own_stream));
  int flag = 0;
  CK(cudaMemcpy(&flag, h->rb.finite_flag, sizeof(int), cudaMemcpyDeviceToHost));
  if (flag) {
    CK(cudaMemset(h->rb.finite_flag, 0, sizeof(int)));
    throw RunErr("non-finite value produced by op 'moe_forward'");
  }
}

cl_status cl_moe_forward_host(cl_moe* h, const void* hidden_host, int64_t T, void* out_host, int32_t io_dtype) {
  return guarded(h, [&] {
    host_enqueue(h, hidden_host, T, out_host, io_dtype);
    host_wait(h);
  });
}

cl_status cl_moe_forward_host_async(cl_moe* h, const void* hidden_host, int64_t T, void* out_host,
                                    int32_t io_dtype) {
  return guarded(h, [&] { host_enqueue(h, hidden_host, T, out_host, io_dtype); });
}

cl_status cl_moe_host_wait(cl_moe* h) {
  return guarded(h, [&] { host_wait(h); });
}

cl_status cl_moe_sync(cl_moe* h, void* stream) {
  return guarded(h, [&] {
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaStreamSynchronize((cudaStream_t)stream));
    int flag = 0;
    CK(cudaMemcpy(&flag, h->rb.finite_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      CK(cudaMemset(h->rb.finite_flag, 0, sizeof(int)));
      if (flag & 2) throw RunErr("expert-parallel receive buffer overflow");
      throw RunErr("non-finite value produced by op 'moe_forward'");
    }
  });
}

cl_status cl_moe_stage_buffers(cl_moe* h, cl_moe_stage_view* v) {
  return guarded(h, [&] {
    if (!v) throw ConfigErr("view is null");
    v->offsets = h->rb.offsets;
    v->perm = h->perm;
    v->inv = h->inv;
    v->row_weight = h->row_w;
    v->x_perm = h->xperm;
    v->act = h->act;
    v->y = h->y;
    v->rows = h->last_rows;
  });
}

cl_status cl_moe_copy_stage(cl_moe* h, int32_t which, void* dst, int64_t bytes, void* stream) {
  return guarded(h, [&] {
    const void* src = nullptr;
    switch (which) {
      case 0: src = h->rb.offsets; break;
      case 1: src = h->perm; break;
      case 2: src = h->inv; break;
      case 3: src = h->row_w; break;
      case 4: src = h->xperm; break;
      case 5: src = h->act; break;
      case 6: src = h->y; break;
      default: throw ConfigErr("unknown stage buffer");
    }
    if (!dst || bytes < 0) throw ConfigErr("bad destination");
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToDevice, (cudaStream_t)stream));
  });
}

cl_status cl_moe_profile(cl_moe* h, int32_t enable) {
  return guarded(h, [&] {
    h->prof = enable != 0;
    h->prof_used = 0;
  });
}

cl_status cl_moe_profile_read(cl_moe* h, double* stage_ms, int64_t* calls) {
  return guarded(h, [&] {
    CK(cudaSetDevice(h->cfg.device));
    for (int s = 0; s < kStages + kBwdStages; ++s) stage_ms[s] = 0.0;
    calls[0] = calls[1] = 0;
    for (size_t c = 0; c < h->prof_used; ++c) {
      auto& ev = h->prof_sets[c];
      const int kind = h->prof_kind[c];
      const int n = kind == 0 ? kStages : kBwdStages;
      CK(cudaEventSynchronize(ev[n]));
      for (int s = 0; s < n; ++s) {
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ev[s], ev[s + 1]));
        stage_ms[(kind == 0 ? 0 : kStages) + s] += ms;
      }
      calls[kind] += 1;
    }
    h->prof_used = 0;
  });
}

cl_status cl_moe_calibrate(cl_moe* h, const void* hidden, int64_t T, int32_t reset, void* stream) {
  return guarded(h, [&] {
    if (!hidden && T != 0) throw ConfigErr("hidden is null");
    CK(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    if (reset) {
      CK(cudaMemsetAsync(h->calib, 0, sizeof(float) * 2 * h->n_local, st));
      CK(cudaMemsetAsync(h->calib_ch, 0, sizeof(float) * h->d, st));
      CK(cudaMemsetAsync(h->calib_counts, 0, sizeof(long long) * h->N, st));
      CK(cudaMemsetAsync(h->calib_all, 0, sizeof(float) * h->N, st));
    }
    if (T == 0) return;  // empty calibration set: statistics unchanged
    if (T < 0) throw ConfigErr("T must be >= 0");
    col_absmax_kernel<<<dim3((unsigned)((h->d + 255) / 256), (unsigned)((T + 255) / 256)), 256, 0, st>>>(
        static_cast<const __nv_bfloat16*>(hidden), T, (int)h->d, 256, h->calib_ch);
    const int saved = h->precision;
    h->precision = CL_MOE_BF16;
    run_router(h, hidden, T, st);
    if (!h->io_out) h->io_out = dalloc<__nv_bfloat16>(h->cap * h->d);
    run_experts(h, hidden, T, h->io_out, false, st);
    h->precision = saved;
    add_counts_kernel<<<1, 128, 0, st>>>(h->rb.counts, (int)h->N, h->calib_counts);
    const int64_t rows = T * h->K;
    if (h->comm) {
      // expert parallel: GEMM1-input maxima at the source for every global expert (all-reduced
      // over the ranks by quantize_fp8), SwiGLU-output maxima at the owner (receive layout)
      route_absmax_kernel<<<(int)((T + 7) / 8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(hidden), (int)T,
                                                              (int)h->d, (int)h->K, h->rb.topk_idx, h->calib_all);
      segment_absmax_kernel<<<(int)((h->recv_cap + 7) / 8), 256, 0, st>>>(h->act_recv, (int)h->f, h->ep_off_dev,
                                                                           h->n_local, h->calib + h->n_local);
    } else {
      segment_absmax_kernel<<<(int)((rows + 7) / 8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(h->xperm),
                                                                   (int)h->d, h->rb.offsets, h->n_local, h->calib);
      segment_absmax_kernel<<<(int)((rows + 7) / 8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(h->act), (int)h->f,
                                                                   h->rb.offsets, h->n_local, h->calib + h->n_local);
    }
    CK(cudaGetLastError());
  });
}

cl_status cl_moe_calibration_stats(cl_moe* h, int64_t* counts, float* x_max, float* mid_max, float* ch_max) {
  return guarded(h, [&] {
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaDeviceSynchronize());
    if (counts) CK(cudaMemcpy(counts, h->calib_counts, sizeof(int64_t) * h->N, cudaMemcpyDeviceToHost));
    if (x_max) CK(cudaMemcpy(x_max, h->calib, sizeof(float) * h->n_local, cudaMemcpyDeviceToHost));
    if (mid_max) CK(cudaMemcpy(mid_max, h->calib + h->n_local, sizeof(float) * h->n_local, cudaMemcpyDeviceToHost));
    if (ch_max) CK(cudaMemcpy(ch_max, h->calib_ch, sizeof(float) * h->d, cudaMemcpyDeviceToHost));
  });
}

cl_status cl_moe_compute_smoothing(cl_moe* h, float alpha, float* s_out) {
  return guarded(h, [&] {
    if (!s_out) throw ConfigErr("s_out is null");
    if (!(alpha >= 0.0f && alpha <= 1.0f)) throw ConfigErr("alpha must be in [0, 1]");
    if (h->cfg.ep_size > 1) throw ConfigErr("compute_smoothing needs every expert's weights (ep_size == 1)");
    CK(cudaSetDevice(h->cfg.device));
    const int64_t d = h->d, N = h->N;
    // joint per-input-channel weight maximum over every expert's W_in and the router
    float* wmax = h->smooth;
    CK(cudaMemset(wmax, 0, sizeof(float) * d));
    const int64_t rows = (int64_t)h->n_local * 2 * h->f;
    col_absmax_kernel<<<dim3((unsigned)((d + 255) / 256), (unsigned)((rows + 1023) / 1024)), 256>>>(h->win, rows, (int)d,
                                                                                                 1024, wmax);
    CK(cudaGetLastError());
    std::vector<float> xm(d), wm(d), wr(d * N);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(xm.data(), h->calib_ch, sizeof(float) * d, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(wm.data(), wmax, sizeof(float) * d, cudaMemcpyDeviceToHost));
    CK(cudaMemcpy(wr.data(), h->wr, sizeof(float) * d * N, cudaMemcpyDeviceToHost));
    for (int64_t l = 0; l < d; ++l) {
      float m = wm[l];
      for (int64_t i = 0; i < N; ++i) m = std::max(m, std::fabs(wr[l * N + i]));
      // s_j = max|X_j|^alpha / max|W_j|^(1-alpha); zero-max channels get s = 1
      s_out[l] = (xm[l] > 0.0f && m > 0.0f)
                     ? static_cast<float>(std::pow(static_cast<double>(xm[l]), alpha) /
                                          std::pow(static_cast<double>(m), 1.0 - alpha))
                     : 1.0f;
    }
  });
}

cl_status cl_moe_fold_smoothing(cl_moe* h, const float* s) {
  return guarded(h, [&] {
    if (!s) throw ConfigErr("s is null");
    const int64_t d = h->d, N = h->N;
    for (int64_t l = 0; l < d; ++l)
      if (!(s[l] > 0.0f) || !std::isfinite(s[l])) throw ConfigErr("smoothing factors must be finite and > 0");
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaMemcpy(h->smooth, s, sizeof(float) * d, cudaMemcpyHostToDevice));
    const int64_t n = (int64_t)h->n_local * 2 * h->f * d;
    scale_cols_bf16_kernel<<<grid_for(n), 256>>>(h->win, n, (int)d, h->smooth);
    scale_rows_f32_kernel<<<(int)((d * N + 255) / 256), 256>>>(h->wr, (int)d, (int)N, h->smooth);
    widen_router_kernel<<<grid_for(d * N), 256>>>(h->wr, (int)d, (int)N, h->wr64);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    // derived copies are stale now
    h->fp8_ready = false;
    h->precision = CL_MOE_BF16;
    h->train_ready = false;
    CK(cudaMemset(h->calib, 0, sizeof(float) * 2 * h->n_local));
    CK(cudaMemset(h->calib_ch, 0, sizeof(float) * d));
  });
}

cl_status cl_moe_quantize_fp8(cl_moe* h, const float* act_scale_in, const float* act_scale_mid) {
  return guarded(h, [&] {
    CK(cudaSetDevice(h->cfg.device));
    ensure_fp8_storage(h);
    const int N = static_cast<int>(h->N), NL = h->n_local;
    const bool ep = h->cfg.ep_size > 1;
    std::vector<float> sin_all(N), smid(NL);
    if (act_scale_in && act_scale_mid) {
      std::copy(act_scale_in, act_scale_in + N, sin_all.begin());  // [N]: every expert's (EP: global table)
      std::copy(act_scale_mid, act_scale_mid + NL, smid.begin());
    } else {
      std::vector<float> c(2 * NL), call(N);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(c.data(), h->calib, sizeof(float) * 2 * NL, cudaMemcpyDeviceToHost));
      if (ep && !h->comm) throw ConfigErr("expert-parallel calibration needs cl_moe_ep_init (or explicit scales)");
      if (h->comm) {  // calibrated through the EP path: source-side maxima of every global expert
        cudaStream_t st = nullptr;
        NCK(NcclApi::get().AllReduce(h->calib_all, h->calib_all, (size_t)N, NcclApi::kFloat32, NcclApi::kMax, h->comm,
                                     st));
        CK(cudaStreamSynchronize(st));
        CK(cudaMemcpy(call.data(), h->calib_all, sizeof(float) * N, cudaMemcpyDeviceToHost));
      } else {
        std::copy(c.begin(), c.begin() + NL, call.begin());
      }
      for (int g = 0; g < N; ++g) {
        if (!(call[g] > 0.0f)) throw RunErr(fmt("quantize_model: missing calibration for expert %d", g));
        sin_all[g] = call[g] / 448.0f;
      }
      for (int e = 0; e < NL; ++e) {
        if (!(c[NL + e] > 0.0f)) throw RunErr(fmt("quantize_model: missing calibration for expert %d", h->e0 + e));
        smid[e] = c[NL + e] / 448.0f;
      }
    }
    for (int g = 0; g < N; ++g)
      if (!(sin_all[g] > 0.0f)) throw ConfigErr("activation scales must be > 0");
    for (int e = 0; e < NL; ++e)
      if (!(smid[e] > 0.0f)) throw ConfigErr("activation scales must be > 0");
    CK(cudaMemcpy(h->sx_in_all, sin_all.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->sx_in, sin_all.data() + h->e0, sizeof(float) * NL, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->sx_mid, smid.data(), sizeof(float) * NL, cudaMemcpyHostToDevice));
    const int64_t r1 = (int64_t)NL * 2 * h->f, r2 = (int64_t)NL * h->d;
    quantize_rows_e4m3_kernel<<<(int)((r1 + 7) / 8), 256>>>(h->win, r1, (int)h->d, h->win8, h->ws_in);
    quantize_rows_e4m3_kernel<<<(int)((r2 + 7) / 8), 256>>>(h->wout, r2, (int)h->f, h->wout8, h->ws_out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    h->fp8_ready = true;
    h->precision = CL_MOE_FP8_E4M3;
  });
}

cl_status cl_moe_set_precision(cl_moe* h, int32_t precision) {
  return guarded(h, [&] {
    if (precision != CL_MOE_BF16 && precision != CL_MOE_FP8_E4M3) throw ConfigErr("unknown precision");
    if (precision == CL_MOE_FP8_E4M3 && !h->fp8_ready) throw ConfigErr("FP8 scheme not quantized yet");
    h->precision = precision;
  });
}

cl_status cl_moe_get_fp8_scales(cl_moe* h, float* act_in, float* act_mid, float* w_in_scale, float* w_out_scale) {
  return guarded(h, [&] {
    if (!h->fp8_ready) throw ConfigErr("FP8 scheme not quantized yet");
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaDeviceSynchronize());
    if (act_in) CK(cudaMemcpy(act_in, h->sx_in, sizeof(float) * h->n_local, cudaMemcpyDeviceToHost));
    if (act_mid) CK(cudaMemcpy(act_mid, h->sx_mid, sizeof(float) * h->n_local, cudaMemcpyDeviceToHost));
    if (w_in_scale) CK(cudaMemcpy(w_in_scale, h->ws_in, sizeof(float) * h->n_local * 2 * h->f, cudaMemcpyDeviceToHost));
    if (w_out_scale) CK(cudaMemcpy(w_out_scale, h->ws_out, sizeof(float) * h->n_local * h->d, cudaMemcpyDeviceToHost));
  });
}

}  // extern "C"
