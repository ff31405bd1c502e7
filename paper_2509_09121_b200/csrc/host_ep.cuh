// Expert parallelism: the NCCL row exchange and the NVLink peer-memory transport (ep.cuh).
// Host side of libcompass_moe.so, included once, in order, by capi.cu (a single translation
// unit; the helpers live in an anonymous namespace).
#pragma once

namespace {

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

// Bounded wait for `st` on an expert-parallel handle (the reference's error contract,
// capi.cpp:57-63: a failure returns CL_ERR_RUN, it does not hang the caller). Polls the stream and
// ncclCommGetAsyncError; on an NCCL async error, or when the stream has not drained within
// CL_MOE_EP_TIMEOUT_S seconds (default 600; a peer rank died or stalled), the communicator is
// aborted (ncclCommAbort) and the call fails with CL_ERR_RUN; every later expert-parallel call on
// the handle fails the same way until cl_moe_ep_init creates a new communicator.
double ep_timeout_s() {
  static const double t = [] {
    const char* e = std::getenv("CL_MOE_EP_TIMEOUT_S");
    return e ? std::atof(e) : 600.0;
  }();
  return t;
}

void ep_abort(cl_moe* h, const std::string& why) {
  if (h->comm) NcclApi::get().CommAbort(h->comm);
  h->comm = nullptr;
  h->ep_abort_reason = why;
  throw RunErr(why);
}

void ep_wait(cl_moe* h, cudaStream_t st, const char* what) {
  if (!h->comm) {
    CK(cudaStreamSynchronize(st));
    return;
  }
  NcclApi& nc = NcclApi::get();
  const auto t0 = std::chrono::steady_clock::now();
  for (int spins = 0;; ++spins) {
    const cudaError_t e = cudaStreamQuery(st);
    if (e == cudaSuccess) return;
    if (e != cudaErrorNotReady) CK(e);
    int aerr = 0;
    const int qr = nc.CommGetAsyncError(h->comm, &aerr);
    if (qr != 0 || aerr != 0)
      ep_abort(h, fmt("expert-parallel %s: NCCL async error (%s); communicator aborted", what,
                      nc.GetErrorString(qr != 0 ? qr : aerr)));
    const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    if (el > ep_timeout_s())
      ep_abort(h, fmt("expert-parallel %s timed out after %.0f s (a peer rank failed or stalled); communicator "
                      "aborted", what, el));
    if (spins > 64) std::this_thread::sleep_for(std::chrono::microseconds(200));
  }
}

// Test hook (CL_MOE_EP_TEST_STALL_MS): a kernel that spins that long at the end of an expert-
// parallel forward, after its collectives — a stand-in for a stalled peer in the single-GPU test of
// the timeout path (tests/test_gpu_ep.py).
__global__ void ep_stall_kernel(long long ns) {
  const long long t0 = clock64();
  long long now = t0;
  while (now - t0 < ns) {  // ~1 cycle per ns at ~1-2 GHz; the exact length does not matter
    __nanosleep(1000);
    now = clock64();
  }
}
void ep_test_stall(cudaStream_t st) {
  static const long long ms = [] {
    const char* e = std::getenv("CL_MOE_EP_TEST_STALL_MS");
    return e ? std::atoll(e) : 0LL;
  }();
  if (ms > 0) ep_stall_kernel<<<1, 1, 0, st>>>(ms * 1000000LL * 2);
}

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
  if (!h->comm && !h->ep_abort_reason.empty()) throw RunErr(h->ep_abort_reason);
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
  ep_wait(h, st, "counts exchange");
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
  ep_test_stall(st);
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
  h->last_dense = false;
  h->last_xperm_padded = false;
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
  h->arrive = dalloc<uint32_t>(h->n_local);
  h->arrive_tgt = dalloc<uint32_t>(h->n_local);
  CK(cudaMemset(h->arrive, 0, sizeof(uint32_t) * h->n_local));
  CK(cudaMemset(h->arrive_tgt, 0, sizeof(uint32_t) * h->n_local));
  h->peer_a_dev = dalloc<char*>(R);
  h->expert_arrive = dalloc<uint32_t*>(h->N);
}

// Dispatch overlapped with the owners' GEMM1 (CL_MOE_EP_OVERLAP=1, read per call): no barrier
// between dispatch and GEMM1; the owner's GEMM1 producer waits on per-expert arrival counters.
bool ep_overlap() {
  const char* e = std::getenv("CL_MOE_EP_OVERLAP");
  return e && e[0] == '1';
}

void ep_peer_layout(cl_moe* h, cudaStream_t st) {
  const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
  const int64_t xrb = h->d * (h->precision == CL_MOE_FP8_E4M3 ? 1 : 2);
  ep_peer_layout_kernel<<<h->n_local * R + 1, 256, 0, st>>>(h->ep_counts_dev, R, (int)h->N, h->cfg.ep_rank, h->recv_cap,
                                                             xrb, h->d * 2, h->peer_x_dev, h->peer_y_dev, h->peer_w_dev,
                                                             h->expert_dst, h->expert_dst_w, h->ep_off_dev, h->row_ptr,
                                                             h->rb.finite_flag, h->peer_dy_dev, h->peer_dx_dev,
                                                             h->expert_dst_dy, h->row_ptr_dx,
                                                             ep_overlap() ? h->peer_a_dev : nullptr, h->expert_arrive,
                                                             h->arrive_tgt, (int)h->K);
  CK(cudaGetLastError());
}

void ep_peer_dispatch(cl_moe* h, const void* x, int64_t T, cudaStream_t st) {
  const int blocks = static_cast<int>((T + 7) / 8);
  if (h->precision == CL_MOE_FP8_E4M3)
    dispatch_kernel<true><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, (int)h->N,
                                                  (int)h->K, h->tpc_cur, h->rb, h->rb.topk_idx, h->rb.combine_w,
                                                  h->xperm, h->perm, h->inv, h->row_w, h->sx_in_all, h->expert_dst,
                                                  h->expert_dst_w, ep_overlap() ? h->expert_arrive : nullptr);
  else
    dispatch_kernel<false><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, (int)h->N,
                                                   (int)h->K, h->tpc_cur, h->rb, h->rb.topk_idx, h->rb.combine_w,
                                                   h->xperm, h->perm, h->inv, h->row_w, nullptr, h->expert_dst,
                                                   h->expert_dst_w, ep_overlap() ? h->expert_arrive : nullptr);
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
  const bool ov = ep_overlap();
  run_gemms(h, h->ep_off_dev, h->act_recv, h->y_recv, train ? nullptr : h->w_recv, h->mA1e, h->mA2e, h->mA1eq,
            h->mA2eq, st, train ? h->Hbuf : nullptr, h->row_ptr, nullptr, ov ? h->arrive : nullptr,
            ov ? h->arrive_tgt : nullptr);
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
  h->last_dense = false;
  h->last_xperm_padded = false;
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
  // overlap: no barrier — GEMM1 starts on the local rows while the peers' rows stream in, expert by
  // expert (its producer waits on the arrival counters the dispatch kernels bump)
  if (!ep_overlap()) NCK(nc.AllReduce(h->bar_buf, h->bar_buf, 1, NcclApi::kFloat32, NcclApi::kSum, h->comm, st));
  ep_peer_experts(h, st, train);
  NCK(nc.AllReduce(h->bar_buf, h->bar_buf, 1, NcclApi::kFloat32, NcclApi::kSum, h->comm, st));
  ep_test_stall(st);
  ep_peer_combine(h, x, T, out, out_f32, st, train);
}

}  // namespace
