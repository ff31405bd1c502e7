// Training: forward_train and the phased backward (combine-bwd, dgrads, dispatch-bwd, wgrads).
// Host side of libcompass_moe.so, included once, in order, by capi.cu (a single translation
// unit; the helpers live in an anonymous namespace).
#pragma once

namespace {

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
    if (ep && !h->dYbuf) h->dYbuf = dalloc<__nv_bfloat16>(rows * d);  // (single GPU: dY lives in dYT)
    h->dXbuf = dalloc<__nv_bfloat16>(rows * d);
    h->XT = dalloc<__nv_bfloat16>(d * h->rp_cap);
    h->AT = dalloc<__nv_bfloat16>(f * h->rp_cap);
    h->dYT = dalloc<__nv_bfloat16>(d * h->rp_cap);
    h->dHT = dalloc<__nv_bfloat16>(2 * f * h->rp_cap);
    h->poff = dalloc<int32_t>(NL + 1);
    h->kb_off = dalloc<int32_t>(NL + 1);
    for (int v = 0; v < 2; ++v) {
      const uint32_t brow = v == 0 ? 256 : 128;
      if (ep) h->mAdg1[v] = make_map(h->dYbuf, false, d, rows, 128);
      h->mAdg1_ready = ep;
      h->mBdg1[v] = make_map(h->wout_ref, false, d, (uint64_t)NL * f, brow);
      h->mAdg2T[v] = make_map(h->dHT, false, 2 * f, h->rp_cap, 128);  // dH, padded row layout
      h->mA1T[v] = make_map(h->XT, false, d, h->rp_cap, 128);          // X (single-GPU training)
      h->mAdg1T[v] = make_map(h->dYT, false, d, h->rp_cap, 128);       // dY (single-GPU training)
      h->mA2T[v] = make_map(h->AT, false, f, h->rp_cap, 128);          // A (single-GPU training)
      h->mBdg2[v] = make_map(h->win_ref, false, 2 * f, (uint64_t)NL * d, brow);
      // weight-gradient operands, MN-major: boxes of 64 columns x 64 padded rows
      h->mAwo[v] = make_map(h->AT, false, f, h->rp_cap, 64);
      h->mBwo[v] = make_map(h->dYT, false, d, h->rp_cap, 64);
      h->mAwi[v] = make_map(h->XT, false, d, h->rp_cap, 64);
      h->mBwi[v] = make_map(h->dHT, false, 2 * f, h->rp_cap, 64);
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
  // the dispatched rows go straight into the padded row layout the dW_in GEMM reads; GEMM1 reads
  // them there too (GemmArgs::a_poff), so no row-layout copy and no pad pass
  pad_plan_kernel<<<1, 32, 0, st>>>(h->rb.offsets, h->n_local, h->poff, h->kb_off);
  dispatch_kernel<false><<<token_grid(T), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(x), (int)T, (int)h->d, N, (int)h->K,
                                                 tpc, h->rb, h->rb.topk_idx, h->rb.combine_w, h->XT, h->perm,
                                                 h->inv, h->row_w, nullptr, nullptr, nullptr, nullptr, h->poff);
  CK(cudaGetLastError());
  prof_mark(h, 2, st);
  run_gemms(h, h->rb.offsets, h->act, h->y, nullptr, h->mA1T, h->mA2, h->mA1q, h->mA2q, st, h->Hbuf, nullptr,
            nullptr, nullptr, nullptr, h->poff, h->mA2T);
  prof_mark(h, 4, st);
  launch_combine<__nv_bfloat16>(h->y, h->inv, (int)T, (int)h->d, (int)h->K, static_cast<__nv_bfloat16*>(out),
                                h->rb.finite_flag, st, h->rb.combine_w);
  CK(cudaGetLastError());
  prof_mark(h, 5, st);
  h->cur_ev = nullptr;
  h->last_rows = T * h->K;
  h->last_dense = false;
  h->last_xperm_padded = true;
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
  // single GPU: dY rows straight into the padded layout dgrad-1 and dW_out read
  combine_bwd_kernel<<<(int)((rows + 7) / 8), 256, 0, st>>>(static_cast<const __nv_bfloat16*>(a.d_out), h->y, h->perm,
                                                           h->rb.combine_w, (int)rows, (int)d, (int)h->K,
                                                           ep ? dY_src : h->dYT, a.d_cw,
                                                           peer ? h->expert_dst_dy : nullptr, h->rb.topk_idx,
                                                           h->rb.offsets, ep ? nullptr : h->poff);
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
  // dH is written once, in the padded row layout both dW_in and dgrad-2 read (a2.a_poff)
  a1.out = nullptr;
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
  a2.a_poff = h->poff;
  // dY: padded on a single GPU (combine-bwd wrote it there), the receive layout under EP
  if (ep && !h->mAdg1_ready)  // training buffers are laid out once, for the mode of the first call
    throw ConfigErr("expert-parallel training needs cl_moe_ep_init before the handle's first forward_train");
  const CUtensorMap* mA_dg1 = ep ? h->mAdg1 : h->mAdg1T;
  if (!ep) a1.a_poff = h->poff;
  if (v) {
    launch_gemm<2, EPI_SWIGLU_BWD, false, false>(h, mA_dg1[v], h->mBdg1[v], a1, st);
    prof_mark(h, 1, st);
    launch_gemm<2, EPI_ROWSCALE, false, false>(h, h->mAdg2T[v], h->mBdg2[v], a2, st);
  } else {
    launch_gemm<1, EPI_SWIGLU_BWD, false, false>(h, mA_dg1[v], h->mBdg1[v], a1, st);
    prof_mark(h, 1, st);
    launch_gemm<1, EPI_ROWSCALE, false, false>(h, h->mAdg2T[v], h->mBdg2[v], a2, st);
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
  // padded row-major operands of the weight gradients: X and dY copied into the padded row
  // layout; A and dH were written there by the GEMM1 / dgrad-1 epilogues (zero their padding)
  const unsigned pr = static_cast<unsigned>(h->rp_cap / 8);
  if (ep) {  // expert parallel: X and dY arrived in the receive layout
    pad_rows_kernel<<<pr, 256, 0, st>>>(static_cast<const __nv_bfloat16*>(es_x), (int)d, es_off, h->poff, NL, h->XT);
    pad_rows_kernel<<<pr, 256, 0, st>>>(h->dYbuf, (int)d, es_off, h->poff, NL, h->dYT);
  } else {   // single GPU: dispatch and combine-bwd wrote them padded; zero the padding rows only
    zero_pad_rows_kernel<<<dim3(8, (unsigned)NL), 256, 0, st>>>(h->XT, (int)d, es_off, h->poff);
    zero_pad_rows_kernel<<<dim3(8, (unsigned)NL), 256, 0, st>>>(h->dYT, (int)d, es_off, h->poff);
  }
  zero_pad_rows_kernel<<<dim3(8, (unsigned)NL), 256, 0, st>>>(h->AT, (int)f, es_off, h->poff);
  zero_pad_rows_kernel<<<dim3(8, (unsigned)NL), 256, 0, st>>>(h->dHT, (int)(2 * f), es_off, h->poff);
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
