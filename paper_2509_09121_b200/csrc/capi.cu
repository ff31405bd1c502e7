// Host orchestration of the MoE layer behind the C ABI of include/compass_moe.h.
//
// Error convention follows the reference C API (proj/src/capi.cpp:44-68): configuration errors
// -> CL_ERR_CONFIG, anything else (CUDA error, non-finite output, invalid runtime input)
// -> CL_ERR_RUN, message kept on the handle. No CPU fallback exists: without a usable sm_100
// device every entry point fails with CL_ERR_RUN.
//
// This file holds the extern "C" entry points; the orchestration they call is in host_handle.cuh
// (handle state), host_forward.cuh (single-GPU forward), host_ep.cuh (expert parallelism) and
// host_train.cuh (training), included below into this one translation unit.
#include <cuda.h>
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <chrono>
#include <cstdlib>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "compass_moe.h"
#include "grouped_gemm.cuh"
#include "moe_kernels.cuh"
#include "router_cert.cuh"
#include "synth_pack.cuh"
#include "ep.cuh"
#include "bwd_kernels.cuh"
#include "ckpt.hpp"
#include "scheme.hpp"

using namespace cmoe;

#include "host_handle.cuh"
#include "host_forward.cuh"
#include "host_ep.cuh"
#include "host_train.cuh"


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
    h->ep_abort_reason.clear();
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
    constexpr int kB = 6;  // x_recv, y, w_recv, for training dYbuf, dXsrc, and the arrival counters
    void* const own[kB] = {h->x_recv, h->y, h->w_recv, h->dYbuf, h->dXsrc, h->arrive};
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
    ep_wait(h, st, "peer-init handle exchange");
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
    ep_wait(h, st, "peer-init vote");
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
    CK(cudaMemcpy(h->peer_a_dev, peer[5].data(), sizeof(void*) * R, cudaMemcpyHostToDevice));
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
  std::vector<char*> px(R), py(R), pdy(R), pdx(R), pa(R);
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
    pa[r] = reinterpret_cast<char*>(h->arrive);
  }
  for (int r = 0; r < R; ++r) {
    CK(cudaMemcpyAsync(hs[r]->peer_x_dev, px.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_y_dev, py.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_w_dev, pw.data(), sizeof(float*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_dy_dev, pdy.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_dx_dev, pdx.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
    CK(cudaMemcpyAsync(hs[r]->peer_a_dev, pa.data(), sizeof(char*) * R, cudaMemcpyHostToDevice, st));
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
    ExactRoute exact_route(h, decision != nullptr);
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
    ExactRoute exact_route(h, true);
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

// Local expert e's weights in the reference layouts (W_in [d][2f], W_out [f][d], fp32 host; either
// may be null): packed bf16 -> reference order on the device (tmp: d*2f bf16), widened on the host.
static void unpack_expert(cl_moe* h, int64_t e, __nv_bfloat16* tmp, std::vector<uint16_t>& hb, float* w_in,
                          float* w_out) {
  const int64_t d = h->d, f = h->f;
  auto widen = [&](float* dst, size_t n) {
    for (size_t i = 0; i < n; ++i) {
      const uint32_t u = static_cast<uint32_t>(hb[i]) << 16;
      std::memcpy(dst + i, &u, 4);
    }
  };
  hb.resize((size_t)d * 2 * f);
  if (w_in) {
    transpose_weight_kernel<true><<<dim3((unsigned)(2 * f / 32), (unsigned)(d / 32)), 256>>>(
        h->win + (size_t)e * 2 * f * d, (int)(2 * f), (int)d, (int)f, tmp);
    CK(cudaGetLastError());
    CK(cudaMemcpy(hb.data(), tmp, sizeof(uint16_t) * d * 2 * f, cudaMemcpyDeviceToHost));
    widen(w_in, (size_t)d * 2 * f);
  }
  if (w_out) {
    transpose_weight_kernel<false><<<dim3((unsigned)(d / 32), (unsigned)(f / 32)), 256>>>(
        h->wout + (size_t)e * d * f, (int)d, (int)f, (int)f, tmp);
    CK(cudaGetLastError());
    CK(cudaMemcpy(hb.data(), tmp, sizeof(uint16_t) * f * d, cudaMemcpyDeviceToHost));
    widen(w_out, (size_t)f * d);
  }
}

cl_status cl_moe_get_weights(cl_moe* h, float* w_router, int64_t expert, float* w_in, float* w_out) {
  return guarded(h, [&] {
    if ((w_in || w_out) && (expert < 0 || expert >= h->n_local)) throw ConfigErr("expert out of range");
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaDeviceSynchronize());
    if (w_router) CK(cudaMemcpy(w_router, h->wr, sizeof(float) * h->d * h->N, cudaMemcpyDeviceToHost));
    if (w_in || w_out) {
      __nv_bfloat16* tmp = dalloc<__nv_bfloat16>((size_t)h->d * 2 * h->f);
      std::vector<uint16_t> hb;
      try {
        unpack_expert(h, expert, tmp, hb, w_in, w_out);
      } catch (...) {
        cudaFree(tmp);
        throw;
      }
      cudaFree(tmp);
    }
  });
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
    std::vector<uint16_t> hb;
    for (int64_t e = 0; e < NL; ++e) unpack_expert(h, e, tmp, hb, win.data() + e * d * 2 * f, wout.data() + e * f * d);
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
    // pre-routing uses the full-precision router (calibration precedes quantization)
    struct Restore {
      cl_moe* h;
      int p;
      ~Restore() { h->precision = p; }
    } restore{h, h->precision};
    h->precision = CL_MOE_BF16;
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
    h->tau = tau;  // QuantScheme.tau (scheme file)
  });
}

cl_status cl_moe_ep_last_counts(cl_moe* h, int64_t* counts) {
  return guarded(h, [&] {
    if (!counts) throw ConfigErr("counts is null");
    if (!h->ep_counts_dev) throw ConfigErr("no expert-parallel forward has run on this handle");
    CK(cudaSetDevice(h->cfg.device));
    const int R = h->cfg.ep_size <= 0 ? 1 : h->cfg.ep_size;
    std::vector<int32_t> c((size_t)R * h->N);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(c.data(), h->ep_counts_dev, sizeof(int32_t) * c.size(), cudaMemcpyDeviceToHost));
    for (size_t i = 0; i < c.size(); ++i) counts[i] = c[i];
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
    ++h->wr_ver;
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
    ++h->wr_ver;
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
  });
}

cl_status cl_moe_route_tokens(cl_moe* h, const void* hidden, int64_t T, const cl_moe_decision* out, void* stream) {
  return guarded(h, [&] {
    ExactRoute exact_route(h, true);
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
    ExactRoute exact_route(h, decision != nullptr);
    if (!hidden || !out) throw ConfigErr("null argument");
    CK(cudaSetDevice(h->cfg.device));
    run_forward(h, hidden, T, out, false, (cudaStream_t)stream);
    export_decision(h, T, decision, (cudaStream_t)stream);
  });
}

cl_status cl_moe_route_tokens_f32(cl_moe* h, const float* hidden, int64_t T, const cl_moe_decision* out,
                                  void* stream) {
  return guarded(h, [&] {
    ExactRoute exact_route(h, true);
    if (!hidden) throw ConfigErr("hidden is null");
    CK(cudaSetDevice(h->cfg.device));
    run_router(h, hidden, T, (cudaStream_t)stream, true, false, true);
    export_decision(h, T, out, (cudaStream_t)stream);
  });
}

cl_status cl_moe_forward_f32(cl_moe* h, const float* hidden, int64_t T, float* out, const cl_moe_decision* decision,
                             void* stream) {
  return guarded(h, [&] {
    ExactRoute exact_route(h, decision != nullptr);
    if (!hidden || !out) throw ConfigErr("null argument");
    if (T < 1) throw RunErr("moe_forward: B must be >= 1");
    if (T > h->cap) throw ConfigErr(fmt("T=%lld exceeds max_tokens=%lld", (long long)T, (long long)h->cap));
    CK(cudaSetDevice(h->cfg.device));
    cudaStream_t st = (cudaStream_t)stream;
    if (!h->x16) h->x16 = dalloc<__nv_bfloat16>(h->cap * h->d);
    const int64_t n = T * h->d;
    f32_to_bf16_kernel<<<grid_for(n), 256, 0, st>>>(hidden, n, h->x16);  // the expert GEMMs' operand
    CK(cudaGetLastError());
    run_forward(h, h->x16, T, out, true, st, hidden, true);
    export_decision(h, T, decision, st);
  });
}

// The single-GPU forward captured once per (hidden, out, T, precision) into a CUDA graph and
// replayed: the six kernels and two counter memsets go out as one launch.
cl_status cl_moe_forward_graph(cl_moe* h, const void* hidden, int64_t T, void* out, void* stream) {
  return guarded(h, [&] {
    if (!hidden || !out) throw ConfigErr("null argument");
    if (h->comm || h->cfg.ep_size > 1) throw ConfigErr("graph capture covers the single-GPU layer only");
    CK(cudaSetDevice(h->cfg.device));
    cudaGraphExec_t exec = nullptr;
    for (auto& g : h->graphs)
      if (g.x == hidden && g.out == out && g.T == T && g.precision == h->precision) exec = g.exec;
    if (!exec) {
      if (!h->cap_stream) CK(cudaStreamCreateWithFlags(&h->cap_stream, cudaStreamNonBlocking));
      if (dense_ok(h, T)) ensure_dense(h);  // no allocation while capturing
      if (cert_enabled()) cert_prepare(h, h->precision == CL_MOE_FP8_E4M3 && h->router_fp8, (cudaStream_t)stream);
      const bool prof = h->prof;
      h->prof = false;  // no timing events inside the graph
      CK(cudaStreamBeginCapture(h->cap_stream, cudaStreamCaptureModeThreadLocal));
      try {
        run_forward(h, hidden, T, out, false, h->cap_stream);
      } catch (...) {
        cudaGraph_t g = nullptr;
        cudaStreamEndCapture(h->cap_stream, &g);
        if (g) cudaGraphDestroy(g);
        h->prof = prof;
        throw;
      }
      h->prof = prof;
      cudaGraph_t g = nullptr;
      CK(cudaStreamEndCapture(h->cap_stream, &g));
      const cudaError_t ie = cudaGraphInstantiate(&exec, g, 0);
      cudaGraphDestroy(g);
      CK(ie);
      if (h->graphs.size() >= 16) {  // bounded cache: drop the oldest
        cudaGraphExecDestroy(h->graphs.front().exec);
        h->graphs.erase(h->graphs.begin());
      }
      h->graphs.push_back({hidden, out, T, h->precision, exec});
    }
    if (cert_enabled())  // the certified router's fp32 W_r copy follows weight updates
      cert_prepare(h, h->precision == CL_MOE_FP8_E4M3 && h->router_fp8, (cudaStream_t)stream);
    CK(cudaGraphLaunch(exec, (cudaStream_t)stream));
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
  // fp32 host tensors: routed on their own fp32 values (bit-exact with the reference's gating on
  // the same Tensor); the expert GEMMs take the bf16 rounding
  run_forward(h, sl.x, T, sl.out, f32, st, f32 ? sl.xf : nullptr, f32);
  CK(cudaEventRecord(sl.done, st));
  CK(cudaStreamWaitEvent(h->s_d2h, sl.done, 0));
  CK(cudaMemcpyAsync(out_host, sl.out, n * (f32 ? 4 : 2), cudaMemcpyDeviceToHost, h->s_d2h));
  CK(cudaEventRecord(sl.d2h, h->s_d2h));
  sl.used = true;
}

static void host_wait(cl_moe* h) {
  CK(cudaSetDevice(h->cfg.device));
  ep_wait(h, h->s_d2h, "host-buffer forward");
  ep_wait(h, h->own_stream, "host-buffer forward");
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
    ep_wait(h, (cudaStream_t)stream, "forward");  // bounded when a communicator exists
    int flag = 0;
    CK(cudaMemcpy(&flag, h->rb.finite_flag, sizeof(int), cudaMemcpyDeviceToHost));
    if (flag) {
      CK(cudaMemset(h->rb.finite_flag, 0, sizeof(int)));
      if (flag & 2) throw RunErr("expert-parallel receive buffer overflow");
      if (flag & 4) throw RunErr("expert-parallel rows did not arrive within 20 s (a peer rank failed)");
      throw RunErr("non-finite value produced by op 'moe_forward'");
    }
  });
}

cl_status cl_moe_stage_buffers(cl_moe* h, cl_moe_stage_view* v) {
  return guarded(h, [&] {
    if (!v) throw ConfigErr("view is null");
    if (h->last_dense) {  // dense decode: every expert x every token, row e*T + t
      v->offsets = h->offd;
      v->perm = nullptr;  // no permutation is materialised
      v->inv = h->invd;
      v->row_weight = h->rwd;
      v->x_perm = h->xd;
      v->act = h->actd;
      v->y = h->yd;
    } else {
      v->offsets = h->rb.offsets;
      v->perm = h->perm;
      v->inv = h->inv;
      v->row_weight = h->row_w;
      v->x_perm = h->last_xperm_padded ? nullptr : h->xperm;  // (single-GPU training: padded)
      v->act = h->last_xperm_padded ? nullptr : h->act;
      v->y = h->y;
    }
    v->rows = h->last_rows;
  });
}

cl_status cl_moe_copy_stage(cl_moe* h, int32_t which, void* dst, int64_t bytes, void* stream) {
  return guarded(h, [&] {
    const void* src = nullptr;
    const bool dn = h->last_dense;
    switch (which) {
      case 0: src = dn ? (const void*)h->offd : h->rb.offsets; break;
      case 1:
        if (dn) throw RunErr("perm is not materialised by a dense-decode forward (CL_MOE_DENSE_DECODE=0 for the sparse path)");
        src = h->perm;
        break;
      case 2: src = dn ? (const void*)h->invd : h->inv; break;
      case 3: src = dn ? (const void*)h->rwd : h->row_w; break;
      case 4:
        if (h->last_xperm_padded)
          throw RunErr("x_perm is kept in the padded row layout after a single-GPU training forward");
        src = dn ? (const void*)h->xd : h->xperm;
        break;
      case 5:
        if (h->last_xperm_padded)
          throw RunErr("act is kept in the padded row layout after a single-GPU training forward");
        src = dn ? (const void*)h->actd : h->act;
        break;
      case 6: src = dn ? (const void*)h->yd : h->y; break;
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
      const int kind = h->prof_kind[c];  // 0 forward, 1 backward, 2 dense-decode forward
      const int n = kind == 1 ? kBwdStages : kStages;
      CK(cudaEventSynchronize(ev[n]));
      for (int s = 0; s < n; ++s) {
        // dense decode: router + plan run on a side stream, so the dispatch stage is timed from
        // the fork point (ev[0]) on the compute stream, not from the end of the plan
        const int from = (kind == 2 && s == 2) ? 0 : s;
        float ms = 0.0f;
        CK(cudaEventElapsedTime(&ms, ev[from], ev[s + 1]));
        stage_ms[(kind == 1 ? kStages : 0) + s] += ms;
      }
      calls[kind == 1 ? 1 : 0] += 1;
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
    h->alpha_smooth = alpha;
  });
}

static void fold_smoothing_impl(cl_moe* h, const float* s) {
    const int64_t d = h->d, N = h->N;
    for (int64_t l = 0; l < d; ++l)
      if (!(s[l] > 0.0f) || !std::isfinite(s[l])) throw ConfigErr("smoothing factors must be finite and > 0");
    CK(cudaSetDevice(h->cfg.device));
    if (h->smooth_applied.empty()) h->smooth_applied.assign(d, 1.0f);
    for (int64_t l = 0; l < d; ++l) h->smooth_applied[l] *= s[l];
    CK(cudaMemcpy(h->smooth, s, sizeof(float) * d, cudaMemcpyHostToDevice));
    const int64_t n = (int64_t)h->n_local * 2 * h->f * d;
    scale_cols_bf16_kernel<<<grid_for(n), 256>>>(h->win, n, (int)d, h->smooth);
    scale_rows_f32_kernel<<<(int)((d * N + 255) / 256), 256>>>(h->wr, (int)d, (int)N, h->smooth);
    widen_router_kernel<<<grid_for(d * N), 256>>>(h->wr, (int)d, (int)N, h->wr64);
    ++h->wr_ver;
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    // derived copies are stale now
    h->fp8_ready = false;
    h->precision = CL_MOE_BF16;
    h->train_ready = false;
    CK(cudaMemset(h->calib, 0, sizeof(float) * 2 * h->n_local));
    CK(cudaMemset(h->calib_ch, 0, sizeof(float) * d));
}

cl_status cl_moe_fold_smoothing(cl_moe* h, const float* s) {
  return guarded(h, [&] {
    if (!s) throw ConfigErr("s is null");
    fold_smoothing_impl(h, s);
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
        ep_wait(h, st, "calibration all-reduce");
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
    // router: per-tensor activation scale = max |hidden| over the calibration tokens
    // / 448 (all ranks' maxima under EP), unless set explicitly; W_r per expert column
    if (!h->sxr_explicit) {
      std::vector<float> ch(h->d);
      if (h->comm) {
        cudaStream_t st = nullptr;
        NCK(NcclApi::get().AllReduce(h->calib_ch, h->calib_ch, (size_t)h->d, NcclApi::kFloat32, NcclApi::kMax, h->comm,
                                     st));
        ep_wait(h, st, "router calibration all-reduce");
      }
      CK(cudaMemcpy(ch.data(), h->calib_ch, sizeof(float) * h->d, cudaMemcpyDeviceToHost));
      float m = 0.0f;
      for (float v : ch) m = std::max(m, v);
      if (h->router_fp8 && !(m > 0.0f))
        throw RunErr("quantize_model: missing calibration for the router (calibrate, or cl_moe_set_router_fp8 "
                     "with an explicit activation scale)");
      h->sxr = m > 0.0f ? m / 448.0f : 1.0f;
    }
    CK(cudaMemcpy(h->sxr_dev, &h->sxr, sizeof(float), cudaMemcpyHostToDevice));
    router_qdq_w_kernel<<<(int)((N + 127) / 128), 128>>>(h->wr, (int)h->d, N, h->wrq, h->wsr);
    widen_router_kernel<<<grid_for(h->d * N), 256>>>(h->wrq, (int)h->d, N, h->wr64q);
    ++h->wrq_ver;
    CK(cudaGetLastError());
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

// ---- FP8 scheme file: JSON manifest + binary scale arrays (scheme.hpp) ----
// W_in's packed row p of an expert (256-row n-blocks of 128 gate + 128 up rows) <-> reference column
static int64_t win_col_of_packed_row(int64_t p, int64_t f) {
  const int64_t b = p / 256, i = p % 256;
  return i < 128 ? b * 128 + i : f + b * 128 + (i - 128);
}

cl_status cl_moe_save_fp8_scheme(cl_moe* h, const char* path) {
  return guarded(h, [&] {
    if (!path) throw ConfigErr("path is null");
    if (!h->fp8_ready) throw ConfigErr("FP8 scheme not quantized yet");
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaDeviceSynchronize());
    const int64_t d = h->d, N = h->N, NL = h->n_local, f = h->f;
    Scheme sc;
    sc.d = d;
    sc.N = N;
    sc.f = f;
    sc.n_local = NL;
    sc.expert0 = h->e0;
    sc.ep_size = h->cfg.ep_size;
    sc.alpha = h->alpha_smooth;
    sc.tau = h->tau;
    sc.router_fp8 = h->router_fp8;
    auto add = [&](const char* name, std::vector<int64_t> shape, std::vector<float> v) {
      sc.arrays.push_back(SchemeArray{name, std::move(shape), std::move(v)});
    };
    add("smoothing", {d}, h->smooth_applied.empty() ? std::vector<float>(d, 1.0f) : h->smooth_applied);
    std::vector<float> v(N);
    CK(cudaMemcpy(v.data(), h->sx_in_all, sizeof(float) * N, cudaMemcpyDeviceToHost));
    add("act_scale_in", {N}, v);
    v.resize(NL);
    CK(cudaMemcpy(v.data(), h->sx_mid, sizeof(float) * NL, cudaMemcpyDeviceToHost));
    add("act_scale_mid", {NL}, v);
    std::vector<float> packed(NL * 2 * f);
    CK(cudaMemcpy(packed.data(), h->ws_in, sizeof(float) * NL * 2 * f, cudaMemcpyDeviceToHost));
    v.assign(NL * 2 * f, 0.0f);
    for (int64_t e = 0; e < NL; ++e)
      for (int64_t p = 0; p < 2 * f; ++p) v[e * 2 * f + win_col_of_packed_row(p, f)] = packed[e * 2 * f + p];
    add("w_in_scale", {NL, 2 * f}, v);
    v.resize(NL * d);
    CK(cudaMemcpy(v.data(), h->ws_out, sizeof(float) * NL * d, cudaMemcpyDeviceToHost));
    add("w_out_scale", {NL, d}, v);
    add("router_act_scale", {1}, std::vector<float>{h->sxr});
    v.resize(N);
    CK(cudaMemcpy(v.data(), h->wsr, sizeof(float) * N, cudaMemcpyDeviceToHost));
    add("router_w_scale", {N}, v);
    write_scheme(path, sc);
  });
}

cl_status cl_moe_load_fp8_scheme(cl_moe* h, const char* path) {
  return guarded(h, [&] {
    if (!path) throw ConfigErr("path is null");
    const Scheme sc = read_scheme(path);
    const int64_t d = h->d, N = h->N, NL = h->n_local, f = h->f;
    if (sc.d != d || sc.N != N || sc.f != f || sc.n_local != NL || sc.expert0 != h->e0)
      throw ConfigErr(fmt("scheme is for d=%lld N=%lld f=%lld experts [%lld, +%lld), this layer d=%lld N=%lld f=%lld "
                          "[%d, +%d)", (long long)sc.d, (long long)sc.N, (long long)sc.f, (long long)sc.expert0,
                          (long long)sc.n_local, (long long)d, (long long)N, (long long)f, h->e0, NL));
    auto arr = [&](const char* name, int64_t n) -> const std::vector<float>& {
      const SchemeArray& a = sc.get(name);
      if ((int64_t)a.data.size() != n) throw ConfigErr(fmt("scheme array %s has %zu values, expected %lld", name,
                                                           a.data.size(), (long long)n));
      return a.data;
    };
    // smoothing: fold it unless this layer already carries exactly that fold
    const std::vector<float>& s = arr("smoothing", d);
    const bool ident = std::all_of(s.begin(), s.end(), [](float x) { return x == 1.0f; });
    const bool have = !h->smooth_applied.empty() &&
                      !std::all_of(h->smooth_applied.begin(), h->smooth_applied.end(), [](float x) { return x == 1.0f; });
    if (have && h->smooth_applied != s)
      throw ConfigErr("scheme smoothing vector differs from the one already folded into this layer");
    if (!ident && !have) fold_smoothing_impl(h, s.data());
    CK(cudaSetDevice(h->cfg.device));
    ensure_fp8_storage(h);
    const std::vector<float>& sin = arr("act_scale_in", N);
    const std::vector<float>& smid = arr("act_scale_mid", NL);
    const std::vector<float>& wi = arr("w_in_scale", NL * 2 * f);
    const std::vector<float>& wo = arr("w_out_scale", NL * d);
    const float sxr = arr("router_act_scale", 1)[0];
    const std::vector<float>& wsr = arr("router_w_scale", N);
    for (const auto* v : {&sin, &smid, &wi, &wo, &wsr})
      for (float x : *v)
        if (!(x > 0.0f) || !std::isfinite(x)) throw ConfigErr("scheme scales must be finite and > 0");
    if (!(sxr > 0.0f) || !std::isfinite(sxr)) throw ConfigErr("scheme scales must be finite and > 0");
    std::vector<float> packed(NL * 2 * f);
    for (int64_t e = 0; e < NL; ++e)
      for (int64_t p = 0; p < 2 * f; ++p) packed[e * 2 * f + p] = wi[e * 2 * f + win_col_of_packed_row(p, f)];
    CK(cudaMemcpy(h->sx_in_all, sin.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->sx_in, sin.data() + h->e0, sizeof(float) * NL, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->sx_mid, smid.data(), sizeof(float) * NL, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->ws_in, packed.data(), sizeof(float) * NL * 2 * f, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->ws_out, wo.data(), sizeof(float) * NL * d, cudaMemcpyHostToDevice));
    CK(cudaMemcpy(h->wsr, wsr.data(), sizeof(float) * N, cudaMemcpyHostToDevice));
    h->sxr = sxr;
    h->sxr_explicit = true;
    h->router_fp8 = sc.router_fp8 ? 1 : 0;
    CK(cudaMemcpy(h->sxr_dev, &h->sxr, sizeof(float), cudaMemcpyHostToDevice));
    const int64_t r1 = NL * 2 * f, r2 = NL * d;
    quantize_rows_e4m3_kernel<<<(int)((r1 + 7) / 8), 256>>>(h->win, r1, (int)d, h->win8, h->ws_in, true);
    quantize_rows_e4m3_kernel<<<(int)((r2 + 7) / 8), 256>>>(h->wout, r2, (int)f, h->wout8, h->ws_out, true);
    router_qdq_w_kernel<<<(int)((N + 127) / 128), 128>>>(h->wr, (int)d, (int)N, h->wrq, h->wsr, true);
    widen_router_kernel<<<grid_for(d * N), 256>>>(h->wrq, (int)d, (int)N, h->wr64q);
    ++h->wrq_ver;
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    h->alpha_smooth = sc.alpha;
    h->tau = sc.tau;
    h->fp8_ready = true;
    h->precision = CL_MOE_FP8_E4M3;
  });
}

cl_status cl_moe_router_stats(cl_moe* h, int64_t* cert_calls, int64_t* last_recomputed) {
  return guarded(h, [&] {
    CK(cudaSetDevice(h->cfg.device));
    CK(cudaDeviceSynchronize());
    if (cert_calls) *cert_calls = h->cert_calls;
    if (last_recomputed) {
      int n = 0;
      if (h->cert_count) CK(cudaMemcpy(&n, h->cert_count, sizeof(int), cudaMemcpyDeviceToHost));
      *last_recomputed = n;
    }
  });
}

cl_status cl_moe_router_variant(cl_moe* h, int32_t* variant, int32_t* dmma_ok) {
  return guarded(h, [&] {
    if (variant) *variant = h->last_router_variant;
    if (dmma_ok) *dmma_ok = h->dmma_ok ? 1 : 0;
  });
}

cl_status cl_moe_set_router_fp8(cl_moe* h, int32_t enable, float act_scale) {
  return guarded(h, [&] {
    if (enable != 0 && enable != 1) throw ConfigErr("enable must be 0 or 1");
    if (act_scale < 0.0f || !std::isfinite(act_scale)) throw ConfigErr("act_scale must be finite and >= 0");
    h->router_fp8 = enable;
    h->sxr_explicit = act_scale > 0.0f;
    if (h->sxr_explicit) {
      h->sxr = act_scale;
      if (h->sxr_dev) {
        CK(cudaSetDevice(h->cfg.device));
        CK(cudaMemcpy(h->sxr_dev, &h->sxr, sizeof(float), cudaMemcpyHostToDevice));
      }
    }
  });
}

cl_status cl_moe_get_router_fp8(cl_moe* h, int32_t* enable, float* act_scale, float* w_scale) {
  return guarded(h, [&] {
    if (enable) *enable = h->router_fp8;
    if (act_scale || w_scale) {
      if (!h->fp8_ready) throw ConfigErr("FP8 scheme not quantized yet");
      if (act_scale) *act_scale = h->sxr;
      if (w_scale) {
        CK(cudaSetDevice(h->cfg.device));
        CK(cudaDeviceSynchronize());
        CK(cudaMemcpy(w_scale, h->wsr, sizeof(float) * h->N, cudaMemcpyDeviceToHost));
      }
    }
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
