/*
 * compass_moe.h — C ABI of the B200-native (sm_100a) MoE-layer hot path.
 *
 * Drop-in for the MoE-layer operations the reference specifies and composes from its tensor
 * primitives:
 *   route_tokens(hidden, router_weights) -> RouterDecision
 *   moe_forward(hidden, decision, experts) -> out
 *   aux_loss(decision) / z_loss(logits)
 *                                (proj/src/tensor.cpp:980-1040 ops::moe_aux_loss / ops::z_loss)
 *   fp8_qdq / quantize_model (expert-aware E4M3 W8A8 scheme)
 * and keeps the conventions of the reference C API proj/include/compass_lab.h:20-50 /
 * proj/src/capi.cpp:13-68: an opaque handle, cl_status return codes (same values as
 * compass_lab.h:23-27), per-handle last-error string owned by the handle ("" if none), configuration
 * errors -> CL_ERR_CONFIG, every other failure (CUDA error, non-finite output, bad runtime input)
 * -> CL_ERR_RUN.
 *
 * Memory: unless a function says "host", tensor pointers are DEVICE pointers on the handle's GPU
 * and `stream` is a cudaStream_t (NULL = legacy default stream). Calls are asynchronous on
 * `stream` except where noted; the handle owns its weights and workspaces. One handle per
 * (process, GPU); callers serialise calls on a handle (as with cl_lab).
 *
 * Layouts (row-major, reference orientation):
 *   hidden / out        [T x d]        bf16 (the device path's storage type)
 *   w_router            [d x N]        fp32 (router gating stays fp32, PAPER §2.3.4)
 *   w_in  (expert e)    [d x 2f]       columns [0,f) = gate, [f,2f) = up
 *   w_out (expert e)    [f x d]
 *   topk_idx            [T x K] int32, descending probability, ties -> lowest expert index
 *   combine_weights     [T x K] fp32  (top-K probabilities renormalised to sum 1)
 */
#ifndef COMPASS_MOE_H
#define COMPASS_MOE_H

#include <stddef.h>
#include <stdint.h>

/* cl_status is the reference's (compass_lab.h:23-27). When the reference header is on the include
 * path, include it here so that either include order works (compass_lab.h defines cl_status
 * unguarded); otherwise define the identical enum. */
#if defined(__has_include)
#if __has_include("compass_lab.h")
#include "compass_lab.h"
#endif
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* otherwise: identical to compass_lab.h:23-27 */
#ifndef COMPASS_LAB_H
typedef enum cl_status {
  CL_OK = 0,        /* success */
  CL_ERR_RUN = 1,   /* validation or runtime failure */
  CL_ERR_CONFIG = 2 /* bad config or bad arguments */
} cl_status;
#endif

typedef struct cl_moe cl_moe;

typedef enum cl_moe_precision {
  CL_MOE_BF16 = 0,    /* bf16 operands, fp32 accumulate */
  CL_MOE_FP8_E4M3 = 1 /* expert-aware W8A8: e4m3 operands, per-expert act scale, per-channel W scale */
} cl_moe_precision;

typedef enum cl_moe_io_dtype { CL_MOE_IO_BF16 = 0, CL_MOE_IO_F32 = 1 } cl_moe_io_dtype;

typedef struct cl_moe_config {
  int64_t d_model;    /* d  (multiple of 256) */
  int64_t n_experts;  /* N  (global expert count, 1..128) */
  int64_t top_k;      /* K  (1..min(N,8)) */
  int64_t d_ff;       /* f  (multiple of 128) */
  int64_t max_tokens; /* capacity: tokens per call on this rank */
  int32_t device;     /* CUDA device ordinal */
  int32_t gemm_ctas;  /* 0 = auto, 1 = cta_group::1 (M=128), 2 = cta_group::2 (M=256) */
  int32_t ep_size;    /* expert-parallel ranks (1 = single GPU) */
  int32_t ep_rank;    /* this rank; owns experts [rank*N/ep_size, (rank+1)*N/ep_size) */
} cl_moe_config;

/* Routing result (SPEC RouterDecision). Device pointers; NULL fields skipped. */
typedef struct cl_moe_decision {
  float* logits;          /* [T x N] */
  float* probs;           /* [T x N] */
  int32_t* topk_idx;      /* [T x K] */
  float* combine_weights; /* [T x K] */
  int64_t* counts;        /* [N]   c_i, sums to T*K exactly */
  float* agg_prob;        /* [N]   p_i = sum_j probs[j][i] */
  float* aux_loss;        /* [1]   N * sum_i (p_i/B)(c_i/(B K))  (ops::moe_aux_loss) */
  float* z_loss;          /* [1]   (1/B) sum_j lse_j^2            (ops::z_loss) */
} cl_moe_decision;

/* Internal per-call workspaces, exposed read-only for stage-level parity checks. */
typedef struct cl_moe_stage_view {
  const int32_t* offsets;  /* [N_local+1] expert segment starts in the permuted row space */
  const int32_t* perm;     /* [T*K] permuted row r -> slot j*K+k */
  const int32_t* inv;      /* [T*K] slot j*K+k -> permuted row r */
  const float* row_weight; /* [T*K] combine weight of permuted row r */
  const void* x_perm;      /* [T*K x d] GEMM1 operand (bf16, or e4m3 in FP8 mode) */
  const void* act;         /* [T*K x f] SwiGLU output / GEMM2 operand (bf16, or e4m3) */
  const void* y;           /* [T*K x d] bf16 weighted expert outputs */
  int64_t rows;            /* T*K of the last call */
} cl_moe_stage_view;

const char* cl_moe_version(void);

/* Creates a layer from reference-layout fp32 HOST weights: w_router [d x N], w_in [N][d][2f],
 * w_out [N][f][d]. The handle keeps bf16 copies repacked K-major for the tensor cores. With
 * ep_size > 1, w_in / w_out hold only this rank's N/ep_size experts. */
cl_status cl_moe_create(const cl_moe_config* cfg, const float* w_router, const float* w_in,
                        const float* w_out, cl_moe** out);

/* Creates a layer from a reference checkpoint file (CLCKPT1, proj/include/compasslab/checkpoint.hpp)
 * holding "<prefix>router" [d x N] and "<prefix>experts.<e>.w_in" [d x 2f] /
 * "<prefix>experts.<e>.w_out" [f x d] (fp32). Missing tensor / wrong shape -> CL_ERR_RUN. */
cl_status cl_moe_create_from_checkpoint(const cl_moe_config* cfg, const char* path, const char* prefix,
                                        cl_moe** out);
/* Writes the layer's weights (as stored: bf16-valued fp32) in the same format and naming; the
 * file round-trips byte-exactly through the reference's load_checkpoint / save_checkpoint. */
cl_status cl_moe_save_checkpoint(cl_moe* h, const char* path, const char* prefix);

/* HOST copies of the weights the layer holds, in the reference layouts (as stored: bf16-valued
 * fp32 for the experts): w_router [d x N], and local expert `expert`'s w_in [d x 2f] / w_out [f x d].
 * Any pointer may be NULL. Synchronous. */
cl_status cl_moe_get_weights(cl_moe* h, float* w_router, int64_t expert, float* w_in, float* w_out);

/* Creates a layer whose weights are generated on the device from the reference counter PRNG
 * (proj/include/compasslab/prng.hpp) exactly as SURVEY.md §8(d) prescribes (root seed `seed`). */
cl_status cl_moe_create_synthetic(const cl_moe_config* cfg, uint64_t seed, cl_moe** out);

void cl_moe_destroy(cl_moe* h);

/* Message of the most recent failing call on this handle ("" if none); owned by the handle.
 * With h == NULL: the most recent failing create entry on this thread. */
const char* cl_moe_last_error(const cl_moe* h);

/* Synthetic tokens x = split(1) N(0,1) of root seed `seed`, rounded to bf16: [T x d] device. */
cl_status cl_moe_synthetic_tokens(cl_moe* h, uint64_t seed, int64_t T, void* x, void* stream);

/* Skewed-routing stress construction: tokens x = N(0,1) + shift (then
 * bf16), and router columns W_r[:, i] += gamma * ln(1/(i+1)^1.2) / d. */
cl_status cl_moe_synthetic_tokens_shifted(cl_moe* h, uint64_t seed, int64_t T, float shift, void* x,
                                          void* stream);
cl_status cl_moe_synthetic_skew(cl_moe* h, double gamma);

/* route_tokens. */
cl_status cl_moe_route_tokens(cl_moe* h, const void* hidden, int64_t T, const cl_moe_decision* out,
                              void* stream);

/* route_tokens on the caller's fp32 hidden [T x d] (device): the gating is computed on the fp32
 * values themselves, so the decision is bit-exact with the reference's
 * route_tokens on the same Tensor (no bf16 rounding before the router). */
cl_status cl_moe_route_tokens_f32(cl_moe* h, const float* hidden, int64_t T, const cl_moe_decision* out,
                                  void* stream);

/* moe_forward with a caller-supplied decision. */
cl_status cl_moe_moe_forward(cl_moe* h, const void* hidden, int64_t T, const int32_t* topk_idx,
                             const float* combine_weights, void* out, void* stream);

/* The fused layer: route_tokens + dispatch + expert FFN + combine. `out` bf16 [T x d].
 * `decision` may be NULL. Single-GPU calls with T <= 128 take the dense-decode path (every
 * expert runs all T tokens while routing runs beside GEMM1 on an internal high-priority stream
 * joined back into `stream`); results are bit-identical to the sparse path. Its buffers
 * (N x 128 rows of x, SwiGLU output and expert output) are allocated on the first such call.
 * Environment: CL_MOE_DENSE_DECODE=0 disables it. */
cl_status cl_moe_forward(cl_moe* h, const void* hidden, int64_t T, void* out,
                         const cl_moe_decision* decision, void* stream);
/* The fused layer on fp32 device tensors (the reference's Tensor dtype): routes on the fp32 hidden
 * (as cl_moe_route_tokens_f32), runs the experts on its bf16 rounding, and writes fp32 `out`
 * [T x d] (the combine's fp32 accumulators, unrounded). */
cl_status cl_moe_forward_f32(cl_moe* h, const float* hidden, int64_t T, float* out, const cl_moe_decision* decision,
                             void* stream);
/* cl_moe_forward without the decision outputs, captured into a CUDA graph on first use for each
 * (hidden, out, T, precision) and replayed afterwards (one launch per call; decode-size steps).
 * Single-GPU layer only. The graph bakes in the buffer addresses: reuse the same buffers. */
cl_status cl_moe_forward_graph(cl_moe* h, const void* hidden, int64_t T, void* out, void* stream);

/* Same layer through HOST buffers (the reference-facing call): copies hidden in, runs the
 * layer and copies the output back; synchronous. io_dtype selects bf16 or fp32 host tensors;
 * fp32 hidden is routed on its fp32 values (as cl_moe_forward_f32). */
cl_status cl_moe_forward_host(cl_moe* h, const void* hidden_host, int64_t T, void* out_host,
                              int32_t io_dtype);

/* Pipelined variant of cl_moe_forward_host: enqueues the H2D copy, the layer and the D2H copy
 * on the handle's internal copy / compute streams and returns. Two internal slots let the copies
 * of neighbouring calls overlap the compute; `hidden_host` must stay valid and `out_host` must
 * not be read until cl_moe_host_wait returns (pinned host memory gives asynchronous copies). */
cl_status cl_moe_forward_host_async(cl_moe* h, const void* hidden_host, int64_t T, void* out_host,
                                    int32_t io_dtype);
/* Waits for every enqueued host-buffer call; reports non-finite outputs like cl_moe_sync. */
cl_status cl_moe_host_wait(cl_moe* h);

/* Waits for `stream` and reports device-side failures: any non-finite router logit or layer
 * output (the reference's check_finite, proj/src/tensor.cpp:35-41) -> CL_ERR_RUN. */
cl_status cl_moe_sync(cl_moe* h, void* stream);

/* Opt-in certified large-batch routing in the fused forward (no decision export; environment
 * CL_MOE_ROUTER_CERT=1, DESIGN.md §4 K1): fp32 logits with a rigorous error bound decide every token
 * whose top-K order is unambiguous, the others are recomputed with the reference's exact fp64
 * chains; routing indices, counts and the permutation are bit-exact either way. cert_calls =
 * certified routing calls so far, last_recomputed = tokens recomputed exactly in the last one.
 * Synchronous. */
cl_status cl_moe_router_stats(cl_moe* h, int64_t* cert_calls, int64_t* last_recomputed);

/* Which router kernel (K1) the last routing call ran, for diagnostics and tests: 0 = 128-thread 1x4
 * blocked, 1 = 32-thread 1x4 with a deep ring, 2 = 4x4 / 2x4 blocked, 3 = latency 1x1, 4 = warp-
 * specialised 1x1 chains (decode), 5 = fp64 tensor cores (DMMA), 6 = certified. dmma_ok = 1 when
 * the handle's device check found DMMA accumulating as the sequential fp64 chain (variant 5 is
 * then used for batches beyond the decode sizes; environment CL_MOE_ROUTER_DMMA=0 disables it). */
cl_status cl_moe_router_variant(cl_moe* h, int32_t* variant, int32_t* dmma_ok);

/* Stage buffers of the last call (valid until the next call on the handle). After a dense-decode
 * forward (single GPU, T <= 128) they are the dense buffers: rows = N*T, row e*T + t = token t for
 * expert e (offsets[e] = e*T), row_weight = the combine weight of (t, e) or 0 when e is not among
 * t's top-K, inv[t*K + k] = the row of token t's k-th expert; perm = NULL (copy_stage(1) ->
 * CL_ERR_RUN): no permutation is materialised. After a single-GPU cl_moe_forward_train the
 * dispatched rows and the SwiGLU output live only in the padded layouts the weight gradients
 * read: x_perm = act = NULL (copy_stage(4) / copy_stage(5) -> CL_ERR_RUN). */
cl_status cl_moe_stage_buffers(cl_moe* h, cl_moe_stage_view* view);

/* Copies stage buffer `which` (0 offsets, 1 perm, 2 inv, 3 row_weight, 4 x_perm, 5 act, 6 y)
 * into the device buffer `dst` (`bytes` bytes), stream-ordered after the last call. */
cl_status cl_moe_copy_stage(cl_moe* h, int32_t which, void* dst, int64_t bytes, void* stream);

/* Per-stage device timing with CUDA events recorded on the launch stream between the kernels of
 * each call. Forward stages 0 router, 1 plan, 2 dispatch, 3 GEMM1(+SwiGLU), 4 GEMM2(+weight),
 * 5 combine; backward stages 6 combine-bwd, 7 dgrad-1(+SwiGLU-bwd), 8 dgrad-2, 9 dispatch-bwd,
 * 10 transposes, 11 wgrad dW_out, 12 wgrad dW_in. profile_read returns the summed milliseconds
 * per stage (stage_ms has 13 entries) since enabling/reading and calls[0] forward / calls[1]
 * backward call counts; it synchronises on the recorded events. */
cl_status cl_moe_profile(cl_moe* h, int32_t enable);
cl_status cl_moe_profile_read(cl_moe* h, double* stage_ms, int64_t* calls);

/* Expert-aware FP8. Calibration (collect_calibration) runs
 * the bf16 layer on `hidden` and accumulates per-expert activation maxima of the GEMM1 input and
 * the SwiGLU output; quantize then sets per-expert activation scales = max/448 and per-(expert,
 * output channel) weight scales = channel absmax/448 and switches the
 * handle's precision. act_scale_* may be given explicitly instead: act_scale_in [N] (every
 * expert's GEMM1-input scale; under expert parallelism the source quantizes each dispatched row
 * with its owner's scale, so all ranks need the same global table) and act_scale_mid [N_local].
 * Under expert parallelism, calibration keeps the GEMM1-input maxima per global expert at the
 * source and quantize all-reduces them (max) over the ranks. */
cl_status cl_moe_calibrate(cl_moe* h, const void* hidden, int64_t T, int32_t reset, void* stream);
cl_status cl_moe_quantize_fp8(cl_moe* h, const float* act_scale_in, const float* act_scale_mid);
/* balance_calibration: with the expert counts of the routed `base` tokens
 * (bf16 device [T_base x d], may be NULL), pre-route the `pool` tokens (router only, in order)
 * and select every pool token routed to an expert still below `tau`, until all counts reach tau.
 * selected (host, capacity P) receives the chosen pool row indices, n_selected their number,
 * final_counts (host [N]) the resulting counts. Pool exhausted with an expert below tau ->
 * CL_ERR_RUN naming the expert; tau < 1 -> CL_ERR_CONFIG. */
cl_status cl_moe_balance_calibration(cl_moe* h, const void* base, int64_t T_base, const void* pool,
                                     int64_t P, int64_t tau, int64_t* selected, int64_t* n_selected,
                                     int64_t* final_counts, void* stream);

/* Unified smoothing. compute: s_j = max|X_j|^alpha / max|W_j|^(1-alpha) from the
 * calibration per-channel maxima of the layer input and the joint per-input-channel maxima of
 * every expert's W_in and W_r (zero-max channels -> 1); s_out is a host array [d]. fold: rows
 * of every W_in and of W_r are scaled by s (the preceding RMSNorm gain must be divided by s by
 * the caller, i.e. later inputs are x / s). Folding invalidates the FP8 scheme (re-calibrate and
 * quantize again) and clears the calibration maxima. */
cl_status cl_moe_compute_smoothing(cl_moe* h, float alpha, float* s_out);
cl_status cl_moe_fold_smoothing(cl_moe* h, const float* s);
cl_status cl_moe_set_precision(cl_moe* h, int32_t precision);
/* Host copies of the FP8 scales in use: [N_local], [N_local], [N_local x 2f], [N_local x d]. */
/* collect_calibration statistics accumulated by cl_moe_calibrate since the last reset (any
 * pointer may be NULL): counts[N] routing counts (sum = tokens x K), x_max[N_local] / mid_max
 * [N_local] per-expert max |GEMM1 input| / |SwiGLU output|, ch_max[d] per-channel max |hidden|.
 * An empty calibration set (T = 0) leaves them unchanged (zero after a reset). */
cl_status cl_moe_calibration_stats(cl_moe* h, int64_t* counts, float* x_max, float* mid_max, float* ch_max);
/* The router under the FP8 scheme. SPEC.md:565 runs "all expert/router ... projection GEMMs"
 * through fp8_qdq: with enable = 1 (the default) an FP8-precision forward routes on
 * qdq(hidden, s_x) . qdq(W_r, s_w[i]) — s_x the per-tensor activation scale (calibration max |hidden|
 * / 448, or act_scale > 0 given here), s_w[i] = absmax of expert column i of W_r / 448 — still with
 * fp64 accumulation, so the decision is bit-exact with the oracle's route on those dequantised
 * values. enable = 0 keeps fp32 gating in FP8 mode (PAPER §2.3.4's training-stability choice).
 * Takes effect on the next forward; quantize_fp8 recomputes W_r's qdq. get: the mode, s_x and
 * s_w [N] (the last two need a quantized scheme). */
cl_status cl_moe_set_router_fp8(cl_moe* h, int32_t enable, float act_scale);
/* QuantScheme file ("JSON manifest + binary scale arrays"; fields SPEC.md:520-523):
 * `path` is the JSON manifest (layer shape, alpha_smooth, tau, router mode, one entry per array
 * {name, dtype, shape, offset}), `path`.bin the little-endian fp32 arrays: smoothing [d] (the
 * product of the folded smoothing vectors), act_scale_in [N], act_scale_mid [N_local], w_in_scale
 * [N_local][2f] (reference W_in column order), w_out_scale [N_local][d], router_act_scale [1],
 * router_w_scale [N]. save needs a quantized scheme. load applies a scheme to a layer holding the
 * same weights: folds its smoothing vector (unless this layer already carries exactly that fold;
 * a different fold -> CL_ERR_CONFIG), takes every scale from the file (no calibration), quantizes
 * the weights with the stored weight scales and switches to FP8 — the FP8 forward is then
 * bit-identical to the layer that saved it. Shape mismatch -> CL_ERR_CONFIG; unreadable or
 * malformed files -> CL_ERR_RUN. */
cl_status cl_moe_save_fp8_scheme(cl_moe* h, const char* path);
cl_status cl_moe_load_fp8_scheme(cl_moe* h, const char* path);
cl_status cl_moe_get_router_fp8(cl_moe* h, int32_t* enable, float* act_scale, float* w_scale);
cl_status cl_moe_get_fp8_scales(cl_moe* h, float* act_in, float* act_mid, float* w_in_scale,
                                float* w_out_scale);

/* ---- Expert-FFN backward (the reference Tape closures of the layer, tensor.cpp:364-372,
 * :318-321, :290-300, :411-418, :587-607, :801-809, :834-842). bf16, single GPU; d_ff % 256 == 0.
 * cl_moe_forward_train = cl_moe_forward that also keeps the SwiGLU pre-activations and the
 * unweighted expert outputs. cl_moe_backward(dOut) then returns, for that call:
 *   d_hidden [T x d] bf16 (through dispatch), d_combine_w [T x K] fp32 (mul_rowwise backward),
 *   dw_in [N_local][d][2f] fp32 and dw_out [N_local][f][d] fp32 (reference layouts, overwritten).
 * The router backward (d probs -> d logits -> dW_r) is not part of this call. ---- */
cl_status cl_moe_forward_train(cl_moe* h, const void* hidden, int64_t T, void* out,
                               const cl_moe_decision* decision, void* stream);
cl_status cl_moe_backward(cl_moe* h, const void* d_out, void* d_hidden, float* d_combine_w,
                          float* dw_in, float* dw_out, void* stream);

/* Full layer backward of the last cl_moe_forward_train, router included:
 * gradient of  sum(out * d_out) + g_aux * L_aux + g_z * L_Z  (the total-loss coefficients of
 * SPEC.md:183-188) with respect to hidden (d_hidden, bf16, expert + router paths summed in fp32),
 * W_r (dw_router [d x N] fp32), W_in / W_out (as cl_moe_backward); d_combine_w optional (NULL).
 * The hidden tensor of the forward call must still be valid. top_k in {1, 2, 4}. */
cl_status cl_moe_backward_full(cl_moe* h, const void* d_out, float g_aux, float g_z, void* d_hidden,
                               float* dw_router, float* dw_in, float* dw_out, float* d_combine_w,
                               void* stream);

/* ---- Expert parallelism. One process per GPU; cfg.ep_size ranks, rank
 * cfg.ep_rank owns experts [rank*N/ep_size, (rank+1)*N/ep_size) (pass only those experts'
 * weights to cl_moe_create). Every rank routes its own tokens over all N experts; rows travel
 * to the owning rank over NCCL (NVLink) and back. ---- */
/* 128-byte NCCL unique id, generated on one rank and distributed by the caller. */
cl_status cl_moe_ep_unique_id(uint8_t* id_out);
/* Collective over the ep_size ranks: creates the handle's communicator. */
cl_status cl_moe_ep_init(cl_moe* h, const uint8_t* id);
/* Expert-parallel layer forward (cl_moe_forward dispatches here when ep_size > 1; with
 * ep_size == 1 this runs the same exchange code in loopback). bf16 only. */
cl_status cl_moe_ep_forward(cl_moe* h, const void* hidden, int64_t T, void* out,
                            const cl_moe_decision* decision, void* stream);
/* Switches an initialised EP handle to the peer-memory (NVLink) transport: collective over the
 * ranks; maps every rank's receive buffer and return buffer into this process (CUDA IPC, handles
 * exchanged over the communicator). Afterwards the forward moves rows with direct peer stores —
 * the dispatch kernel writes into the owners' receive buffers and the GEMM2 epilogue writes each
 * output row back into its source rank's buffer — and NCCL carries only the counts and two
 * barriers; training too (the combine-backward kernel stores dY rows into the owners' buffers,
 * the dgrad-2 epilogue stores dX rows back). Needs P2P access between the devices; if any
 * rank cannot map its peers, every rank returns CL_ERR_RUN and keeps the NCCL transport. */
cl_status cl_moe_ep_peer_init(cl_moe* h);
/* Single-process, single-device emulation of an R-rank EP group (handles hs[r] created with
 * ep_size = R, ep_rank = r on the same device, no communicator): runs the peer-transport forward
 * for every rank, phase by phase, with the other handles' buffers as the "peer" addresses. */
cl_status cl_moe_ep_group_forward(cl_moe* const* hs, int32_t R, const void* const* hidden,
                                  const int64_t* T, void* const* out, void* stream);
/* Training step of an emulated single-device group (see cl_moe_ep_group_forward): forward_train
 * and the expert-FFN backward (cl_moe_backward semantics) of every rank, with the backward's row
 * exchanges as peer stores (combine-backward kernel into the owners' dY buffers, dgrad-2 epilogue
 * into the sources' dX buffers). Per-rank arrays of R pointers. */
cl_status cl_moe_ep_group_train_step(cl_moe* const* hs, int32_t R, const void* const* hidden,
                                     const int64_t* T, void* const* out, const void* const* d_out,
                                     void* const* d_hidden, float* const* d_combine_w,
                                     float* const* dw_in, float* const* dw_out, void* stream);
/* The all-gathered R x N routing counts of the last expert-parallel forward (row = source rank),
 * e.g. to account the bytes each rank sent over NVLink. */
cl_status cl_moe_ep_last_counts(cl_moe* h, int64_t* counts);
/* Pure host helper (no GPU): peer-transport layout of `rank` from counts[R][N]:
 * dispatch_row[g] = first row of this rank's piece for expert g in the owner's receive buffer;
 * return_row[e*R+s] = first row of piece (local expert e, source s) in s's permutation;
 * local_offsets[N/R+1] as in cl_moe_ep_layout. */
cl_status cl_moe_ep_peer_layout(const int64_t* counts, int32_t R, int32_t N, int32_t rank,
                                int64_t* dispatch_row, int64_t* return_row, int64_t* local_offsets);
/* Pure host helper (no GPU): receive layout of `rank` from the all-gathered count matrix
 * counts[R][N] (row = source rank). local_offsets[N/R+1], recv_piece[(N/R)*R] indexed
 * e*R + s = first receive row of (local expert e, source s); recv_total = rows received. */
cl_status cl_moe_ep_layout(const int64_t* counts, int32_t R, int32_t N, int32_t rank,
                           int64_t* local_offsets, int64_t* recv_piece, int64_t* recv_total);

#ifdef __cplusplus
}
#endif

#endif /* COMPASS_MOE_H */
