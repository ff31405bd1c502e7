// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// The reference's MoE layer, composed from the reference's OWN primitives. The reference
// (compass-lab) implements every building block (compasslab::ops in proj/src/tensor.cpp) but
// not the layer itself, which exists only in SPEC.md:147-182. This file is the thinnest possible
// composition of those ops per SPEC; it is compiled TOGETHER WITH the reference sources, straight
// from /root/reference/proj/src (see oracle/Makefile, target `ref`), into oracle/_ref/. Nothing
// from the reference is copied into this repository.
//
// Used (a) to validate the restatement oracle/moe_oracle.cpp bit-for-bit, (b) to generate the
// golden vectors in tests/golden/, and (c) as the "reference" CPU arm of bench.py.

#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "compasslab/checkpoint.hpp"
#include "compasslab/common.hpp"
#include "compasslab/gradcheck.hpp"
#include "compasslab/prng.hpp"
#include "compasslab/tensor.hpp"

using compasslab::Tape;
using compasslab::Tensor;
namespace ops = compasslab::ops;

namespace {
thread_local std::string g_err;

std::vector<float> vec(const float* p, std::int64_t n) { return std::vector<float>(p, p + n); }

template <typename Fn>
int guarded(Fn fn) {
  try {
    fn();
    return 0;
  } catch (const compasslab::ConfigError& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 1;
  }
}
}  // namespace

extern "C" {

const char* ref_last_error(void) { return g_err.c_str(); }

// The reference's own counter PRNG (proj/include/compasslab/prng.hpp), exported so the oracle's
// restatement (orc_split_seed / orc_normals) and its replay properties can be pinned to it.
std::uint64_t ref_prng_split(std::uint64_t seed, std::uint64_t stream) {
  return compasslab::Prng(seed).split(stream).seed();
}
void ref_prng_u64(std::uint64_t seed, std::uint64_t counter, std::int64_t n, std::uint64_t* out) {
  compasslab::Prng p(seed, counter);
  for (std::int64_t i = 0; i < n; ++i) out[i] = p.next_u64();
}
void ref_prng_doubles(std::uint64_t seed, std::int64_t n, double* out) {
  compasslab::Prng p(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = p.next_double();
}
void ref_prng_normals(std::uint64_t seed, std::int64_t n, float mean, float stddev, float* out) {
  compasslab::Prng p(seed);
  for (std::int64_t i = 0; i < n; ++i) out[i] = p.next_normal_f(mean, stddev);
}

// route_tokens from ops::matmul, ops::softmax_rows, ops::top_k, ops::col_sums.
int ref_route(const float* x, const float* wr, std::int64_t T, std::int64_t d, std::int64_t N,
              std::int64_t K, float* logits, float* probs, std::int64_t* idx, float* w,
              std::int64_t* counts, float* agg_prob) {
  return guarded([&] {
    Tensor xt = Tensor::from_values({T, d}, vec(x, T * d));
    Tensor wt = Tensor::from_values({d, N}, vec(wr, d * N));
    Tensor z = ops::matmul(xt, wt);
    Tensor p = ops::softmax_rows(z);
    std::memcpy(logits, z.values().data(), sizeof(float) * T * N);
    std::memcpy(probs, p.values().data(), sizeof(float) * T * N);
    std::vector<float> val(static_cast<std::size_t>(K));
    for (std::int64_t i = 0; i < N; ++i) counts[i] = 0;
    for (std::int64_t j = 0; j < T; ++j) {
      ops::top_k(p.values().data() + j * N, N, K, idx + j * K, val.data());
      double s = 0.0;
      for (std::int64_t k = 0; k < K; ++k) s += static_cast<double>(val[static_cast<std::size_t>(k)]);
      for (std::int64_t k = 0; k < K; ++k) {
        w[j * K + k] = static_cast<float>(static_cast<double>(val[static_cast<std::size_t>(k)]) / s);
        counts[idx[j * K + k]] += 1;
      }
    }
    Tensor cs = ops::col_sums(p);
    std::memcpy(agg_prob, cs.values().data(), sizeof(float) * N);
  });
}

int ref_aux_loss(const float* probs, const std::int64_t* counts, std::int64_t B, std::int64_t N,
                 std::int64_t K, float* out) {
  return guarded([&] {
    Tensor p = Tensor::from_values({B, N}, vec(probs, B * N));
    std::vector<std::int64_t> c(counts, counts + N);
    *out = ops::moe_aux_loss(p, c, K).scalar();
  });
}

int ref_z_loss(const float* logits, std::int64_t B, std::int64_t N, float* out) {
  return guarded([&] { *out = ops::z_loss(Tensor::from_values({B, N}, vec(logits, B * N))).scalar(); });
}

int ref_top_k(const float* x, std::int64_t n, std::int64_t k, std::int64_t* idx, float* val) {
  return guarded([&] { ops::top_k(x, n, k, idx, val); });
}

// moe_forward: per expert gather_rows -> matmul -> slice_cols x2 -> silu -> mul
// -> matmul -> mul_rowwise -> scatter_add_rows; experts fanned out with the reference's own
// parallel_for (common.cpp:141-168); outputs summed with ops::add in expert order.
int ref_moe_forward(const float* x, std::int64_t T, std::int64_t d, std::int64_t N, std::int64_t K,
                    std::int64_t f, const float* w_in, const float* w_out, const std::int64_t* idx,
                    const float* w, float* out, int jobs) {
  return guarded([&] {
    Tensor xt = Tensor::from_values({T, d}, vec(x, T * d));
    std::vector<std::vector<std::int64_t>> rows(static_cast<std::size_t>(N));
    std::vector<std::vector<float>> wcol(static_cast<std::size_t>(N));
    for (std::int64_t j = 0; j < T; ++j)
      for (std::int64_t k = 0; k < K; ++k) {
        rows[static_cast<std::size_t>(idx[j * K + k])].push_back(j);
        wcol[static_cast<std::size_t>(idx[j * K + k])].push_back(w[j * K + k]);
      }
    std::vector<Tensor> contrib(static_cast<std::size_t>(N));
    compasslab::parallel_for(static_cast<std::size_t>(N), jobs, [&](std::size_t e) {
      if (rows[e].empty()) return;
      const auto m = static_cast<std::int64_t>(rows[e].size());
      Tensor win = Tensor::from_values({d, 2 * f}, vec(w_in + static_cast<std::int64_t>(e) * d * 2 * f, d * 2 * f));
      Tensor wout = Tensor::from_values({f, d}, vec(w_out + static_cast<std::int64_t>(e) * f * d, f * d));
      Tensor xe = ops::gather_rows(xt, rows[e]);
      Tensor h = ops::matmul(xe, win);
      Tensor a = ops::mul(ops::silu(ops::slice_cols(h, 0, f)), ops::slice_cols(h, f, 2 * f));
      Tensor y = ops::matmul(a, wout);
      Tensor yw = ops::mul_rowwise(y, Tensor::from_values({m, 1}, wcol[e]));
      contrib[e] = ops::scatter_add_rows(T, yw, rows[e]);
    });
    Tensor acc = Tensor::zeros({T, d});
    for (std::int64_t e = 0; e < N; ++e)
      if (contrib[static_cast<std::size_t>(e)].defined()) acc = ops::add(acc, contrib[static_cast<std::size_t>(e)]);
    std::memcpy(out, acc.values().data(), sizeof(float) * T * d);
  });
}

// Expert-FFN backward through the reference Tape (tensor.cpp:133-150): loss = sum(Y * stop(dY))
// seeds dL/dY = dY exactly; the Tape then replays matmul/mul/silu/slice_cols backward closures.
int ref_expert_ffn_backward(const float* xe, std::int64_t m, std::int64_t d, std::int64_t f,
                            const float* w_in, const float* w_out, const float* dy, float* dx,
                            float* dw_in, float* dw_out) {
  return guarded([&] {
    Tensor x = Tensor::param({m, d}, vec(xe, m * d));
    Tensor win = Tensor::param({d, 2 * f}, vec(w_in, d * 2 * f));
    Tensor wout = Tensor::param({f, d}, vec(w_out, f * d));
    Tensor g = Tensor::from_values({m, d}, vec(dy, m * d));
    Tape tape;
    Tape::Scope scope(tape);
    Tensor h = ops::matmul(x, win);
    Tensor a = ops::mul(ops::silu(ops::slice_cols(h, 0, f)), ops::slice_cols(h, f, 2 * f));
    Tensor y = ops::matmul(a, wout);
    Tensor loss = ops::sum_all(ops::mul(y, ops::stop_grad(g)));
    tape.backward(loss);
    std::memcpy(dx, x.grad().data(), sizeof(float) * m * d);
    std::memcpy(dw_in, win.grad().data(), sizeof(float) * d * 2 * f);
    std::memcpy(dw_out, wout.grad().data(), sizeof(float) * f * d);
  });
}

// Full MoE layer backward through the reference Tape: forward composed as in ref_moe_forward
// (sequential over experts so the tape is single-threaded), loss = sum(out * stop(dOut)), with
// x, every expert's W_in / W_out and the combine-weight columns as leaves.
int ref_moe_backward(const float* x, std::int64_t T, std::int64_t d, std::int64_t N, std::int64_t K, std::int64_t f,
                     const float* w_in, const float* w_out, const std::int64_t* idx, const float* w,
                     const float* d_out, float* d_hidden, float* d_combine_w, float* dw_in, float* dw_out) {
  return guarded([&] {
    Tensor xt = Tensor::param({T, d}, vec(x, T * d));
    std::vector<std::vector<std::int64_t>> rows(static_cast<std::size_t>(N)), slot(static_cast<std::size_t>(N));
    std::vector<std::vector<float>> wcol(static_cast<std::size_t>(N));
    for (std::int64_t j = 0; j < T; ++j)
      for (std::int64_t k = 0; k < K; ++k) {
        rows[static_cast<std::size_t>(idx[j * K + k])].push_back(j);
        slot[static_cast<std::size_t>(idx[j * K + k])].push_back(j * K + k);
        wcol[static_cast<std::size_t>(idx[j * K + k])].push_back(w[j * K + k]);
      }
    std::vector<Tensor> win(static_cast<std::size_t>(N)), wout(static_cast<std::size_t>(N)), wc(static_cast<std::size_t>(N));
    Tape tape;
    Tape::Scope scope(tape);
    Tensor acc = Tensor::zeros({T, d});
    for (std::int64_t e = 0; e < N; ++e) {
      win[static_cast<std::size_t>(e)] = Tensor::param({d, 2 * f}, vec(w_in + e * d * 2 * f, d * 2 * f));
      wout[static_cast<std::size_t>(e)] = Tensor::param({f, d}, vec(w_out + e * f * d, f * d));
      const auto& re = rows[static_cast<std::size_t>(e)];
      if (re.empty()) continue;
      const auto m = static_cast<std::int64_t>(re.size());
      wc[static_cast<std::size_t>(e)] = Tensor::param({m, 1}, wcol[static_cast<std::size_t>(e)]);
      Tensor xe = ops::gather_rows(xt, re);
      Tensor h = ops::matmul(xe, win[static_cast<std::size_t>(e)]);
      Tensor a = ops::mul(ops::silu(ops::slice_cols(h, 0, f)), ops::slice_cols(h, f, 2 * f));
      Tensor y = ops::matmul(a, wout[static_cast<std::size_t>(e)]);
      Tensor yw = ops::mul_rowwise(y, wc[static_cast<std::size_t>(e)]);
      acc = ops::add(acc, ops::scatter_add_rows(T, yw, re));
    }
    Tensor g = Tensor::from_values({T, d}, vec(d_out, T * d));
    tape.backward(ops::sum_all(ops::mul(acc, ops::stop_grad(g))));
    std::memcpy(d_hidden, xt.grad().data(), sizeof(float) * T * d);
    for (std::int64_t e = 0; e < N; ++e) {
      std::memcpy(dw_in + e * d * 2 * f, win[static_cast<std::size_t>(e)].grad().data(), sizeof(float) * d * 2 * f);
      std::memcpy(dw_out + e * f * d, wout[static_cast<std::size_t>(e)].grad().data(), sizeof(float) * f * d);
      const auto& se = slot[static_cast<std::size_t>(e)];
      if (se.empty()) continue;
      const auto& gw = wc[static_cast<std::size_t>(e)].grad();
      for (std::size_t r = 0; r < se.size(); ++r) d_combine_w[se[r]] = gw[r];
    }
  });
}

// Full training step of the layer through the reference Tape, router included:
//   z = matmul(x, W_r); p = softmax_rows(z); vals = gather_cols_per_row(p, idx, K);
//   w = mul_rowwise(vals, recip(row_sums(vals)))          (renormalised top-K, differentiable)
//   per expert: w_e = gather_elems_col(w, slots_e), the expert chain, mul_rowwise(y, w_e),
//   scatter_add_rows, add; loss = sum(out * stop(dOut)) + g_aux * moe_aux_loss(p, c, K)
//   + g_z * z_loss(z). Outputs dx, dW_r, dW_in, dW_out.
int ref_moe_backward_full(const float* x, const float* wr, std::int64_t T, std::int64_t d, std::int64_t N,
                          std::int64_t K, std::int64_t f, const float* w_in, const float* w_out, const float* d_out,
                          float g_aux, float g_z, float* d_hidden, float* dw_router, float* dw_in, float* dw_out) {
  return guarded([&] {
    Tensor xt = Tensor::param({T, d}, vec(x, T * d));
    Tensor wrt = Tensor::param({d, N}, vec(wr, d * N));
    std::vector<Tensor> win(static_cast<std::size_t>(N)), wout(static_cast<std::size_t>(N));
    Tape tape;
    Tape::Scope scope(tape);
    Tensor z = ops::matmul(xt, wrt);
    Tensor p = ops::softmax_rows(z);
    std::vector<std::int64_t> idx(static_cast<std::size_t>(T * K));
    std::vector<float> val(static_cast<std::size_t>(K));
    std::vector<std::int64_t> counts(static_cast<std::size_t>(N), 0);
    for (std::int64_t j = 0; j < T; ++j) {
      ops::top_k(p.values().data() + j * N, N, K, idx.data() + j * K, val.data());
      for (std::int64_t k = 0; k < K; ++k) counts[static_cast<std::size_t>(idx[j * K + k])] += 1;
    }
    Tensor vals = ops::gather_cols_per_row(p, idx, K);
    Tensor w = ops::mul_rowwise(vals, ops::recip(ops::row_sums(vals)));
    std::vector<std::vector<std::int64_t>> rows(static_cast<std::size_t>(N));
    std::vector<std::vector<std::pair<std::int64_t, std::int64_t>>> coords(static_cast<std::size_t>(N));
    for (std::int64_t j = 0; j < T; ++j)
      for (std::int64_t k = 0; k < K; ++k) {
        rows[static_cast<std::size_t>(idx[j * K + k])].push_back(j);
        coords[static_cast<std::size_t>(idx[j * K + k])].push_back({j, k});
      }
    Tensor acc = Tensor::zeros({T, d});
    for (std::int64_t e = 0; e < N; ++e) {
      win[static_cast<std::size_t>(e)] = Tensor::param({d, 2 * f}, vec(w_in + e * d * 2 * f, d * 2 * f));
      wout[static_cast<std::size_t>(e)] = Tensor::param({f, d}, vec(w_out + e * f * d, f * d));
      const auto& re = rows[static_cast<std::size_t>(e)];
      if (re.empty()) continue;
      Tensor xe = ops::gather_rows(xt, re);
      Tensor h = ops::matmul(xe, win[static_cast<std::size_t>(e)]);
      Tensor a = ops::mul(ops::silu(ops::slice_cols(h, 0, f)), ops::slice_cols(h, f, 2 * f));
      Tensor y = ops::matmul(a, wout[static_cast<std::size_t>(e)]);
      Tensor yw = ops::mul_rowwise(y, ops::gather_elems_col(w, coords[static_cast<std::size_t>(e)]));
      acc = ops::add(acc, ops::scatter_add_rows(T, yw, re));
    }
    Tensor g = Tensor::from_values({T, d}, vec(d_out, T * d));
    Tensor loss = ops::add(ops::add(ops::sum_all(ops::mul(acc, ops::stop_grad(g))),
                                    ops::scale(ops::moe_aux_loss(p, counts, K), g_aux)),
                           ops::scale(ops::z_loss(z), g_z));
    tape.backward(loss);
    std::memcpy(d_hidden, xt.grad().data(), sizeof(float) * T * d);
    std::memcpy(dw_router, wrt.grad().data(), sizeof(float) * d * N);
    for (std::int64_t e = 0; e < N; ++e) {
      std::memcpy(dw_in + e * d * 2 * f, win[static_cast<std::size_t>(e)].grad().data(), sizeof(float) * d * 2 * f);
      std::memcpy(dw_out + e * f * d, wout[static_cast<std::size_t>(e)].grad().data(), sizeof(float) * f * d);
    }
  });
}

// The reference's own finite-difference gradient suite (gradcheck.cpp:610-656); returns the
// number of failing ops (0 = all pass) and the number of ops checked in *n_ops.
// The reference's own checkpoint code (proj/src/checkpoint.cpp): load `in_path`, save it again to
// `out_path`. A file our writer made is byte-identical to its reference re-save iff the two
// writers agree; a load failure surfaces the reference's validation message.
int ref_ckpt_resave(const char* in_path, const char* out_path) {
  return guarded([&] { compasslab::save_checkpoint(out_path, compasslab::load_checkpoint(in_path)); });
}

// Writes tensors with the reference's save_checkpoint: names joined by '\n', shapes as
// (rank, dims...) int64 records, values concatenated in the same order.
int ref_ckpt_write(const char* out_path, const char* names, const std::int64_t* shapes, const float* values) {
  return guarded([&] {
    std::map<std::string, Tensor> ts;
    std::string all(names);
    size_t pos = 0;
    const std::int64_t* sp = shapes;
    const float* vp = values;
    while (pos <= all.size() && !all.empty()) {
      const size_t nl = all.find('\n', pos);
      const std::string name = all.substr(pos, nl == std::string::npos ? std::string::npos : nl - pos);
      const std::int64_t rank = *sp++;
      compasslab::Shape shape(sp, sp + rank);
      sp += rank;
      std::int64_t n = 1;
      for (auto e : shape) n *= e;
      ts.emplace(name, Tensor::from_values(shape, vec(vp, n)));
      vp += n;
      if (nl == std::string::npos) break;
      pos = nl + 1;
    }
    compasslab::save_checkpoint(out_path, ts);
  });
}

int ref_gradcheck(std::uint64_t seed, int cases, double tol, int* n_ops) {
  const auto res = compasslab::run_gradcheck(seed, cases, tol);
  int fails = 0;
  for (const auto& r : res) fails += r.pass ? 0 : 1;
  *n_ops = static_cast<int>(res.size());
  return fails;
}

}  // extern "C"
