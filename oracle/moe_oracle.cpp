// ORACLE — TEST INFRASTRUCTURE ONLY.
//
// CPU restatement of the reference (compass-lab, /root/reference/proj) arithmetic for the
// MoE-layer hot path: route_tokens / moe_forward / aux_loss / z_loss and the
// E4M3 quantize-dequantize of the expert-quantizer, composed exactly the way
// the reference's own primitives compute them (proj/src/tensor.cpp). Only tests/, bench.py's
// cpu_baseline leg and __graft_entry__.smoke() may load this library, and only as the checker.
// The product path (paper_2509_09121_b200/) never links or calls it.
//
// Parity pin: tests/test_oracle.py checks every function here against (a) the SPEC examples,
// (b) the reference's own unit-test cases for top_k / softmax / gather-scatter
// (proj/tests/tensor_test.cpp:98-199, :344-353), (c) golden vectors in tests/golden/ produced by
// oracle/_ref (the reference's own tensor.cpp compiled from /root/reference, composed by
// oracle/ref_compose.cpp), and (d) oracle/_ref directly, bit-for-bit, when it is built.
//
// Every function names the reference file:line whose arithmetic (accumulation type and order,
// casts, tie rules) it restates.

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

namespace {

thread_local std::string g_err;

int fail(const char* msg) {
  g_err = msg;
  return 1;
}

// ---- splitmix64 counter PRNG (proj/include/compasslab/prng.hpp:15-70) ----
constexpr std::uint64_t kGolden = 0x9e3779b97f4a7c15ull;
constexpr double kPi = 3.14159265358979323846;

inline std::uint64_t mix64(std::uint64_t x) {  // prng.hpp:20-24
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

// Draw number `ctr` (1-based) of stream `seed` as a double in [0,1) (prng.hpp:29-37).
inline double draw_double(std::uint64_t seed, std::uint64_t ctr) {
  return static_cast<double>(mix64(seed + ctr * kGolden) >> 11) * 0x1.0p-53;
}

// Non-finite check applied to every op output (tensor.cpp:35-41).
bool all_finite(const float* v, std::size_t n) {
  for (std::size_t i = 0; i < n; ++i)
    if (!std::isfinite(v[i])) return false;
  return true;
}

// stable_sigmoid in double (tensor.cpp:51-55).
inline double stable_sigmoid(double x) {
  if (x >= 0.0) return 1.0 / (1.0 + std::exp(-x));
  const double e = std::exp(x);
  return e / (1.0 + e);
}

// C[m x n] = A[m x k] B[k x n]; one double accumulator per output, summed over l ascending,
// then cast to float (gemm_nn, tensor.cpp:157-173). Rows of C are independent, so a caller may
// split rows across threads without changing any result bit.
void gemm_nn(const float* a, const float* b, std::int64_t m, std::int64_t k, std::int64_t n,
             float* out) {
  std::vector<double> row(static_cast<std::size_t>(n));
  for (std::int64_t i = 0; i < m; ++i) {
    std::fill(row.begin(), row.end(), 0.0);
    const float* ai = a + i * k;
    for (std::int64_t l = 0; l < k; ++l) {
      const double av = ai[l];
      const float* bl = b + l * n;
      double* r = row.data();
      for (std::int64_t j = 0; j < n; ++j) r[j] += av * static_cast<double>(bl[j]);
    }
    float* oi = out + i * n;
    for (std::int64_t j = 0; j < n; ++j) oi[j] = static_cast<float>(row[static_cast<std::size_t>(j)]);
  }
}

// C[m x k] = A[m x n] B^T, B is [k x n] (gemm_nt, tensor.cpp:176-189).
void gemm_nt(const float* a, const float* b, std::int64_t m, std::int64_t n, std::int64_t k,
             float* out) {
  for (std::int64_t i = 0; i < m; ++i) {
    const float* ai = a + i * n;
    for (std::int64_t l = 0; l < k; ++l) {
      const float* bl = b + l * n;
      double acc = 0.0;
      for (std::int64_t j = 0; j < n; ++j) acc += static_cast<double>(ai[j]) * bl[j];
      out[i * k + l] = static_cast<float>(acc);
    }
  }
}

// C[k x n] = A^T B, A is [m x k], B is [m x n]; double accumulators summed over i ascending
// (gemm_tn, tensor.cpp:192-206).
void gemm_tn(const float* a, const float* b, std::int64_t m, std::int64_t k, std::int64_t n,
             float* out) {
  std::vector<double> acc(static_cast<std::size_t>(k * n), 0.0);
  for (std::int64_t i = 0; i < m; ++i) {
    const float* ai = a + i * k;
    const float* bi = b + i * n;
    for (std::int64_t l = 0; l < k; ++l) {
      const double av = ai[l];
      double* al = acc.data() + l * n;
      for (std::int64_t j = 0; j < n; ++j) al[j] += av * bi[j];
    }
  }
  for (std::size_t i = 0; i < acc.size(); ++i) out[i] = static_cast<float>(acc[i]);
}

// Runs fn(0..n-1) on `jobs` threads, each index owning its output slot (common.cpp:141-168).
template <typename Fn>
void run_parallel(std::int64_t n, int jobs, Fn fn) {
  if (n <= 0) return;
  const int workers = std::max(1, std::min<int>(jobs, static_cast<int>(n)));
  if (workers == 1) {
    for (std::int64_t i = 0; i < n; ++i) fn(i);
    return;
  }
  std::atomic<std::int64_t> next{0};
  std::vector<std::thread> ts;
  for (int w = 0; w < workers; ++w)
    ts.emplace_back([&]() {
      for (;;) {
        const std::int64_t i = next.fetch_add(1);
        if (i >= n) return;
        fn(i);
      }
    });
  for (auto& t : ts) t.join();
}

// E4M3 grid: code c in [0,126] -> value; 127 is NaN and never produced.
float e4m3_value(int c) {
  const int e = c >> 3, m = c & 7;
  if (e == 0) return std::ldexp(static_cast<float>(m), -9);
  return std::ldexp(1.0f + static_cast<float>(m) / 8.0f, e - 7);
}

}  // namespace

extern "C" {

const char* orc_last_error(void) { return g_err.c_str(); }

// ---- PRNG -----------------------------------------------------------------------------------

// Prng(root).split(stream).seed() (prng.hpp:60-62).
std::uint64_t orc_split_seed(std::uint64_t root, std::uint64_t stream) {
  return mix64(root ^ mix64(stream * kGolden + 0x632be59bd9b4e019ull));
}

// n calls of Prng(seed).next_normal_f(mean, stddev) (prng.hpp:48-56): Box-Muller, two draws per
// value, value i uses counters 2i+1 and 2i+2.
void orc_normals(std::uint64_t seed, std::int64_t n, float mean, float stddev, float* out) {
  for (std::int64_t i = 0; i < n; ++i) {
    const std::uint64_t c = 2 * static_cast<std::uint64_t>(i);
    const double u1 = 1.0 - draw_double(seed, c + 1);
    const double u2 = draw_double(seed, c + 2);
    const double z = std::sqrt(-2.0 * std::log(u1)) * std::cos(2.0 * kPi * u2);
    out[i] = mean + stddev * static_cast<float>(z);
  }
}

// fp32 -> bf16 (round to nearest even) -> fp32. Used to hand the oracle the exact values the
// bf16 device path consumes.
void orc_round_bf16(const float* in, float* out, std::int64_t n) {
  for (std::int64_t i = 0; i < n; ++i) {
    std::uint32_t u;
    std::memcpy(&u, &in[i], 4);
    if ((u & 0x7f800000u) != 0x7f800000u) u += 0x7fffu + ((u >> 16) & 1u);
    u &= 0xffff0000u;
    std::memcpy(&out[i], &u, 4);
  }
}

// ---- primitives (exported for primitive-level tests) -------------------------------------

// ops::matmul forward (tensor.cpp:350-375 -> gemm_nn :157-173).
int orc_matmul(const float* a, const float* b, std::int64_t m, std::int64_t k, std::int64_t n,
               float* out) {
  gemm_nn(a, b, m, k, n, out);
  return all_finite(out, static_cast<std::size_t>(m * n)) ? 0 : fail("non-finite value produced by op 'matmul'");
}

// ops::softmax_rows (tensor.cpp:614-621, :633-655): double max, double exp-sum in column order,
// each output exp(x-max)/denom cast to float.
int orc_softmax_rows(const float* x, std::int64_t r, std::int64_t c, float* out) {
  for (std::int64_t i = 0; i < r; ++i) {
    const float* xi = x + i * c;
    double mx = xi[0];
    for (std::int64_t j = 1; j < c; ++j) mx = std::max(mx, static_cast<double>(xi[j]));
    double denom = 0.0;
    for (std::int64_t j = 0; j < c; ++j) denom += std::exp(static_cast<double>(xi[j]) - mx);
    for (std::int64_t j = 0; j < c; ++j)
      out[i * c + j] = static_cast<float>(std::exp(static_cast<double>(xi[j]) - mx) / denom);
  }
  return all_finite(out, static_cast<std::size_t>(r * c)) ? 0 : fail("non-finite value produced by op 'softmax_rows'");
}

// ops::top_k (tensor.cpp:1046-1060): k largest, ties to the lowest index, output in descending
// (value, then ascending index) order; k outside [1, n] is a ValidationError (returned as 1).
int orc_top_k(const float* x, std::int64_t n, std::int64_t k, std::int64_t* out_idx, float* out_val) {
  if (k < 1 || k > n) return fail("top_k: k out of range");
  std::vector<char> taken(static_cast<std::size_t>(n), 0);
  for (std::int64_t s = 0; s < k; ++s) {
    std::int64_t best = -1;
    for (std::int64_t j = 0; j < n; ++j) {
      if (taken[static_cast<std::size_t>(j)]) continue;
      if (best < 0 || x[j] > x[best]) best = j;  // strict '>' keeps the lowest index on ties
    }
    taken[static_cast<std::size_t>(best)] = 1;
    out_idx[s] = best;
    out_val[s] = x[best];
  }
  return 0;
}

// ---- route_tokens -----------------------------------
// logits = matmul(x, W_r) (fp64 accumulate), probs = softmax_rows(logits), per token top_k on the
// fp32 probs, combine_w[k] = (float)((double)val[k] / sum_k (double)val[k]), counts c_i, and
// agg_prob p = col_sums(probs) (tensor.cpp:545-565: double sums over tokens ascending -> float).
int orc_route(const float* x, const float* wr, std::int64_t T, std::int64_t d, std::int64_t N,
              std::int64_t K, float* logits, float* probs, std::int64_t* idx, float* w,
              std::int64_t* counts, float* agg_prob) {
  if (T < 1) return fail("route_tokens: B must be >= 1");
  if (orc_matmul(x, wr, T, d, N, logits)) return 1;
  if (orc_softmax_rows(logits, T, N, probs)) return 1;
  std::vector<float> val(static_cast<std::size_t>(K));
  for (std::int64_t i = 0; i < N; ++i) counts[i] = 0;
  for (std::int64_t j = 0; j < T; ++j) {
    if (orc_top_k(probs + j * N, N, K, idx + j * K, val.data())) return 1;
    double s = 0.0;
    for (std::int64_t k = 0; k < K; ++k) s += static_cast<double>(val[static_cast<std::size_t>(k)]);
    for (std::int64_t k = 0; k < K; ++k) {
      w[j * K + k] = static_cast<float>(static_cast<double>(val[static_cast<std::size_t>(k)]) / s);
      counts[idx[j * K + k]] += 1;
    }
  }
  std::vector<double> acc(static_cast<std::size_t>(N), 0.0);
  for (std::int64_t j = 0; j < T; ++j)
    for (std::int64_t i = 0; i < N; ++i) acc[static_cast<std::size_t>(i)] += probs[j * N + i];
  for (std::int64_t i = 0; i < N; ++i) agg_prob[i] = static_cast<float>(acc[static_cast<std::size_t>(i)]);
  return 0;
}

// ops::moe_aux_loss (tensor.cpp:980-1009): coef = N/(B^2 K); sum_i (sum_j probs[j][i]) * c_i,
// every sum in double; result cast to float.
int orc_aux_loss(const float* probs, const std::int64_t* counts, std::int64_t B, std::int64_t N,
                 std::int64_t K, float* out) {
  if (B == 0) return fail("moe_aux_loss: empty batch");
  const double coef = static_cast<double>(N) / (static_cast<double>(B) * B * static_cast<double>(K));
  double acc = 0.0;
  for (std::int64_t i = 0; i < N; ++i) {
    double p = 0.0;
    for (std::int64_t j = 0; j < B; ++j) p += probs[j * N + i];
    acc += p * static_cast<double>(counts[i]);
  }
  *out = static_cast<float>(coef * acc);
  return 0;
}

// ops::z_loss (tensor.cpp:1011-1040 with row_logsumexp :623-629): mean over rows of lse^2, all
// in double, cast to float.
int orc_z_loss(const float* logits, std::int64_t B, std::int64_t N, float* out) {
  if (B == 0) return fail("z_loss: empty batch");
  double acc = 0.0;
  for (std::int64_t j = 0; j < B; ++j) {
    const float* x = logits + j * N;
    double mx = x[0];
    for (std::int64_t i = 1; i < N; ++i) mx = std::max(mx, static_cast<double>(x[i]));
    double denom = 0.0;
    for (std::int64_t i = 0; i < N; ++i) denom += std::exp(static_cast<double>(x[i]) - mx);
    const double l = mx + std::log(denom);
    acc += l * l;
  }
  *out = static_cast<float>(acc / static_cast<double>(B));
  return 0;
}

// ---- dispatch plan ---------------------------------------------------
// Expert-major, token-ascending within an expert: a stable counting sort of the (j,k) slots in
// token-major order. offsets = exclusive prefix sum of counts (N+1 entries); perm[r] = j*K+k;
// inv[j*K+k] = r. This is exactly the row order of the per-expert index lists the reference
// composition hands to gather_rows (tensor.cpp:784-812).
void orc_plan(const std::int64_t* idx, std::int64_t T, std::int64_t N, std::int64_t K,
              std::int64_t* offsets, std::int64_t* perm, std::int64_t* inv) {
  std::vector<std::int64_t> cursor(static_cast<std::size_t>(N) + 1, 0);
  for (std::int64_t s = 0; s < T * K; ++s) cursor[static_cast<std::size_t>(idx[s]) + 1] += 1;
  for (std::int64_t e = 0; e < N; ++e) cursor[static_cast<std::size_t>(e) + 1] += cursor[static_cast<std::size_t>(e)];
  for (std::int64_t e = 0; e <= N; ++e) offsets[e] = cursor[static_cast<std::size_t>(e)];
  for (std::int64_t s = 0; s < T * K; ++s) {
    const std::int64_t r = cursor[static_cast<std::size_t>(idx[s])]++;
    perm[r] = s;
    inv[s] = r;
  }
}

// ---- expert FFN for one expert ("gated two-matrix feed-forward") ---------------
// H = X_e W_in (gemm_nn), G = H[:, :f], U = H[:, f:] (slice_cols tensor.cpp:398-420),
// A = silu(G) * U (silu tensor.cpp:315-322 via unary_op :227-244: float(x * sigmoid_d(x)); mul
// :283-303 in float), Y = A W_out (gemm_nn). Writes A [m x f] (if non-null) and Y [m x d].
int orc_expert_ffn(const float* xe, std::int64_t m, std::int64_t d, std::int64_t f,
                   const float* w_in, const float* w_out, float* a_out, float* y_out) {
  std::vector<float> h(static_cast<std::size_t>(m * 2 * f));
  gemm_nn(xe, w_in, m, d, 2 * f, h.data());
  if (!all_finite(h.data(), h.size())) return fail("non-finite value produced by op 'matmul'");
  std::vector<float> a(static_cast<std::size_t>(m * f));
  for (std::int64_t r = 0; r < m; ++r)
    for (std::int64_t c = 0; c < f; ++c) {
      const float g = h[static_cast<std::size_t>(r * 2 * f + c)];
      const float u = h[static_cast<std::size_t>(r * 2 * f + f + c)];
      const float s = static_cast<float>(g * stable_sigmoid(g));
      a[static_cast<std::size_t>(r * f + c)] = s * u;
    }
  if (!all_finite(a.data(), a.size())) return fail("non-finite value produced by op 'mul'");
  gemm_nn(a.data(), w_out, m, f, d, y_out);
  if (!all_finite(y_out, static_cast<std::size_t>(m * d))) return fail("non-finite value produced by op 'matmul'");
  if (a_out) std::memcpy(a_out, a.data(), a.size() * sizeof(float));
  return 0;
}

// ---- moe_forward --------------------------------
// For every expert e with at least one token (gather_rows rejects an empty index list,
// tensor.cpp:13-20): rows_e = ascending tokens routed to e, X_e = gather_rows(x, rows_e),
// Y_e = expert_ffn(X_e), Yw = mul_rowwise(Y_e, w[rows_e]) (tensor.cpp:572-610, float product),
// out = add(out, scatter_add_rows(T, Yw, rows_e)) in expert order (tensor.cpp:814-845, :248-262).
// Experts run on `jobs` threads (the reference's parallel_for fan-out); the cross-expert sum is
// taken afterwards in expert order, so the result does not depend on `jobs`.
// w_in is [N][d][2f], w_out is [N][f][d] (reference row-major layout).
int orc_moe_forward(const float* x, std::int64_t T, std::int64_t d, std::int64_t N, std::int64_t K,
                    std::int64_t f, const float* w_in, const float* w_out, const std::int64_t* idx,
                    const float* w, float* out, int jobs) {
  std::vector<std::vector<std::int64_t>> rows(static_cast<std::size_t>(N));
  std::vector<std::vector<float>> wcol(static_cast<std::size_t>(N));
  for (std::int64_t j = 0; j < T; ++j)
    for (std::int64_t k = 0; k < K; ++k) {
      const std::int64_t e = idx[j * K + k];
      if (e < 0 || e >= N) return fail("moe_forward: expert index out of range");
      rows[static_cast<std::size_t>(e)].push_back(j);
      wcol[static_cast<std::size_t>(e)].push_back(w[j * K + k]);
    }
  std::vector<std::vector<float>> yw(static_cast<std::size_t>(N));
  std::atomic<int> bad{0};
  run_parallel(N, jobs, [&](std::int64_t e) {
    const auto& re = rows[static_cast<std::size_t>(e)];
    const std::int64_t m = static_cast<std::int64_t>(re.size());
    if (m == 0) return;
    std::vector<float> xe(static_cast<std::size_t>(m * d));
    for (std::int64_t r = 0; r < m; ++r)
      std::memcpy(&xe[static_cast<std::size_t>(r * d)], x + re[static_cast<std::size_t>(r)] * d, d * sizeof(float));
    auto& y = yw[static_cast<std::size_t>(e)];
    y.resize(static_cast<std::size_t>(m * d));
    if (orc_expert_ffn(xe.data(), m, d, f, w_in + e * d * 2 * f, w_out + e * f * d, nullptr, y.data())) {
      bad = 1;
      return;
    }
    const auto& wc = wcol[static_cast<std::size_t>(e)];
    for (std::int64_t r = 0; r < m; ++r)
      for (std::int64_t c = 0; c < d; ++c) y[static_cast<std::size_t>(r * d + c)] *= wc[static_cast<std::size_t>(r)];
  });
  if (bad) return fail("moe_forward: non-finite value produced by an expert");
  std::memset(out, 0, static_cast<std::size_t>(T * d) * sizeof(float));
  for (std::int64_t e = 0; e < N; ++e) {
    const auto& re = rows[static_cast<std::size_t>(e)];
    const auto& y = yw[static_cast<std::size_t>(e)];
    for (std::size_t r = 0; r < re.size(); ++r) {
      float* o = out + re[r] * d;
      const float* s = y.data() + r * static_cast<std::size_t>(d);
      for (std::int64_t c = 0; c < d; ++c) o[c] = o[c] + s[c];
    }
  }
  return all_finite(out, static_cast<std::size_t>(T * d)) ? 0 : fail("non-finite value produced by op 'add'");
}

// ---- expert FFN backward for one expert (the Tape replay of tensor.cpp:364-372, :318-321,
// :290-300, :411-418 for the composition in orc_expert_ffn) -------------------------------------
// Given X_e [m x d], dY [m x d] (gradient of Y = expert output before the combine weight):
//   dA = dY W_out^T (gemm_nt), dW_out = A^T dY (gemm_tn),
//   dG = dA * U * silu'(G), dU = dA * silu(G) (mul bwd :290-300, silu bwd :318-321),
//   dH = concat(dG, dU) (slice_cols bwd :411-418), dX = dH W_in^T, dW_in = X^T dH.
int orc_expert_ffn_backward(const float* xe, std::int64_t m, std::int64_t d, std::int64_t f,
                            const float* w_in, const float* w_out, const float* dy, float* dx,
                            float* dw_in, float* dw_out) {
  std::vector<float> h(static_cast<std::size_t>(m * 2 * f));
  gemm_nn(xe, w_in, m, d, 2 * f, h.data());
  std::vector<float> a(static_cast<std::size_t>(m * f)), sg(static_cast<std::size_t>(m * f));
  for (std::int64_t r = 0; r < m; ++r)
    for (std::int64_t c = 0; c < f; ++c) {
      const float g = h[static_cast<std::size_t>(r * 2 * f + c)];
      const float u = h[static_cast<std::size_t>(r * 2 * f + f + c)];
      sg[static_cast<std::size_t>(r * f + c)] = static_cast<float>(g * stable_sigmoid(g));
      a[static_cast<std::size_t>(r * f + c)] = sg[static_cast<std::size_t>(r * f + c)] * u;
    }
  std::vector<float> da(static_cast<std::size_t>(m * f));
  gemm_nt(dy, w_out, m, d, f, da.data());
  gemm_tn(a.data(), dy, m, f, d, dw_out);
  std::vector<float> dh(static_cast<std::size_t>(m * 2 * f));
  for (std::int64_t r = 0; r < m; ++r)
    for (std::int64_t c = 0; c < f; ++c) {
      const std::size_t i = static_cast<std::size_t>(r * f + c);
      const float g = h[static_cast<std::size_t>(r * 2 * f + c)];
      const float u = h[static_cast<std::size_t>(r * 2 * f + f + c)];
      const float dsg = da[i] * u;  // mul bwd wrt silu(G)
      const double s = stable_sigmoid(g);
      dh[static_cast<std::size_t>(r * 2 * f + c)] = dsg * static_cast<float>(s * (1.0 + g * (1.0 - s)));
      dh[static_cast<std::size_t>(r * 2 * f + f + c)] = da[i] * sg[i];
    }
  gemm_nt(dh.data(), w_in, m, 2 * f, d, dx);
  gemm_tn(xe, dh.data(), m, d, 2 * f, dw_in);
  return 0;
}

// ---- MoE layer backward (the Tape replay of the moe_forward composition) --------------------
// Given dOut [T x d]: per expert e with rows_e (ascending tokens) and weights w_e:
//   scatter_add_rows bwd (tensor.cpp:834-842): dYw[r] = dOut[rows_e[r]]
//   mul_rowwise bwd (tensor.cpp:587-607):      dY[r] = dYw[r] * w[r] (float);
//                                              d_w[r] = (float) sum_c (double)dYw[r][c] * Y[r][c]
//   expert FFN bwd (orc_expert_ffn_backward);  dW_in[e], dW_out[e]
//   gather_rows bwd (tensor.cpp:801-809):      d_hidden[rows_e[r]] += dX[r]
// Experts are replayed in reverse creation order like Tape::backward (tensor.cpp:142-150).
// d_combine_w is indexed like topk_idx ([T][K]); dw_in [N][d][2f], dw_out [N][f][d].
int orc_moe_backward(const float* x, std::int64_t T, std::int64_t d, std::int64_t N, std::int64_t K, std::int64_t f,
                     const float* w_in, const float* w_out, const std::int64_t* idx, const float* w,
                     const float* d_out, float* d_hidden, float* d_combine_w, float* dw_in, float* dw_out, int jobs) {
  std::vector<std::vector<std::int64_t>> rows(static_cast<std::size_t>(N)), slot(static_cast<std::size_t>(N));
  for (std::int64_t j = 0; j < T; ++j)
    for (std::int64_t k = 0; k < K; ++k) {
      const std::int64_t e = idx[j * K + k];
      if (e < 0 || e >= N) return fail("moe_backward: expert index out of range");
      rows[static_cast<std::size_t>(e)].push_back(j);
      slot[static_cast<std::size_t>(e)].push_back(j * K + k);
    }
  std::vector<std::vector<float>> dx(static_cast<std::size_t>(N));
  run_parallel(N, jobs, [&](std::int64_t e) {
    const auto& re = rows[static_cast<std::size_t>(e)];
    const auto& se = slot[static_cast<std::size_t>(e)];
    const std::int64_t m = static_cast<std::int64_t>(re.size());
    float* gwi = dw_in + e * d * 2 * f;
    float* gwo = dw_out + e * f * d;
    if (m == 0) {
      std::memset(gwi, 0, sizeof(float) * d * 2 * f);
      std::memset(gwo, 0, sizeof(float) * f * d);
      return;
    }
    std::vector<float> xe(static_cast<std::size_t>(m * d)), y(static_cast<std::size_t>(m * d)),
        dy(static_cast<std::size_t>(m * d));
    for (std::int64_t r = 0; r < m; ++r)
      std::memcpy(&xe[static_cast<std::size_t>(r * d)], x + re[static_cast<std::size_t>(r)] * d, d * sizeof(float));
    orc_expert_ffn(xe.data(), m, d, f, w_in + e * d * 2 * f, w_out + e * f * d, nullptr, y.data());
    for (std::int64_t r = 0; r < m; ++r) {
      const float* g = d_out + re[static_cast<std::size_t>(r)] * d;
      const float wr = w[se[static_cast<std::size_t>(r)]];
      double acc = 0.0;
      for (std::int64_t c = 0; c < d; ++c) {
        dy[static_cast<std::size_t>(r * d + c)] = g[c] * wr;
        acc += static_cast<double>(g[c]) * y[static_cast<std::size_t>(r * d + c)];
      }
      d_combine_w[se[static_cast<std::size_t>(r)]] = static_cast<float>(acc);
    }
    auto& dxe = dx[static_cast<std::size_t>(e)];
    dxe.resize(static_cast<std::size_t>(m * d));
    orc_expert_ffn_backward(xe.data(), m, d, f, w_in + e * d * 2 * f, w_out + e * f * d, dy.data(), dxe.data(), gwi,
                            gwo);
  });
  std::memset(d_hidden, 0, sizeof(float) * T * d);
  for (std::int64_t e = N - 1; e >= 0; --e) {
    const auto& re = rows[static_cast<std::size_t>(e)];
    for (std::size_t r = 0; r < re.size(); ++r) {
      float* o = d_hidden + re[r] * d;
      const float* s = dx[static_cast<std::size_t>(e)].data() + r * static_cast<std::size_t>(d);
      for (std::int64_t c = 0; c < d; ++c) o[c] += s[c];
    }
  }
  return 0;
}

// ---- router backward --------------------------------------
// Gradient of  sum_jk d_cw[j,k] * w[j,k]  +  g_aux * L_aux  +  g_z * L_Z  with respect to the router
// logits, then through matmul(x, W_r). Analytic, in fp64 (the reference Tape composition of the
// same function -- gather_cols_per_row, row_sums, recip, mul_rowwise (tensor.cpp:847-874, :510-543,
// :324-328, :572-610), moe_aux_loss / z_loss backward (:998-1006, :1026-1037), softmax_rows
// backward (:641-652), matmul backward (:364-372) -- is compared in tests with a 1e-5 tolerance):
//   w_k = v_k / s, s = sum_k v_k, v_k = p[idx_k]:   dv_k = (d_cw_k - sum_k' d_cw_k' w_k') / s
//   dp_i = sum_{k: idx_k = i} dv_k + g_aux * N / (B^2 K) * c_i
//   dz_i = p_i (dp_i - sum_i' dp_i' p_i') + g_z * 2 lse / B * p_i
//   dx += dz W_r^T (added into dx_accum),  dW_r = x^T dz.
int orc_router_backward(const float* x, const float* wr, std::int64_t T, std::int64_t d, std::int64_t N,
                        std::int64_t K, const float* logits, const float* probs, const std::int64_t* idx,
                        const std::int64_t* counts, const float* d_cw, float g_aux, float g_z, float* dx_accum,
                        float* dw_router) {
  if (T == 0) return fail("router_backward: empty batch");
  std::vector<double> dz(static_cast<std::size_t>(T * N));
  const double coef = static_cast<double>(N) / (static_cast<double>(T) * T * static_cast<double>(K));
  for (std::int64_t j = 0; j < T; ++j) {
    const float* p = probs + j * N;
    const float* zr = logits + j * N;
    double s = 0.0;
    for (std::int64_t k = 0; k < K; ++k) s += p[idx[j * K + k]];
    double dot_w = 0.0;
    for (std::int64_t k = 0; k < K; ++k) dot_w += static_cast<double>(d_cw[j * K + k]) * (p[idx[j * K + k]] / s);
    std::vector<double> dp(static_cast<std::size_t>(N), 0.0);
    for (std::int64_t k = 0; k < K; ++k)
      dp[static_cast<std::size_t>(idx[j * K + k])] += (static_cast<double>(d_cw[j * K + k]) - dot_w) / s;
    for (std::int64_t i = 0; i < N; ++i) dp[static_cast<std::size_t>(i)] += g_aux * coef * static_cast<double>(counts[i]);
    double dot = 0.0;
    for (std::int64_t i = 0; i < N; ++i) dot += dp[static_cast<std::size_t>(i)] * p[i];
    double mx = zr[0];
    for (std::int64_t i = 1; i < N; ++i) mx = std::max(mx, static_cast<double>(zr[i]));
    double den = 0.0;
    for (std::int64_t i = 0; i < N; ++i) den += std::exp(static_cast<double>(zr[i]) - mx);
    const double lse = mx + std::log(den);
    for (std::int64_t i = 0; i < N; ++i)
      dz[static_cast<std::size_t>(j * N + i)] =
          p[i] * (dp[static_cast<std::size_t>(i)] - dot) + g_z * 2.0 * lse / static_cast<double>(T) * p[i];
  }
  for (std::int64_t j = 0; j < T; ++j)
    for (std::int64_t l = 0; l < d; ++l) {
      double a = 0.0;
      for (std::int64_t i = 0; i < N; ++i) a += dz[static_cast<std::size_t>(j * N + i)] * wr[l * N + i];
      dx_accum[j * d + l] = static_cast<float>(dx_accum[j * d + l] + a);
    }
  std::vector<double> acc(static_cast<std::size_t>(d * N), 0.0);
  for (std::int64_t j = 0; j < T; ++j)
    for (std::int64_t l = 0; l < d; ++l) {
      const double xv = x[j * d + l];
      for (std::int64_t i = 0; i < N; ++i) acc[static_cast<std::size_t>(l * N + i)] += xv * dz[static_cast<std::size_t>(j * N + i)];
    }
  for (std::size_t i = 0; i < acc.size(); ++i) dw_router[i] = static_cast<float>(acc[i]);
  return 0;
}

// ---- unified smoothing -------------------------------------------------------
// compute_smoothing: s_j = max|X_j|^alpha / (max|W_j|)^(1-alpha), W_j = row j of every expert's W_in
// AND of W_r (joint maximum); zero-max channels get s = 1.
void orc_compute_smoothing(const float* x, std::int64_t T, std::int64_t d, std::int64_t N, std::int64_t f,
                           const float* w_in, const float* wr, float alpha, float* s) {
  for (std::int64_t l = 0; l < d; ++l) {
    float xm = 0.0f, wm = 0.0f;
    for (std::int64_t j = 0; j < T; ++j) xm = std::max(xm, std::fabs(x[j * d + l]));
    for (std::int64_t e = 0; e < N; ++e)
      for (std::int64_t c = 0; c < 2 * f; ++c) wm = std::max(wm, std::fabs(w_in[(e * d + l) * 2 * f + c]));
    for (std::int64_t i = 0; i < N; ++i) wm = std::max(wm, std::fabs(wr[l * N + i]));
    s[l] = (xm > 0.0f && wm > 0.0f)
               ? static_cast<float>(std::pow(static_cast<double>(xm), alpha) / std::pow(static_cast<double>(wm), 1.0 - alpha))
               : 1.0f;
  }
}

// fold_smoothing: gain <- gain / s (upstream: inputs become x / s), W_in rows and W_r rows <- * s.
void orc_fold_smoothing(const float* s, std::int64_t d, std::int64_t N, std::int64_t f, float* w_in, float* wr,
                        float* x, std::int64_t T) {
  for (std::int64_t e = 0; e < N; ++e)
    for (std::int64_t l = 0; l < d; ++l)
      for (std::int64_t c = 0; c < 2 * f; ++c) w_in[(e * d + l) * 2 * f + c] *= s[l];
  for (std::int64_t l = 0; l < d; ++l)
    for (std::int64_t i = 0; i < N; ++i) wr[l * N + i] *= s[l];
  for (std::int64_t j = 0; j < T; ++j)
    for (std::int64_t l = 0; l < d; ++l) x[j * d + l] /= s[l];
}

// ---- FP8 E4M3 quantize-dequantize -----------------------------------------
// q = x/scale in float; RNE onto the enumerated E4M3 grid (ties to the even code), |q| > 448
// clamps to +-448; result q_hat * scale in float. Non-finite input is an error.
int orc_fp8_qdq(const float* x, std::int64_t n, float scale, float* out) {
  if (!(scale > 0.0f)) return fail("fp8_qdq: scale must be > 0");
  static float grid[127];
  static bool init = false;
  if (!init) {
    for (int c = 0; c < 127; ++c) grid[c] = e4m3_value(c);
    init = true;
  }
  for (std::int64_t i = 0; i < n; ++i) {
    if (!std::isfinite(x[i])) return fail("fp8_qdq: non-finite input");
    const float q = x[i] / scale;
    const float a = std::fabs(q);
    float r;
    if (a >= 448.0f) {
      r = 448.0f;
    } else {
      // grid is increasing; find the bracketing pair.
      int hi = static_cast<int>(std::upper_bound(grid, grid + 127, a) - grid);  // first > a
      int lo = hi - 1;
      if (grid[lo] == a) {
        r = a;
      } else {
        const float dl = a - grid[lo], dh = grid[hi] - a;
        if (dl < dh) r = grid[lo];
        else if (dh < dl) r = grid[hi];
        else r = (lo & 1) ? grid[hi] : grid[lo];
      }
    }
    out[i] = std::copysign(r, q) * scale;
  }
  return 0;
}

// Index (0..126) of the E4M3 code nearest to |q| by the same rule, sign in bit 7 (for tests that
// compare device-produced E4M3 bytes).
int orc_fp8_encode(const float* q, std::int64_t n, std::uint8_t* codes) {
  std::vector<float> tmp(static_cast<std::size_t>(n));
  if (orc_fp8_qdq(q, n, 1.0f, tmp.data())) return 1;
  for (std::int64_t i = 0; i < n; ++i) {
    const float a = std::fabs(tmp[static_cast<std::size_t>(i)]);
    int c = 0;
    while (c < 126 && e4m3_value(c) != a) ++c;
    codes[i] = static_cast<std::uint8_t>(c | (std::signbit(tmp[static_cast<std::size_t>(i)]) ? 0x80 : 0));
  }
  return 0;
}

}  // extern "C"
