// Compiled reference-side consumer of libcompass_moe.so: the INTEGRATION.md "Binding from the
// reference (C++)" snippet made runnable. Reads a layer and a batch from a raw fp32 file, runs
// the drop-in host call (cl_moe_forward_host, CL_MOE_IO_F32), writes the output, and checks the
// reference C API conventions (proj/src/capi.cpp:57-63, compass_lab.h:23-27, :50): ConfigError ->
// CL_ERR_CONFIG, every other failure -> CL_ERR_RUN with the message in last_error ("" after a
// success). Built with compass_lab.h first when the reference headers are on the include path.
//
// usage: consumer <in.bin> <out.bin>; in.bin = int64 {d, N, K, f, T} then fp32 w_router [d][N],
// w_in [N][d][2f], w_out [N][f][d], hidden [T][d]; out.bin = fp32 [T][d].
#ifdef COMPASS_HAVE_LAB
#include "compass_lab.h"  // cl_status (the reference's)
#endif
#include "compass_moe.h"

#include <cmath>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <limits>
#include <vector>

#define CHECK(cond, ...)                     \
  do {                                       \
    if (!(cond)) {                           \
      std::fprintf(stderr, "FAIL: " __VA_ARGS__); \
      std::fprintf(stderr, "\n");            \
      return 1;                              \
    }                                        \
  } while (0)

int main(int argc, char** argv) {
  if (argc != 3) return 2;
  std::ifstream in(argv[1], std::ios::binary);
  int64_t dims[5];
  in.read(reinterpret_cast<char*>(dims), sizeof dims);
  const int64_t d = dims[0], N = dims[1], K = dims[2], f = dims[3], B = dims[4];
  std::vector<float> w_router(d * N), win_all(N * d * 2 * f), wout_all(N * f * d), hidden(B * d);
  for (auto* v : {&w_router, &win_all, &wout_all, &hidden})
    in.read(reinterpret_cast<char*>(v->data()), static_cast<std::streamsize>(v->size() * sizeof(float)));
  CHECK(in.good(), "short input file");

  // ConfigError -> CL_ERR_CONFIG (a d_model that is not a multiple of 256), message via last_error(NULL)
  cl_moe_config bad{d + 1, N, K, f, B, 0, 0, 1, 0};
  cl_moe* hb = nullptr;
  CHECK(cl_moe_create(&bad, w_router.data(), win_all.data(), wout_all.data(), &hb) == CL_ERR_CONFIG,
        "bad config must give CL_ERR_CONFIG");
  CHECK(hb == nullptr && std::strlen(cl_moe_last_error(nullptr)) > 0, "create error message");

  // the snippet
  cl_moe_config cfg{d, N, K, f, /*max_tokens=*/B, /*device=*/0, /*gemm_ctas=*/0, 1, 0};
  cl_moe* h = nullptr;
  CHECK(cl_moe_create(&cfg, w_router.data(), win_all.data(), wout_all.data(), &h) == CL_OK, "create: %s",
        cl_moe_last_error(nullptr));
  std::vector<float> out(B * d);
  CHECK(cl_moe_forward_host(h, hidden.data(), B, out.data(), CL_MOE_IO_F32) == CL_OK, "forward: %s",
        cl_moe_last_error(h));
  CHECK(std::strcmp(cl_moe_last_error(h), "") == 0, "last_error must be \"\" after a success");

  // more than max_tokens -> CL_ERR_CONFIG; bad io dtype -> CL_ERR_CONFIG
  std::vector<float> big((B + 1) * d, 0.0f), big_out((B + 1) * d);
  CHECK(cl_moe_forward_host(h, big.data(), B + 1, big_out.data(), CL_MOE_IO_F32) == CL_ERR_CONFIG, "T > max_tokens");
  CHECK(std::strlen(cl_moe_last_error(h)) > 0, "message for T > max_tokens");
  CHECK(cl_moe_forward_host(h, hidden.data(), B, out.data(), 7) == CL_ERR_CONFIG, "io dtype");
  // non-finite input -> ValidationError -> CL_ERR_RUN (check_finite, tensor.cpp:35-41)
  std::vector<float> nan_in(hidden);
  nan_in[3] = std::numeric_limits<float>::quiet_NaN();
  std::vector<float> nan_out(B * d);
  CHECK(cl_moe_forward_host(h, nan_in.data(), B, nan_out.data(), CL_MOE_IO_F32) == CL_ERR_RUN, "NaN input");
  CHECK(std::strstr(cl_moe_last_error(h), "non-finite") != nullptr, "NaN message: %s", cl_moe_last_error(h));
  // the handle stays usable: same result again
  std::vector<float> out2(B * d);
  CHECK(cl_moe_forward_host(h, hidden.data(), B, out2.data(), CL_MOE_IO_F32) == CL_OK, "forward after error");
  CHECK(std::memcmp(out.data(), out2.data(), out.size() * sizeof(float)) == 0, "deterministic output");
  cl_moe_destroy(h);

  std::ofstream o(argv[2], std::ios::binary);
  o.write(reinterpret_cast<const char*>(out.data()), static_cast<std::streamsize>(out.size() * sizeof(float)));
  std::printf("ok %s\n", cl_moe_version());
  return 0;
}
