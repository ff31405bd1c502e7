// Expert parallelism — host side.
//
// Experts are sharded contiguously: rank r owns global experts [r*NL, (r+1)*NL), NL = N/R.
// Tokens are data-parallel (each rank routes its own batch). One forward is
//   route (all N experts) -> plan -> dispatch into this rank's global expert-major permutation
//   -> all-gather of the per-expert counts (an R x N matrix)
//   -> exchange: the piece (dest r, expert g) of the permutation goes to rank r, landing in r's
//      receive buffer at (local expert, source rank, token) order, so every local expert's rows
//      are contiguous and the grouped GEMMs run unchanged
//   -> local grouped GEMMs -> reverse exchange into the source's permutation slots -> weighted
//      combine at the source.
// NCCL is loaded at run time (dlopen) so the single-GPU library has no NCCL dependency; with
// torch already in the process this resolves to the same libnccl.so.2 torch uses.
#pragma once
#include <dlfcn.h>

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

namespace cmoe {

// Minimal NCCL ABI (nccl.h 2.27/2.28): the few entry points the exchange needs.
struct NcclApi {
  using Comm = void*;
  struct UniqueId {
    char internal[128];
  };
  enum DataType { kUint8 = 1, kInt32 = 2, kFloat32 = 7 };
  enum RedOp { kSum = 0 };
  int (*GetUniqueId)(UniqueId*) = nullptr;
  int (*CommInitRank)(Comm*, int, UniqueId, int) = nullptr;
  int (*CommDestroy)(Comm) = nullptr;
  int (*AllGather)(const void*, void*, size_t, int, Comm, cudaStream_t) = nullptr;
  int (*AllReduce)(const void*, void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Send)(const void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*Recv)(void*, size_t, int, int, Comm, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(int) = nullptr;

  static NcclApi& get() {
    static NcclApi api;
    static bool loaded = false;
    if (!loaded) {
      void* lib = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
      if (!lib) lib = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
      if (!lib) throw std::runtime_error(std::string("cannot load NCCL: ") + dlerror());
      auto sym = [&](const char* n) {
        void* p = dlsym(lib, n);
        if (!p) throw std::runtime_error(std::string("NCCL symbol missing: ") + n);
        return p;
      };
      api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
      api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
      api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
      api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
      api.AllReduce = reinterpret_cast<decltype(api.AllReduce)>(sym("ncclAllReduce"));
      api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
      api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
      api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
      api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
      api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
      loaded = true;
    }
    return api;
  }
};

// Receive-side layout for `rank` from the all-gathered counts C[s][g] (R x N, row = source).
//   local_offsets[e]   (NL+1)  first receive row of local expert e
//   recv_piece[e*R+s]  (NL*R)  first receive row of the piece (local expert e, source s)
// Pieces are ordered (local expert, source rank); inside a piece rows keep the source's token
// order, so every local expert's segment is contiguous.
inline int64_t ep_layout(const int64_t* C, int R, int N, int rank, int64_t* local_offsets, int64_t* recv_piece) {
  const int NL = N / R;
  int64_t row = 0;
  for (int e = 0; e < NL; ++e) {
    local_offsets[e] = row;
    const int g = rank * NL + e;
    for (int s = 0; s < R; ++s) {
      recv_piece[e * R + s] = row;
      row += C[(int64_t)s * N + g];
    }
  }
  local_offsets[NL] = row;
  return row;
}

}  // namespace cmoe
