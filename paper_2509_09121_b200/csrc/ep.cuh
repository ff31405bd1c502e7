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
  enum RedOp { kSum = 0, kMax = 2 };
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
  int (*CommGetAsyncError)(Comm, int*) = nullptr;
  int (*CommAbort)(Comm) = nullptr;

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
      api.CommGetAsyncError = reinterpret_cast<decltype(api.CommGetAsyncError)>(sym("ncclCommGetAsyncError"));
      api.CommAbort = reinterpret_cast<decltype(api.CommAbort)>(sym("ncclCommAbort"));
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

// ---- peer-memory (NVLink) transport ----
// With every rank's receive buffer x_recv and return buffer y mapped into every peer (CUDA IPC),
// the two exchanges need no copy engine and no NCCL data movement:
//   dispatch: the source's dispatch kernel stores each (token, k) row straight into the owner's
//             x_recv at the row ep_piece_row(owner, e, source) + rank-within-expert, and its
//             combine weight into the owner's w_recv (GEMM2 scales rows exactly as on one GPU,
//             so the layer output is bit-identical for every EP degree);
//   return:   the owner's GEMM2 epilogue stores each output row straight into the source's y at
//             ep_src_row(source, g) + row-within-piece, so the return exchange overlaps GEMM2
//             tile by tile.
// All ranks evaluate these from the same all-gathered C, so the layout is consistent by
// construction. The helpers below are shared by the host restatement (cl_moe_ep_peer_layout,
// tested on the CPU) and the device layout kernel.
template <typename CT>
__host__ __device__ inline int64_t ep_piece_row(const CT* C, int R, int N, int owner, int e, int s) {
  const int NL = N / R;
  int64_t row = 0;
  for (int e2 = 0; e2 < e; ++e2)
    for (int s2 = 0; s2 < R; ++s2) row += C[(int64_t)s2 * N + owner * NL + e2];
  for (int s2 = 0; s2 < s; ++s2) row += C[(int64_t)s2 * N + owner * NL + e];
  return row;
}

// First row of global expert g's piece in source s's expert-major permutation.
template <typename CT>
__host__ __device__ inline int64_t ep_src_row(const CT* C, int N, int s, int g) {
  int64_t row = 0;
  for (int g2 = 0; g2 < g; ++g2) row += C[(int64_t)s * N + g2];
  return row;
}

#ifdef __CUDACC__
// Device layout for `rank` from the all-gathered counts C (R x N int32); x rows are x_row_bytes
// long (bf16 or e4m3), returned rows row_bytes (bf16):
//   expert_dst[g]   address of this rank's first row for expert g in the owner's x_recv
//   expert_dst_w[g] the same row in the owner's w_recv (combine weight of each received row)
//   ep_off[e]       (NL+1) local expert offsets in this rank's x_recv (GEMM row groups)
//   row_ptr[r]      for every received row r: its return address in the source rank's y
// and, for training (peer_dy / peer_dx mapped): expert_dst_dy[g] (this rank's dY piece in the
// owner's dYbuf) and row_ptr_dx[r] (the received row's dX slot in the source's dXsrc)
// Blocks 0..NL*R-1 fill row_ptr for one (local expert, source) piece each; the last block checks
// every owner's receive total against recv_cap (the same verdict on all ranks) and on overflow
// sets bit 2 of `flag`, nulls expert_dst and zeroes ep_off, so nothing is written anywhere.
__global__ void __launch_bounds__(256) ep_peer_layout_kernel(const int32_t* __restrict__ C, int R, int N, int rank,
                                                             int64_t recv_cap, int64_t x_row_bytes, int64_t row_bytes,
                                                             char* const* __restrict__ peer_x,
                                                             char* const* __restrict__ peer_y,
                                                             float* const* __restrict__ peer_w, void** expert_dst,
                                                             float** expert_dst_w, int32_t* ep_off, void** row_ptr,
                                                             int32_t* flag, char* const* __restrict__ peer_dy,
                                                             char* const* __restrict__ peer_dx, void** expert_dst_dy,
                                                             void** row_ptr_dx, char* const* __restrict__ peer_a = nullptr,
                                                             uint32_t** expert_arrive = nullptr,
                                                             uint32_t* arrive_tgt = nullptr, int K = 1) {
  const int NL = N / R;
  if (blockIdx.x < (unsigned)(NL * R)) {
    const int e = blockIdx.x / R, s = blockIdx.x % R, g = rank * NL + e;
    const int64_t start = ep_piece_row(C, R, N, rank, e, s);
    const int64_t n = C[(int64_t)s * N + g];
    const int64_t src_row = ep_src_row(C, N, s, g);
    char* dst = peer_y[s] + src_row * row_bytes;
    char* dxb = peer_dx ? peer_dx[s] : nullptr;
    for (int64_t j = threadIdx.x; j < n && start + j < recv_cap; j += blockDim.x) {
      row_ptr[start + j] = dst + j * row_bytes;
      if (dxb) row_ptr_dx[start + j] = dxb + (src_row + j) * row_bytes;
    }
    return;
  }
  __shared__ int ok;
  if (threadIdx.x == 0) {
    int good = 1;
    for (int o = 0; o < R; ++o)
      if (ep_piece_row(C, R, N, o, NL, 0) > recv_cap) good = 0;
    ok = good;
    if (!good) atomicOr(flag, 2);
  }
  __syncthreads();
  for (int g = threadIdx.x; g < N; g += blockDim.x) {
    const int o = g / NL, e = g % NL;
    const int64_t row = ep_piece_row(C, R, N, o, e, rank);
    expert_dst[g] = ok ? peer_x[o] + row * x_row_bytes : nullptr;
    expert_dst_w[g] = ok ? peer_w[o] + row : nullptr;
    char* dyb = peer_dy ? peer_dy[o] : nullptr;
    expert_dst_dy[g] = (ok && dyb) ? dyb + row * row_bytes : nullptr;
  }
  for (int e = threadIdx.x; e <= NL; e += blockDim.x)
    ep_off[e] = ok ? static_cast<int32_t>(ep_piece_row(C, R, N, rank, e, 0)) : 0;
  if (peer_a) {  // dispatch overlap: where this rank's pieces are counted, and what this rank awaits
    for (int g = threadIdx.x; g < N; g += blockDim.x)
      expert_arrive[g] = ok ? reinterpret_cast<uint32_t*>(peer_a[g / NL]) + g % NL : nullptr;
    for (int e = threadIdx.x; e < NL && ok; e += blockDim.x) {
      uint32_t add = 0;
      for (int s = 0; s < R; ++s) {  // source s writes each row in token_grid(T_s).y column slices
        int64_t ts = 0;
        for (int g = 0; g < N; ++g) ts += C[(int64_t)s * N + g];
        ts /= K;
        const int64_t blocks = (ts + 7) / 8;
        const int64_t slices = blocks ? (int64_t)max(1LL, min(8LL, (4LL * kTargetSms + blocks - 1) / blocks)) : 1;
        add += (uint32_t)(C[(int64_t)s * N + rank * NL + e] * slices);
      }
      arrive_tgt[e] += add;
    }
  }
}
#endif

}  // namespace cmoe
