// Grouped (per-expert) GEMM on the 5th-generation tensor cores for the MoE expert FFN, forward
// and backward.
//
// Row-grouped modes (M = the rows of one expert segment, K fixed):
//   EPI_SWIGLU       A_act[r,:] = silu(X[r,:] W_gate[e]) * (X[r,:] W_up[e])   (bf16 or e4m3 out;
//                    training mode also stores the pre-activations H = [G | U], bf16)
//   EPI_ROWSCALE     Y[r,:] = w[r] * (A_act[r,:] W_out[e])                      (bf16; w optional)
//   EPI_SWIGLU_BWD   dA = dY[r,:] W_out[e]^T, fused with the SwiGLU backward:
//                    dH[r, c] = dA*U*silu'(G), dH[r, f+c] = dA*silu(G)           (bf16)
// K-grouped mode (kWgrad; M, N = weight dims, K = the rows of expert e, variable):
//   EPI_WGRAD        dW[e] = Lhs_e^T Rhs_e accumulated over the expert's rows    (fp32)
//                    Both operands are read MN-major straight from row-major [rows][C] buffers
//                    whose expert segments are padded to 64 zero rows (no transposes).
//
// Replaces the per-expert ops::matmul + slice_cols + silu + mul (+ mul_rowwise) chain of the
// reference composition and its Tape backward closures (proj/src/tensor.cpp:350-375 incl. the
// gemm_nt / gemm_tn closures :364-372, :398-420, :315-322, :283-303, :572-610).
//
// Design (sm_100a):
//  * persistent kernel, one CTA (or CTA pair) per SM, static round-robin over output tiles in
//    (expert, n-block, m-block) order so CTAs running together share the B n-block in L2;
//  * warp-specialised: warp 0 = TMA producer, warp 1 = tcgen05.mma issuer (one elected thread),
//    warp 2 = TMEM allocator, warps 4-7 = epilogue (TMEM -> registers -> global);
//  * operands staged by TMA into 128-byte-swizzled K-major tiles, kStages-deep mbarrier ring;
//  * FP32 accumulators in TMEM, double-buffered (2 x 256 columns) so the epilogue of tile i
//    overlaps the main loop of tile i+1;
//  * kCtaGroup == 2: cta_group::2 MMA with M=256 over a CTA pair (each CTA stages 128 rows of A
//    and half of the 256-wide B tile), halving per-SM operand traffic.
#pragma once
#include <cuda_fp8.h>

#include "ptx.cuh"

namespace cmoe {

enum GemmEpi : int { EPI_SWIGLU = 0, EPI_ROWSCALE = 1, EPI_SWIGLU_BWD = 2, EPI_WGRAD = 3 };

struct GemmArgs {
  const int32_t* offsets;   // row-grouped: [n_experts+1] first permuted row of each expert
  int32_t n_experts;        // experts on this rank
  int32_t n_tiles_n;        // 256-wide n-blocks per expert
  int32_t num_kb;           // row-grouped: 128-byte k-blocks
  int32_t b_rows_per_expert;
  void* out;                // output (bf16 / e4m3 / fp32)
  int32_t ldo;              // output row stride (elements)
  const float* row_scale;   // EPI_ROWSCALE: per permuted row combine weight (nullable)
  const float* act_scale;   // FP8: per-expert activation scale of the A operand [n_experts]
  const float* w_scale;     // FP8: per-(expert, B row) weight scale [n_experts][b_rows_per_expert]
  const float* out_scale;   // FP8 EPI_SWIGLU: per-expert scale of the e4m3 output [n_experts]
  void* aux;                // EPI_SWIGLU: H out (nullable, [rows][2f]); EPI_SWIGLU_BWD: H in
  int32_t ffn;              // f (column offset of the up half in H / dH)
  const int32_t* kb_off;    // kWgrad: [n_experts+1] first k-block of each expert's (padded) rows
  int32_t m_tiles;          // kWgrad: m-tiles per expert
  int64_t out_estride;      // kWgrad: elements between consecutive experts' outputs
  int* tile_counter;        // dynamic tile scheduler: global counter, zeroed before the launch
  void* aux_t;              // training: copy of the output in the padded row layout, bf16 [rp][C]
                            // (expert e's rows from poff[e]; operand of the weight gradients)
  int64_t rp;               // padded-row capacity of aux_t
  const int32_t* poff;      // [n_experts+1] 64-aligned first padded row of each expert
  void* const* row_ptr;     // EPI_ROWSCALE peer transport: destination address of each row (nullable)
  int32_t m_group;          // row-grouped tile order: m-tiles per group (0 = all), see decode_tile;
                            // kWgrad: the smallest group (the budget may allow more)
  int64_t group_bytes;      // kWgrad tile order: L2 budget of a resident A group (0 = m fastest)
  int32_t half_tail;        // 2-CTA, forward epilogues: an expert's last m-tile with <= 128 rows runs
                            // as an M=128 pair MMA (64 rows per CTA, half the tensor time)
  const uint32_t* arrive;       // EP dispatch overlap (row-grouped, nullable): per local expert, pieces of
  const uint32_t* arrive_tgt;   // rows stored by the sources; the producer waits arrive >= target
  int32_t* err_flag;            // bit 2: rows did not arrive within the device-side timeout
  int32_t prefetch_kb;      // row-grouped: k-blocks of the NEXT tile prefetched into L2 (0 = off) ...
  int32_t prefetch_lead;    // ... issued this many k-blocks before the end of the current tile, where
                            // the producer also claims the next tile index
  uint64_t a_hint, b_hint;  // TMA L2 cache hints of the A / B loads (0 = the kernel's default)
  const int32_t* a_poff;    // row-grouped, nullable: A rows come from the padded row layout (expert e
                            // from a_poff[e]); output rows, masks and row scales stay in the row layout
};

constexpr int kGemmThreads = 384;  // warps 0-3: TMA / MMA / TMEM alloc / idle; warps 4-11: epilogue
constexpr int kEpiWarps = 8;      // two warps per TMEM lane quarter, each owning half of the columns
constexpr int kBN = 256;                 // MMA N (output columns of one tile, pre-SwiGLU)
constexpr int kBKBytes = 128;            // one swizzle atom along K
constexpr int kMaxExperts = 128;  // experts per rank (cl_moe validates N <= 128)
constexpr int kTileSlots = 4;            // depth of the tile-index broadcast ring

template <int kCtaGroup>
struct GemmCfg {
  static constexpr int kRowsPerCta = 128;
  static constexpr int kBM = 128 * kCtaGroup;
  static constexpr int kBRowsPerCta = kBN / kCtaGroup;
  static constexpr int kStageA = kRowsPerCta * kBKBytes;
  static constexpr int kStageB = kBRowsPerCta * kBKBytes;
  static constexpr int kStageBytes = kStageA + kStageB;
  static constexpr int kStages = kCtaGroup == 1 ? 4 : 6;
  // half tiles (2-CTA): gate/up exchange between TMEM lane halves, [64 rows][129 fp32] (padded)
  static constexpr int kXStride = 129;
  static constexpr int kXBytes = kCtaGroup == 2 ? 64 * kXStride * 4 : 0;
  // per-expert tables cached in smem (tile prefix + row / k-block offsets): a tile decode must not
  // wait on global memory, or the MMA issuer idles the tensor pipe between tiles
  static constexpr int kSmemCtl = 1024 /*align*/ + 256 /*barriers*/ + 2 * (kMaxExperts + 1) * 4;
  static constexpr int kSmem = kStages * kStageBytes + kSmemCtl + kXBytes;
  static_assert(kSmem <= 232448, "shared memory budget");
};

struct TileInfo {
  int e, mt, nt;
  int a_row;     // first A row of the tile (this CTA's half added by the caller)
  int b_row;     // first B row of the tile
  int row_end;   // row-grouped: end of the expert segment (epilogue mask)
  int kb0, nkb;  // k-block range
  bool half;     // 2-CTA tail tile run as M=128 (64 rows per CTA)
};

// Row-grouped decode: tiles of expert e = mtiles(e) x n_tiles_n. The expert's m-tiles are taken
// in groups of m_group; inside a group m is fastest and the group sweeps every n-block before the
// next group starts. The group's A rows stay resident in L2 while the weight n-blocks stream past
// (an expert whose rows exceed L2 would otherwise re-stream its rows for every n-block).
__device__ __forceinline__ bool decode_tile(int tile, const int* mt_prefix, const int* s_off, const GemmArgs& a, int bm,
                                            TileInfo& ti) {
  if (tile >= mt_prefix[a.n_experts] * a.n_tiles_n) return false;
  int e = 0;
  while (tile >= mt_prefix[e + 1] * a.n_tiles_n) ++e;
  const int local = tile - mt_prefix[e] * a.n_tiles_n;
  const int mtiles = mt_prefix[e + 1] - mt_prefix[e];
  const int gm = (a.m_group > 0 && a.m_group < mtiles) ? a.m_group : mtiles;
  const int g = local / (gm * a.n_tiles_n);
  const int within = local - g * gm * a.n_tiles_n;
  const int gsz = min(gm, mtiles - g * gm);
  ti.e = e;
  ti.nt = within / gsz;
  ti.mt = g * gm + (within - ti.nt * gsz);
  ti.a_row = s_off[e] + ti.mt * bm;
  ti.b_row = e * a.b_rows_per_expert + ti.nt * kBN;
  ti.row_end = s_off[e + 1];
  ti.kb0 = 0;
  ti.nkb = a.num_kb;
  ti.half = a.half_tail && ti.row_end - ti.a_row <= bm / 2;
  return true;
}

// Row-grouped decode with clusters of two CTA pairs (kCM == 2): a tile is an m-tile PAIR x one
// n-block; pair p of the cluster takes m-tile 2 mp + p (inactive when the expert has no such
// m-tile: it still streams its share of the shared B tile). mp_prefix = expert prefix of m-pairs;
// m_group counts m-pairs.
__device__ __forceinline__ bool decode_tile_mc(int tile, const int* mp_prefix, const int* s_off, const GemmArgs& a,
                                               int bm, int pair, TileInfo& ti, bool& active) {
  if (tile >= mp_prefix[a.n_experts] * a.n_tiles_n) return false;
  int e = 0;
  while (tile >= mp_prefix[e + 1] * a.n_tiles_n) ++e;
  const int local = tile - mp_prefix[e] * a.n_tiles_n;
  const int mpairs = mp_prefix[e + 1] - mp_prefix[e];
  const int gm = (a.m_group > 0 && a.m_group < mpairs) ? a.m_group : mpairs;
  const int g = local / (gm * a.n_tiles_n);
  const int within = local - g * gm * a.n_tiles_n;
  const int gsz = min(gm, mpairs - g * gm);
  ti.e = e;
  ti.nt = within / gsz;
  const int mp = g * gm + (within - ti.nt * gsz);
  ti.mt = 2 * mp + pair;
  const int mtiles = (s_off[e + 1] - s_off[e] + bm - 1) / bm;
  active = ti.mt < mtiles;
  ti.a_row = s_off[e] + ti.mt * bm;
  ti.b_row = e * a.b_rows_per_expert + ti.nt * kBN;
  ti.row_end = s_off[e + 1];
  ti.kb0 = 0;
  ti.nkb = a.num_kb;
  ti.half = active && a.half_tail && ti.row_end - ti.a_row <= bm / 2;
  return true;
}

// K-grouped decode (weight gradients): every expert has m_tiles x n_tiles_n tiles; the K range
// is the expert's padded row range, so its operand slabs grow with its row count. m-tiles go in
// groups whose A slabs fit `group_bytes` of L2 but of at least m_group m-tiles (m fastest inside,
// sweeping every n-block), as in decode_tile: a hot expert's A slab is then read once per group
// instead of once per n-block, and its B slabs once per group instead of once per m-tile.
__device__ __forceinline__ bool decode_tile_wgrad(int tile, const int* s_kb, const GemmArgs& a, int bm, TileInfo& ti) {
  const int per = a.m_tiles * a.n_tiles_n;
  if (tile >= a.n_experts * per) return false;
  const int e = tile / per;
  const int local = tile - e * per;
  const int nkb = s_kb[e + 1] - s_kb[e];
  int gm = a.m_tiles;
  if (a.group_bytes > 0 && nkb > 0) {
    const int64_t g = a.group_bytes / ((int64_t)bm * nkb * kBKBytes);
    gm = (int)min((int64_t)a.m_tiles, max((int64_t)max(1, a.m_group), g));
  }
  const int g = local / (gm * a.n_tiles_n);
  const int within = local - g * gm * a.n_tiles_n;
  const int gsz = min(gm, a.m_tiles - g * gm);
  ti.e = e;
  ti.nt = within / gsz;
  ti.mt = g * gm + (within - ti.nt * gsz);
  ti.a_row = ti.mt * bm;
  ti.b_row = ti.nt * kBN;
  ti.row_end = 1 << 30;
  ti.kb0 = s_kb[e];
  ti.nkb = nkb;
  ti.half = false;
  return true;
}

// 32 consecutive per-column scales as 8 vector loads (FP8 epilogues; read-only, L1-cached)
__device__ __forceinline__ void load_f32x32(const float* __restrict__ p, float* v) {
#pragma unroll
  for (int i = 0; i < 8; ++i) {
    const float4 t = __ldg(reinterpret_cast<const float4*>(p) + i);
    v[4 * i] = t.x;
    v[4 * i + 1] = t.y;
    v[4 * i + 2] = t.z;
    v[4 * i + 3] = t.w;
  }
}

// SiLU with the MUFU exp2 / reciprocal pair (2 ulp in fp32; the result is rounded to bf16 / e4m3)
__device__ __forceinline__ float silu_f(float g) { return __fdividef(g, 1.0f + __expf(-g)); }

__device__ __forceinline__ void store_bf16x32(__nv_bfloat16* dst, const float* v) {
  const uint64_t pol = l2_policy_evict_first();
#pragma unroll
  for (int i = 0; i < 2; ++i) {
    uint32_t p[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) p[j] = pack_bf16(v[16 * i + 2 * j], v[16 * i + 2 * j + 1]);
    st_global_v8_hint(dst + 16 * i, p, pol);
  }
}
__device__ __forceinline__ void store_bf16x32_plain(__nv_bfloat16* dst, const float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i)
    st_global_v4(dst + 8 * i, pack_bf16(v[8 * i], v[8 * i + 1]), pack_bf16(v[8 * i + 2], v[8 * i + 3]),
                 pack_bf16(v[8 * i + 4], v[8 * i + 5]), pack_bf16(v[8 * i + 6], v[8 * i + 7]));
}
__device__ __forceinline__ void load_bf16x32(const __nv_bfloat16* src, float* v) {
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int4 r = *reinterpret_cast<const int4*>(src + 8 * i);
    const __nv_bfloat16* h = reinterpret_cast<const __nv_bfloat16*>(&r);
#pragma unroll
    for (int j = 0; j < 8; ++j) v[8 * i + j] = __bfloat162float(h[j]);
  }
}

// Transposed store of 32 consecutive columns of one row: lanes of a warp hold consecutive rows, so
// each 2-byte store instruction writes one contiguous 64-byte run of the transposed matrix.
__device__ __forceinline__ void store_t_bf16x32(__nv_bfloat16* dst, int64_t stride, const float* v) {
#pragma unroll
  for (int i = 0; i < 32; ++i) dst[(size_t)i * stride] = __float2bfloat16_rn(v[i]);
}

// kCM (CTA pairs per cluster, 1 or 2; 2 needs kCtaGroup == 2 and a row-grouped mode): with 2, the
// two pairs of a cluster compute adjacent m-tiles of the same n-block and share its B tile through
// TMA multicast — each CTA loads one 64-row quarter box and multicasts it to the same-half CTA of
// the other pair — halving the B operand's L2 -> SM traffic; a stage slot is refilled only when
// both pairs' MMAs have released it (tcgen05.commit multicast to all four CTAs, empty count 2).
template <int kCtaGroup, int kEpi, bool kFp8, bool kOutFp8, bool kWgrad = false, int kCM = 1>
__global__ void __launch_bounds__(kGemmThreads, 1)
    grouped_gemm_kernel(const __grid_constant__ CUtensorMap tmA, const __grid_constant__ CUtensorMap tmB,
                        const GemmArgs args) {
  static_assert(kCM == 1 || (kCM == 2 && kCtaGroup == 2 && !kWgrad), "multicast clusters: pair mode, row-grouped");
  using Cfg = GemmCfg<kCtaGroup>;
  constexpr int kCS = kCtaGroup * kCM;  // cluster size
  constexpr int S = Cfg::kStages;
  constexpr int kUmmaKBytes = 32;                    // 16 bf16 or 32 e4m3 per MMA
  constexpr int kMmaPerKb = kBKBytes / kUmmaKBytes;  // 4
  constexpr uint32_t kIdesc = idesc_f32acc<kFp8>(Cfg::kBM, kBN) | (kWgrad ? kIdescMnMajorAB : 0u);
  constexpr uint32_t kIdescHalf = idesc_f32acc<kFp8>(128, kBN);  // 2-CTA tail tiles
  constexpr int kElemBytes = kFp8 ? 1 : 2;
  constexpr int kBKElems = kBKBytes / kElemBytes;
  // Row-grouped: the A rows of an expert are re-read for every n-block -> keep them in L2.
  const uint64_t kAHint = args.a_hint ? args.a_hint : (kWgrad ? kEvictNormal : kEvictLast);
  const uint64_t kBHint = args.b_hint ? args.b_hint : kEvictNormal;

  extern __shared__ uint8_t smem_raw[];
  // 1024-byte aligned by an offset from the shared array itself, so the compiler keeps the pointer
  // in the shared window (LDS/STS, 32-bit addresses) instead of generic loads
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
  uint8_t* sA = smem;
  uint8_t* sB = smem + S * Cfg::kStageA;
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + S * Cfg::kStageBytes);
  uint64_t* empty = full + S;
  uint64_t* tfull = empty + S;
  uint64_t* tempty = tfull + 2;
  uint64_t* tfill = tempty + 2;          // tile-index ring: filled by the leader's producer
  uint64_t* tfree = tfill + kTileSlots;  //   freed by every consumer role (leader CTA only)
  int* tile_ring = reinterpret_cast<int*>(tfree + kTileSlots);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tile_ring + kTileSlots);
  int* mt_prefix = reinterpret_cast<int*>(smem + S * Cfg::kStageBytes + 256);
  int* s_off = mt_prefix + (kMaxExperts + 1);  // expert row offsets (row-grouped) or k-block offsets (kWgrad)
  float* xbuf = reinterpret_cast<float*>(smem + S * Cfg::kStageBytes + Cfg::kSmemCtl - 1024);

  const uint32_t warp = warp_id();
  const uint32_t lane = lane_id();
  const uint32_t crank = kCS == 1 ? 0 : cluster_ctarank();  // rank in the cluster
  const uint32_t cta_rank = crank & (kCtaGroup - 1);          // rank in the CTA pair
  const uint32_t pair = crank / kCtaGroup;                      // pair in the cluster (kCM == 2)
  const uint32_t pleader = crank & ~(uint32_t)(kCtaGroup - 1);  // the pair leader's cluster rank
  const bool sched = crank == 0;                                // the cluster's tile scheduler
  const uint16_t pair_mask = (uint16_t)(((1u << kCtaGroup) - 1) << pleader);
  const uint16_t all_mask = (uint16_t)((1u << kCS) - 1);

  for (int i = threadIdx.x; i <= args.n_experts; i += blockDim.x) s_off[i] = kWgrad ? args.kb_off[i] : args.offsets[i];
  if (!kWgrad && threadIdx.x == 0) {  // (kCM == 2: prefix of m-tile pairs)
    int acc = 0;
    mt_prefix[0] = 0;
    for (int e = 0; e < args.n_experts; ++e) {
      const int cnt = args.offsets[e + 1] - args.offsets[e];
      acc += ((cnt + Cfg::kBM - 1) / Cfg::kBM + kCM - 1) / kCM;
      mt_prefix[e + 1] = acc;
    }
  }
  if (warp == 0 && lane == 0) {
    tma_prefetch_desc(&tmA);
    tma_prefetch_desc(&tmB);
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < S; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], kCM);  // released by every pair's MMA (kCM == 2: the slot is shared)
    }
    for (int a = 0; a < 2; ++a) {
      mbar_init(&tfull[a], 1);
      mbar_init(&tempty[a], kEpiWarps * kCtaGroup);
    }
    // consumers of a tile index: every pair leader's MMA issuer, every other CTA's producer and
    // every CTA's epilogue warps
    for (int i = 0; i < kTileSlots; ++i) {
      mbar_init(&tfill[i], 1);
      mbar_init(&tfree[i], kCM + (kCS - 1) + kCS * kEpiWarps);
    }
    fence_mbar_init();
  }
  if (warp == 2) tmem_alloc<kCtaGroup>(tmem_slot, 512);
  tc_fence_before();
  if constexpr (kCS > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  // `active`: this pair has a tile (kCM == 2: the cluster's second m-tile may not exist)
  auto decode = [&](int tile, TileInfo& ti, bool& active) -> bool {
    active = true;
    if constexpr (kWgrad) return decode_tile_wgrad(tile, s_off, args, Cfg::kBM, ti);
    else if constexpr (kCM == 2) return decode_tile_mc(tile, mt_prefix, s_off, args, Cfg::kBM, pair, ti, active);
    else return decode_tile(tile, mt_prefix, s_off, args, Cfg::kBM, ti);
  };
  const int total_tiles = kWgrad ? args.n_experts * args.m_tiles * args.n_tiles_n : mt_prefix[args.n_experts] * args.n_tiles_n;
  // Dynamic in-order tile scheduler: the leader's producer takes tiles from a global counter and
  // broadcasts each index through a small smem ring (written into the peer CTA too), so the
  // clusters running at any moment always work on consecutive tiles -- they share the weight
  // n-block and the expert's rows in L2 (a static round-robin drifts apart over ~200 tiles and
  // thrashes L2). The index total_tiles is the stop sentinel.
  auto take_tile = [&](int i, bool peer_data) -> int {
    const int slot = i % kTileSlots;
    const uint32_t ph = (i / kTileSlots) & 1;
    if (peer_data) mbar_wait_cluster(&tfill[slot], ph);
    else mbar_wait(&tfill[slot], ph);
    return *reinterpret_cast<volatile int*>(&tile_ring[slot]);
  };
  // `tile` is the value just read from the slot: the arrive is control-dependent on that read, so
  // a relaxed arrive cannot overtake it (the producer rewrites the slot once every consumer freed it).
  auto free_tile = [&](int i, int tile) {
    const int slot = i % kTileSlots;
    if (tile < 0) return;
    if (sched) mbar_arrive_relaxed(&tfree[slot]);
    else mbar_arrive_cluster_relaxed(&tfree[slot], 0);
  };

  if (warp == 0) {
    // ===================== TMA producer (leader: also the tile scheduler) =====================
    if (elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      TileInfo ti, tn;
      // tile index i: the leader takes it from the global counter and publishes it to every
      // consumer (and the peer CTA); the peer's producer reads it from the ring
      auto claim = [&](int i) -> int {
        int tile;
        if (sched) {
          const int slot = i % kTileSlots;
          mbar_wait(&tfree[slot], ((i / kTileSlots) & 1) ^ 1);
          tile = min(atomicAdd(args.tile_counter, 1), total_tiles);
          tile_ring[slot] = tile;
#pragma unroll
          for (int r = 1; r < kCS; ++r) st_shared_cluster_u32(mapa(smem_u32(&tile_ring[slot]), r), (uint32_t)tile);
          mbar_arrive(&tfill[slot]);
#pragma unroll
          for (int r = 1; r < kCS; ++r) mbar_arrive_cluster(&tfill[slot], r);
        } else {
          tile = take_tile(i, true);
          free_tile(i, tile);
        }
        return tile;
      };
      // Next-tile prefetch (row-grouped): at prefetch_lead k-blocks before the end of a tile the
      // producer claims the next tile and asks L2 for its first prefetch_kb k-blocks (this CTA's
      // A rows and B rows), so the first stages of the next tile do not wait a DRAM round trip at
      // the tile boundary (where the ring's few stages of slack run out).
      const bool pf = !kWgrad && kCM == 1 && args.prefetch_kb > 0;
      int ready_e = -1;  // EP overlap: the last expert whose rows were all seen arriving
      int tile = claim(0);
      for (int i = 0;; ++i) {
        bool active, nactive;
        if (tile >= total_tiles || !decode(tile, ti, active)) break;
        if (!kWgrad && args.arrive && active && ti.e != ready_e) {
          // the sources' dispatch kernels publish their pieces with system-scope releases; once
          // all arrived, order the TMA (async-proxy) reads after them
          const uint64_t t0 = globaltimer_ns();
          while ((int32_t)(ld_acquire_sys(args.arrive + ti.e) - args.arrive_tgt[ti.e]) < 0) {
            __nanosleep(256);
            if (globaltimer_ns() - t0 > 20000000000ull) {  // 20 s: a peer died; fail loudly, do not hang
              atomicOr(args.err_flag, 4);
              break;
            }
          }
          fence_proxy_async_global();
          ready_e = ti.e;
        }
        const bool half_t = kCtaGroup == 2 && ti.half;
        const int a_src = (!kWgrad && args.a_poff) ? __ldg(args.a_poff + ti.e) + (ti.a_row - s_off[ti.e]) : ti.a_row;
        const int a_row = a_src + cta_rank * (half_t ? 64 : Cfg::kRowsPerCta);
        const int b_row = ti.b_row + cta_rank * Cfg::kBRowsPerCta;
        int next = -1;
        const int claim_kb = pf ? ti.kb0 + max(0, ti.nkb - args.prefetch_lead) : 1 << 30;
        for (int kb = ti.kb0; kb < ti.kb0 + ti.nkb; ++kb) {
          if (kb == claim_kb) {
            next = claim(i + 1);
            if (next < total_tiles && decode(next, tn, nactive)) {
              const int na_src = args.a_poff ? __ldg(args.a_poff + tn.e) + (tn.a_row - s_off[tn.e]) : tn.a_row;
              const int na = na_src + cta_rank * Cfg::kRowsPerCta, nb = tn.b_row + cta_rank * Cfg::kBRowsPerCta;
              for (int k = tn.kb0; k < tn.kb0 + min(tn.nkb, args.prefetch_kb); ++k) {
                tma_prefetch_2d(&tmA, k * kBKElems, na);
                tma_prefetch_2d(&tmB, k * kBKElems, nb);
              }
            }
          }
          mbar_wait(&empty[s], ph ^ 1);
          if constexpr (kWgrad) {
            // MN-major operands: boxes {64 columns, 64 rows} of the padded row-major buffers;
            // a_row / b_row are column offsets here, the k-block is a block of 64 rows
            if (kCtaGroup == 1 || cta_rank == 0) mbar_arrive_expect_tx(&full[s], kCtaGroup * Cfg::kStageBytes);
#pragma unroll
            for (int c = 0; c < Cfg::kRowsPerCta / 64; ++c) {
              if constexpr (kCtaGroup == 1)
                tma_load_2d(&tmA, &full[s], sA + s * Cfg::kStageA + c * 8192, a_row + c * 64, kb * 64, kAHint);
              else
                tma_load_2d_pair(&tmA, &full[s], sA + s * Cfg::kStageA + c * 8192, a_row + c * 64, kb * 64, kAHint);
            }
#pragma unroll
            for (int c = 0; c < Cfg::kBRowsPerCta / 64; ++c) {
              if constexpr (kCtaGroup == 1)
                tma_load_2d(&tmB, &full[s], sB + s * Cfg::kStageB + c * 8192, b_row + c * 64, kb * 64, kBHint);
              else
                tma_load_2d_pair(&tmB, &full[s], sB + s * Cfg::kStageB + c * 8192, b_row + c * 64, kb * 64, kBHint);
            }
          } else if constexpr (kCtaGroup == 1) {
            mbar_arrive_expect_tx(&full[s], Cfg::kStageBytes);
            tma_load_2d(&tmA, &full[s], sA + s * Cfg::kStageA, kb * kBKElems, a_row, kAHint);
            tma_load_2d(&tmB, &full[s], sB + s * Cfg::kStageB, kb * kBKElems, b_row, kBHint);
          } else if constexpr (kCM == 2) {
            // A: this CTA's rows of its pair's m-tile; B: one 64-row quarter of the n-block's
            // 256 rows (this CTA's half, the pair's share), multicast to the same-half CTA of
            // both pairs. Each pair leader's barrier counts what lands in its two CTAs.
            if (cta_rank == 0) mbar_arrive_expect_tx(&full[s], (active ? 2 * Cfg::kStageA : 0) + 2 * Cfg::kStageB);
            if (active) tma_load_2d_pair(&tmA, &full[s], sA + s * Cfg::kStageA, kb * kBKElems, a_row, kAHint, pleader);
            tma_load_2d_pair_mc(&tmB, &full[s], sB + s * Cfg::kStageB + pair * (Cfg::kStageB / 2), kb * kBKElems,
                                b_row + pair * (Cfg::kBRowsPerCta / 2), (uint16_t)((1u << cta_rank) | (4u << cta_rank)),
                                kBHint, pleader);
          } else {
            if (cta_rank == 0) mbar_arrive_expect_tx(&full[s], 2 * Cfg::kStageBytes);
            tma_load_2d_pair(&tmA, &full[s], sA + s * Cfg::kStageA, kb * kBKElems, a_row, kAHint);
            tma_load_2d_pair(&tmB, &full[s], sB + s * Cfg::kStageB, kb * kBKElems, b_row, kBHint);
          }
          if (++s == S) { s = 0; ph ^= 1; }
        }
        tile = next >= 0 ? next : claim(i + 1);
      }
    }
    __syncwarp();
  } else if (warp == 1) {
    // ===================== MMA issuer (leader CTA) =====================
    if ((kCtaGroup == 1 || cta_rank == 0) && elect_one()) {
      int s = 0;
      uint32_t ph = 0;
      int acc = 0;
      uint32_t aph = 0;
      TileInfo ti;
      for (int i = 0;; ++i) {
        const int tile = take_tile(i, !sched);
        free_tile(i, tile);
        bool active;
        if (tile >= total_tiles || !decode(tile, ti, active)) break;
        if (kCM == 2 && !active) {  // no m-tile for this pair: release the stages the B multicast filled
          for (int kb = 0; kb < ti.nkb; ++kb) {
            mbar_wait(&full[s], ph);
            tc_fence_after();
            mma_commit<kCtaGroup>(&empty[s], all_mask);
            if (++s == S) { s = 0; ph ^= 1; }
          }
          continue;
        }
        mbar_wait(&tempty[acc], aph ^ 1);
        tc_fence_after();
        const uint32_t d_tmem = tmem_base + acc * kBN;
        const uint32_t idesc = (kCtaGroup == 2 && ti.half) ? kIdescHalf : kIdesc;
        for (int kb = 0; kb < ti.nkb; ++kb) {
          mbar_wait(&full[s], ph);
          tc_fence_after();
          // K-major: a K=16 step is 32 B along the swizzled row; MN-major (weight gradients): 16 rows
          const uint64_t adesc = kWgrad ? sdesc_mn_sw128(smem_u32(sA + s * Cfg::kStageA), 8192)
                                        : sdesc_k_sw128(smem_u32(sA + s * Cfg::kStageA));
          const uint64_t bdesc = kWgrad ? sdesc_mn_sw128(smem_u32(sB + s * Cfg::kStageB), 8192)
                                        : sdesc_k_sw128(smem_u32(sB + s * Cfg::kStageB));
          constexpr int kStepBytes = kWgrad ? 16 * 128 : kUmmaKBytes;
#pragma unroll
          for (int k = 0; k < kMmaPerKb; ++k) {
            const uint64_t koff = static_cast<uint64_t>((k * kStepBytes) >> 4);
            mma_ss<kCtaGroup, kFp8>(d_tmem, adesc + koff, bdesc + koff, idesc, (kb | k) != 0);
          }
          mma_commit<kCtaGroup>(&empty[s], kCM == 2 ? all_mask : pair_mask);
          if (++s == S) { s = 0; ph ^= 1; }
        }
        // (an empty k-range commits with no MMA outstanding: the epilogue then writes zeros)
        mma_commit<kCtaGroup>(&tfull[acc], pair_mask);
        if (++acc == 2) { acc = 0; aph ^= 1; }
      }
    }
    __syncwarp();
  } else if (warp >= 4) {
    // ===================== epilogue: TMEM -> registers -> global =====================
    const uint32_t q = warp & 3;  // TMEM lane quarter this warp may access
    const int half = (warp - 4) >> 2;  // which half of the tile's columns this warp handles
    const int row_in_cta = q * 32 + lane;
    int acc = 0;
    uint32_t aph = 0;
    TileInfo ti;
    for (int i = 0;; ++i) {
      const int tile = take_tile(i, !sched);
      __syncwarp();
      if (lane == 0) free_tile(i, tile);
      bool active;
      if (tile >= total_tiles || !decode(tile, ti, active)) break;
      if (!active) continue;  // (kCM == 2) this pair has no m-tile here
      mbar_wait(&tfull[acc], aph);
      tc_fence_after();
      const int row = ti.a_row + cta_rank * Cfg::kRowsPerCta + row_in_cta;
      const bool valid = row < ti.row_end;
      const bool has_acc = ti.nkb > 0;
      const int64_t prow = args.aux_t ? (int64_t)args.poff[ti.e] + (row - args.offsets[ti.e]) : 0;
      const uint32_t t_row = tmem_base + ((q * 32u) << 16) + acc * kBN;
      if constexpr (kEpi == EPI_SWIGLU) {
        float sg = 1.0f, su = 1.0f, so = 1.0f;
        const float* wsg = nullptr;
        const float* wsu = nullptr;
        if constexpr (kFp8) {
          const float sx = args.act_scale[ti.e];
          sg = sx;
          su = sx;
          wsg = args.w_scale + (size_t)ti.e * args.b_rows_per_expert + ti.nt * kBN;
          wsu = wsg + kBN / 2;
        }
        if constexpr (kOutFp8) so = 1.0f / args.out_scale[ti.e];  // act / s_mid as a multiply
        // stores of one 32-channel chunk of one row: A_act (bf16 / e4m3), training H and A^T
        auto emit = [&](int row, int64_t prow, int col, const float* v, const float* gv, const float* uv) {
          if constexpr (kOutFp8) {
            uint32_t p[8];
#pragma unroll
            for (int i = 0; i < 8; ++i) {
              const __nv_fp8x2_storage_t lo = __nv_cvt_float2_to_fp8x2(
                  make_float2(v[4 * i] * so, v[4 * i + 1] * so), __NV_SATFINITE, __NV_E4M3);
              const __nv_fp8x2_storage_t hi = __nv_cvt_float2_to_fp8x2(
                  make_float2(v[4 * i + 2] * so, v[4 * i + 3] * so), __NV_SATFINITE, __NV_E4M3);
              p[i] = static_cast<uint32_t>(lo) | (static_cast<uint32_t>(hi) << 16);
            }
            st_global_v8(reinterpret_cast<uint8_t*>(args.out) + (size_t)row * args.ldo + col, p);
          } else {
            if (args.out)  // (single-GPU training: null — A lives only in the padded copy below)
              store_bf16x32(reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)row * args.ldo + col, v);
            if (args.aux) {  // training: keep H = [G | U] for the SwiGLU backward
              __nv_bfloat16* hrow = reinterpret_cast<__nv_bfloat16*>(args.aux) + (size_t)row * (2 * args.ffn);
              store_bf16x32(hrow + col, gv);
              store_bf16x32(hrow + args.ffn + col, uv);
            }
            if (args.aux_t)  // training: A in the padded row layout (dW_out gradient operand)
              store_bf16x32(reinterpret_cast<__nv_bfloat16*>(args.aux_t) + (size_t)prow * args.ffn + col, v);
          }
        };
        if (kCtaGroup == 2 && ti.half) {
          // M=128 pair tile: TMEM lane r (< 64) holds gate channels of row r, lane 64 + r the up
          // channels of the same row (same columns). Up-lane warps pass their (scaled) values
          // through shared memory; gate-lane warps finish the SwiGLU and store.
          const int r64 = row_in_cta & 63;
          const int hrow = ti.a_row + cta_rank * 64 + r64;
          const bool hvalid = hrow < ti.row_end;
          const int64_t hprow = args.aux_t ? (int64_t)args.poff[ti.e] + (hrow - args.offsets[ti.e]) : 0;
          if (q >= 2) {
#pragma unroll 1
            for (int c = half * 2; c < half * 2 + 2; ++c) {
              uint32_t u[32];
              float wu[32];
              if constexpr (kFp8) load_f32x32(wsu + c * 32, wu);
              tmem_ld32(t_row + c * 32, u);
              tmem_ld_wait();
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                float uv = __uint_as_float(u[i]) * su;
                if constexpr (kFp8) uv *= wu[i];
                xbuf[r64 * Cfg::kXStride + c * 32 + i] = uv;
              }
            }
          }
          named_bar_sync(1, kEpiWarps * 32);
          if (q < 2) {
#pragma unroll 1
            for (int c = half * 2; c < half * 2 + 2; ++c) {
              uint32_t g[32];
              float wg[32];
              if constexpr (kFp8) load_f32x32(wsg + c * 32, wg);
              tmem_ld32(t_row + c * 32, g);
              tmem_ld_wait();
              float v[32], gv[32], uv[32];
#pragma unroll
              for (int i = 0; i < 32; ++i) {
                gv[i] = __uint_as_float(g[i]) * sg;
                if constexpr (kFp8) gv[i] *= wg[i];
                uv[i] = xbuf[r64 * Cfg::kXStride + c * 32 + i];
                v[i] = silu_f(gv[i]) * uv[i];
              }
              if (hvalid) emit(hrow, hprow, ti.nt * (kBN / 2) + c * 32, v, gv, uv);
            }
          }
          named_bar_sync(1, kEpiWarps * 32);  // xbuf free for the next half tile
        } else {
#pragma unroll 1
          for (int c = half * (kBN / 64 / 2); c < (half + 1) * (kBN / 64 / 2); ++c) {
            uint32_t g[32], u[32];
            float wg[32], wu[32];
            if constexpr (kFp8) {
              load_f32x32(wsg + c * 32, wg);
              load_f32x32(wsu + c * 32, wu);
            }
            tmem_ld32(t_row + c * 32, g);
            tmem_ld32(t_row + kBN / 2 + c * 32, u);
            tmem_ld_wait();
            float v[32], gv[32], uv[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              gv[i] = __uint_as_float(g[i]) * sg;
              uv[i] = __uint_as_float(u[i]) * su;
              if constexpr (kFp8) {
                gv[i] *= wg[i];
                uv[i] *= wu[i];
              }
              v[i] = silu_f(gv[i]) * uv[i];
            }
            if (valid) emit(row, prow, ti.nt * (kBN / 2) + c * 32, v, gv, uv);
          }
        }
      } else if constexpr (kEpi == EPI_ROWSCALE) {
        // M=128 pair tile: lane r (< 64) holds columns [0,128) of row r, lane 64 + r columns
        // [128,256) of the same row, both in TMEM columns [0,128).
        const bool ht = kCtaGroup == 2 && ti.half;
        const int erow = ht ? ti.a_row + cta_rank * 64 + (row_in_cta & 63) : row;
        const bool evalid = erow < ti.row_end;
        const int col0 = ht ? (q >= 2 ? kBN / 2 : 0) : 0;
        const int c_lo = ht ? half * 2 : half * (kBN / 64);
        const int c_hi = ht ? half * 2 + 2 : (half + 1) * (kBN / 64);
        float rs = evalid ? (args.row_scale ? args.row_scale[erow] : 1.0f) : 0.0f;
        const float* ws = nullptr;
        if constexpr (kFp8) {
          rs *= args.act_scale[ti.e];
          ws = args.w_scale + (size_t)ti.e * args.b_rows_per_expert + ti.nt * kBN + col0;
        }
#pragma unroll 1
        for (int c = c_lo; c < c_hi; ++c) {
          uint32_t a[32];
          float wv[32];
          if constexpr (kFp8) load_f32x32(ws + c * 32, wv);
          tmem_ld32(t_row + c * 32, a);
          tmem_ld_wait();
          if (evalid) {
            float v[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              v[i] = __uint_as_float(a[i]) * rs;
              if constexpr (kFp8) v[i] *= wv[i];
            }
            const int col = ti.nt * kBN + col0 + c * 32;
            if (args.row_ptr)  // peer transport: the row returns to its source rank over NVLink
              store_bf16x32_plain(static_cast<__nv_bfloat16*>(args.row_ptr[erow]) + col, v);
            else
              store_bf16x32(reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)erow * args.ldo + col, v);
          }
        }
      } else if constexpr (kEpi == EPI_SWIGLU_BWD) {
        // acc = dA for FFN channels [nt*256, nt*256+256); H = [G | U] of the forward pass.
        // H of chunk c+1 is requested before chunk c is processed (hides the global latency).
        const __nv_bfloat16* hrow = reinterpret_cast<const __nv_bfloat16*>(args.aux) + (size_t)row * (2 * args.ffn);
        int4 hg[4], hu[4];
        auto fetch = [&](int c) {
          const int col = ti.nt * kBN + c * 32;
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            hg[i] = *reinterpret_cast<const int4*>(hrow + col + 8 * i);
            hu[i] = *reinterpret_cast<const int4*>(hrow + args.ffn + col + 8 * i);
          }
        };
        const int c_begin = half * (kBN / 64), c_end = (half + 1) * (kBN / 64);
        if (valid) fetch(c_begin);
#pragma unroll 1
        for (int c = c_begin; c < c_end; ++c) {
          uint32_t a[32];
          tmem_ld32(t_row + c * 32, a);
          float g[32], u[32];
#pragma unroll
          for (int i = 0; i < 4; ++i) {
            const __nv_bfloat16* pg = reinterpret_cast<const __nv_bfloat16*>(&hg[i]);
            const __nv_bfloat16* pu = reinterpret_cast<const __nv_bfloat16*>(&hu[i]);
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              g[8 * i + j] = __bfloat162float(pg[j]);
              u[8 * i + j] = __bfloat162float(pu[j]);
            }
          }
          if (valid && c + 1 < c_end) fetch(c + 1);
          tmem_ld_wait();
          if (valid) {
            const int col = ti.nt * kBN + c * 32;
            float dg[32], du[32];
#pragma unroll
            for (int i = 0; i < 32; ++i) {
              const float da = __uint_as_float(a[i]);
              const float s = __fdividef(1.0f, 1.0f + __expf(-g[i]));
              du[i] = da * (g[i] * s);
              dg[i] = da * u[i] * (s * (1.0f + g[i] * (1.0f - s)));
            }
            if (args.out) {  // (training: null — dgrad-2 reads dH from the padded copy below)
              __nv_bfloat16* drow = reinterpret_cast<__nv_bfloat16*>(args.out) + (size_t)row * (2 * args.ffn);
              store_bf16x32(drow + col, dg);
              store_bf16x32(drow + args.ffn + col, du);
            }
            if (args.aux_t) {  // dH in the padded row layout (dW_in gradient operand)
              __nv_bfloat16* t = reinterpret_cast<__nv_bfloat16*>(args.aux_t) + (size_t)prow * (2 * args.ffn);
              store_bf16x32(t + col, dg);
              store_bf16x32(t + args.ffn + col, du);
            }
          }
        }
      } else {  // EPI_WGRAD: fp32 [M][N] per expert
        float* base = reinterpret_cast<float*>(args.out) + (size_t)ti.e * args.out_estride + (size_t)row * args.ldo +
                      ti.nt * kBN;
#pragma unroll 1
        for (int c = half * (kBN / 64); c < (half + 1) * (kBN / 64); ++c) {
          uint32_t a[32];
          if (has_acc) {
            tmem_ld32(t_row + c * 32, a);
            tmem_ld_wait();
          } else {
#pragma unroll
            for (int i = 0; i < 32; ++i) a[i] = 0u;
          }
          float* dst = base + c * 32;
#pragma unroll
          for (int i = 0; i < 4; ++i) st_global_v8(dst + 8 * i, a + 8 * i);
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        // relaxed: the tcgen05 fence above orders the TMEM reads; the tile's global stores need
        // not be complete before the accumulator is reused
        if constexpr (kCtaGroup == 1) mbar_arrive_relaxed(&tempty[acc]);
        else mbar_arrive_cluster_relaxed(&tempty[acc], pleader);
      }
      if (++acc == 2) { acc = 0; aph ^= 1; }
    }
  }

  if constexpr (kEpi == EPI_ROWSCALE)
    if (args.row_ptr && warp >= 4) __threadfence_system();  // peer rows visible before the exchange barrier
  tc_fence_before();
  if constexpr (kCS > 1) cluster_sync(); else __syncthreads();
  tc_fence_after();
  if (warp == 2) tmem_dealloc<kCtaGroup>(tmem_base, 512);
}

}  // namespace cmoe
