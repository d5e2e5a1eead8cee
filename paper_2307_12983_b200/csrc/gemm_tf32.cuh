// tcgen05 TF32 GEMM family for the MLP layers of the learners and the actor.
//
//   D[m, n] = sum_k A(m, k) * B(n, k)        fp32 storage, tf32 multiply,
//                                            fp32 accumulation in TMEM
//
// The reference computes every layer with three fp32 loops
// (pql/kernels/scalar.hpp:12-55 / src/kernels/avx2.cpp:37-300):
//   forward  out = in * W            A = activations  (K-major),  B = W (N-major)
//   dgrad    din = g * W^T           A = g            (K-major),  B = W (K-major)
//   wgrad    dW  = in^T * g          A = activations  (M-major),  B = g (N-major)
// so one kernel template covers all three by choosing each operand's major
// mode.  K-major operands use the 128B swizzle; MN-major tf32 operands must use
// the 128B/32B-atom swizzle (the only MN-major tf32 smem layout UMMA accepts).
// Operand tensor maps are typed TFLOAT32 so TMA rounds fp32 -> tf32 to
// nearest on the way into shared memory (the MMA alone would truncate).
//
// Structure: a persistent kernel (grid = min(tiles, SMs), one CTA per SM)
// walking 128 x BN output tiles round-robin:
//   warp 0      TMA producer   (one elected lane, kStages-deep smem ring that
//               runs on across tile boundaries)
//   warp 1      TMEM allocator + MMA issuer (one elected lane); the
//               accumulator is double-buffered in TMEM (2 x BN columns), so
//               tile i+1's mainloop runs while the epilogue drains tile i
//   warps 2..   epilogue (4 warps, or 8 when the tile is >= 128 columns wide:
//               two warps per TMEM lane quadrant, one per column half):
//               Epi::prepare() loads per-tile constants, then tcgen05.ld 32
//               columns at a time -> Epi::chunk() -> 128B-swizzled staging
//               (two 4 KB buffers per warp) -> TMA bulk tensor store.
// Split-K over the z tile coordinate lets the K=8192 weight-gradient GEMMs
// fill 148 SMs; their epilogue stores partial tiles that a fixed-order
// reduction sums.
//
// k3x (the fp32-faithful "3xTF32" mode, pqlg_config::precision): operands
// arrive as raw fp32 (FLOAT32 tensor maps), four converter warps split every
// stage in shared memory into x_hi = rna_tf32(x) (in place) and
// x_lo = rna_tf32(x - x_hi) (a mirror region of the stage), and the MMA warp
// issues lo_A*hi_B + hi_A*lo_B + hi_A*hi_B per UMMA K step into the same TMEM
// accumulator.  The representation error is ~2^-24 |x|, so products match
// fp32 to a few ulps (the dropped lo*lo term is ~2^-22 relative) at 3x the
// MMA work.
#pragma once

#include <cstdint>

#include "epilogues.cuh"
#include "pdl.cuh"
#include "ptx.cuh"

namespace pqlg::gemm {

// Phase timestamps per CTA (tools/gemm_trace.cu builds a traced copy of the
// kernel with -DPQLG_GEMM_TRACE; the library itself never defines it).
#ifdef PQLG_GEMM_TRACE
__device__ unsigned long long* g_trace;
__device__ __forceinline__ unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
#define PQLG_TRACE(slot, value)                                                       \
  do {                                                                                \
    if (g_trace) {                                                                    \
      const unsigned bid = blockIdx.x + gridDim.x * (blockIdx.y + gridDim.y * blockIdx.z); \
      g_trace[bid * 16 + (slot)] = (value);                                           \
    }                                                                                 \
  } while (0)
#else
#define PQLG_TRACE(slot, value) \
  do {                          \
  } while (0)
#endif

constexpr int kBM = 128;       // UMMA M (cta_group::1)
constexpr int kBK = 32;        // fp32 elements per 128-byte swizzle row
constexpr int kUmmaK = 8;      // K per tcgen05.mma.kind::tf32
constexpr int kScratchBytes = 2048;  // per-tile epilogue constants
constexpr int kMaxDynSmem = 232448;  // 227 KB per CTA on sm_100

constexpr int kMaxGroups = 4;  // online + target twin critics share one launch

struct Operands {
  CUtensorMap a[kMaxGroups];  // one per group
  CUtensorMap b[kMaxGroups];
  CUtensorMap d[kMaxGroups];  // output maps (Epi::kStoreRank > 0)
};

struct Problem {
  int M, N, K;
  int k_tiles;          // ceil(K / kBK)
  int k_tiles_per_split;
  int splits;
  int groups;
};

// Epilogue warp count: two warps per TMEM lane quadrant (column halves) for
// tiles >= 128 columns whose epilogue supports it (four per quadrant was
// measured slower: DESIGN 9c).
template <int BN, class Epi, bool kPair = false, bool k3x = false>
constexpr int epi_warps() {
  return (BN >= 128 && Epi::kSplitCols) ? 8 : 4;
}

constexpr int kConvWarps = 4;  // 3xTF32 hi/lo converter warps

// kPair: the tile is computed by a CTA pair (cluster of 2, tcgen05
// cta_group::2, UMMA M = 256): each CTA stages its own 128 A rows and half of
// the BN B columns, so per-CTA operand traffic drops from (128 + BN) to
// (128 + BN/2) rows per k-step -- the hidden-layer GEMMs are L2-bandwidth
// bound at 1 CTA per tile.
template <int BN, class Epi, bool kPair = false, bool k3x = false>
struct SmemLayout {
  static constexpr int kEpiWarps = epi_warps<BN, Epi, kPair, k3x>();
  static constexpr int kConvWarps3 = k3x ? kConvWarps : 0;
  static constexpr int kThreads = 64 + 32 * kEpiWarps + 32 * kConvWarps3;
  static constexpr int kABytes = kBM * kBK * 4;  // 16 KB
  static constexpr int kBBytes = (kPair ? BN / 2 : BN) * kBK * 4;
  static constexpr int kLoadBytes = kABytes + kBBytes;  // TMA bytes per stage and CTA
  // 3xTF32: [A_hi | B_hi | A_lo | B_lo] per stage
  static constexpr int kStageBytes = k3x ? 2 * kLoadBytes : kLoadBytes;
  // one 4 KB (32 x 32 fp32, 128B-swizzled) TMA-store staging buffer per warp
  // (a second one per warp was measured slower: tools/gpu_ab2.sh, DESIGN 9c)
  static constexpr int kStagingBytes = Epi::kStoreRank > 0 ? kEpiWarps * 4096 : 0;
  static constexpr int kFixed = kStagingBytes + kScratchBytes + 256;
  static constexpr int kFit = (kMaxDynSmem - kFixed) / kStageBytes;
  static constexpr int kStages = kFit > 8 ? 8 : kFit;
  static_assert(kStages >= (k3x ? 2 : 4), "pipeline too shallow");
  static constexpr int kPipeBytes = kStages * kStageBytes;
  static constexpr int kStagingOffset = kPipeBytes;
  static constexpr int kScratchOffset = kStagingOffset + kStagingBytes;
  static constexpr int kBarOffset = kScratchOffset + kScratchBytes;
  // full[kStages], empty[kStages], tmem_full[2], tmem_empty[2],
  // (3xTF32) conv[kStages], tmem pointer
  static constexpr int kTotal = kBarOffset + ((k3x ? 3 : 2) * kStages + 4) * 8 + 16;
  // the dynamic window starts 1024B-aligned (no static smem in this kernel;
  // checked at entry), so no alignment slack is reserved
  static constexpr int kDynamic = kTotal;
  static_assert(kDynamic <= kMaxDynSmem, "shared memory budget");
  static constexpr uint32_t kTmemCols = 2 * BN < 32 ? 32 : 2 * BN;  // double-buffered accumulator
};

// UMMA shared-memory descriptor (sm_100 "version 1" format).
__device__ __forceinline__ uint64_t make_desc(uint32_t saddr, uint32_t lbo, uint32_t sbo,
                                              uint32_t layout) {
  uint64_t d = 0;
  d |= static_cast<uint64_t>((saddr >> 4) & 0x3FFF);
  d |= static_cast<uint64_t>((lbo >> 4) & 0x3FFF) << 16;
  d |= static_cast<uint64_t>((sbo >> 4) & 0x3FFF) << 32;
  d |= static_cast<uint64_t>(1) << 46;  // version
  d |= static_cast<uint64_t>(layout & 0x7) << 61;
  return d;
}

constexpr uint32_t kLayoutSW128 = 2;
constexpr uint32_t kLayoutSW128Base32 = 1;

template <bool kMN>
__device__ __forceinline__ uint64_t operand_desc(uint32_t saddr) {
  if constexpr (kMN) {
    // ((32 elems, n atoms), (4 rows, k atoms)) : ((1, LBO), (128B, SBO))
    return make_desc(saddr, /*lbo=*/kBK * 128, /*sbo=*/512, kLayoutSW128Base32);
  } else {
    // ((8 rows, m groups), 32 elems) : ((128B, SBO), 1)
    return make_desc(saddr, /*lbo=*/0, /*sbo=*/1024, kLayoutSW128);
  }
}

// Byte advance of the descriptor start address per UMMA K step.
template <bool kMN>
constexpr uint32_t k_step_bytes() {
  return kMN ? kUmmaK * 128 : kUmmaK * 4;
}

template <int BN, bool kAMN, bool kBMN, bool kPair = false>
constexpr uint32_t make_idesc() {
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N");
  uint32_t d = 0;
  d |= 1u << 4;                      // D format f32
  d |= 2u << 7;                      // A format tf32
  d |= 2u << 10;                     // B format tf32
  d |= (kAMN ? 1u : 0u) << 15;       // A major
  d |= (kBMN ? 1u : 0u) << 16;       // B major
  d |= static_cast<uint32_t>(BN >> 3) << 17;
  d |= static_cast<uint32_t>((kPair ? 2 * kBM : kBM) >> 4) << 24;
  return d;
}

__device__ __forceinline__ void tma_store_2d(const CUtensorMap* map, const void* smem, int32_t c0,
                                             int32_t c1) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(ptx::smem_u32(smem)), "r"(c0), "r"(c1)
      : "memory");
}

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* smem, int32_t c0,
                                             int32_t c1, int32_t c2) {
  asm volatile(
      "cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];" ::"l"(
          reinterpret_cast<uint64_t>(map)),
      "r"(ptx::smem_u32(smem)), "r"(c0), "r"(c1), "r"(c2)
      : "memory");
}

// Epi concept (see epilogues.cuh, epi::Ctx):
//   static constexpr int kStoreRank;   // 0: Epi stores itself; 2/3: TMA store of v
//   static constexpr bool kSplitCols;  // two warps may share a row (column halves)
//   struct Row;                        // per-thread row state
//   __device__ void prepare(Row&, const epi::Ctx&, float* scratch) const;
//       per tile, all epilogue threads, before the accumulator is ready; the
//       kernel synchronises the epilogue threads before and after it
//   __device__ bool chunk(Row&, const epi::Ctx&, int n0, float (&v)[32], float* scratch) const;
//       transforms v (columns n0..n0+31 of the row); true = TMA-store v
//   __device__ void end(Row&, const epi::Ctx&) const;
// `m` may be >= M (rows beyond the problem are zero-filled by TMA; TMA stores
// clip them); the epilogue masks its own direct stores.
struct TileCoord {
  int m_tile, n_tile, split, group;
};

__device__ __forceinline__ TileCoord tile_coord(int t, const Problem& p, int tiles_m,
                                                int tiles_n) {
  TileCoord c;
  c.m_tile = t % tiles_m;
  const int r = t / tiles_m;
  c.n_tile = r % tiles_n;
  const int z = r / tiles_n;
  c.split = z % p.splits;
  c.group = z / p.splits;
  return c;
}

// One converter pass over stage `st` (3xTF32): x -> (hi in place, lo mirror).
template <int kLoadBytes>
__device__ __forceinline__ void split_stage(uint8_t* st, int ct) {
  float4* hi = reinterpret_cast<float4*>(st);
  float4* lo = reinterpret_cast<float4*>(st + kLoadBytes);
  constexpr int kVec = kLoadBytes / 16;
  constexpr int kT = 32 * kConvWarps;
  static_assert(kVec % kT == 0, "stage size");
#pragma unroll 4
  for (int e = ct; e < kVec; e += kT) {
    const float4 x = hi[e];
    float4 h, l;
    h.x = ptx::to_tf32(x.x);
    h.y = ptx::to_tf32(x.y);
    h.z = ptx::to_tf32(x.z);
    h.w = ptx::to_tf32(x.w);
    l.x = ptx::to_tf32(__fsub_rn(x.x, h.x));
    l.y = ptx::to_tf32(__fsub_rn(x.y, h.y));
    l.z = ptx::to_tf32(__fsub_rn(x.z, h.z));
    l.w = ptx::to_tf32(__fsub_rn(x.w, h.w));
    hi[e] = h;
    lo[e] = l;
  }
}

template <int BN, bool kAMN, bool kBMN, class Epi, bool kPair = false, bool k3x = false>
__global__ void __launch_bounds__(SmemLayout<BN, Epi, kPair, k3x>::kThreads, 1)
    gemm_tf32_kernel(const __grid_constant__ Operands ops, const Problem prob,
                     const __grid_constant__ Epi epi) {
  using L = SmemLayout<BN, Epi, kPair, k3x>;
  constexpr int kStages = L::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((ptx::smem_u32(smem) & 1023) != 0) __trap();  // SW128 tiles need 1024B alignment
  float* scratch = reinterpret_cast<float*>(smem + L::kScratchOffset);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;   // [2]
  uint64_t* tmem_empty = tmem_full + 2;    // [2]
  uint64_t* conv = tmem_empty + 2;         // [kStages] (3xTF32 only)
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(conv + (k3x ? kStages : 0));

  const int warp = threadIdx.x >> 5;
  const int tiles_m = (prob.M + kBM - 1) / kBM;
  const int tiles_n = (prob.N + BN - 1) / BN;
  // Work units: tiles (1 CTA each) or, paired, m-tile pairs (cluster of 2).
  const uint32_t rank = kPair ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit_m = kPair ? tiles_m / 2 : tiles_m;
  const int n_units = unit_m * tiles_n * prob.splits * prob.groups;
  const int unit0 = kPair ? static_cast<int>(ptx::cluster_id_x()) : static_cast<int>(blockIdx.x);
  const int unit_step = kPair ? static_cast<int>(ptx::nclusters_x()) : static_cast<int>(gridDim.x);
  auto coord = [&](int u) {
    TileCoord c = tile_coord(u, prob, unit_m, tiles_n);
    if constexpr (kPair) c.m_tile = 2 * c.m_tile + static_cast<int>(rank);
    return c;
  };

  if (warp == 0 && ptx::elect_one()) {
    for (int g = 0; g < prob.groups; ++g) {
      ptx::tma_prefetch(&ops.a[g]);
      ptx::tma_prefetch(&ops.b[g]);
    }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
      // the leader's MMA waits for every converter warp of the pair
      if constexpr (k3x) ptx::mbar_init(&conv[s], kConvWarps * (kPair ? 2 : 1));
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      // the leader's MMA waits for both CTAs' epilogues to drain a buffer
      ptx::mbar_init(&tmem_empty[a], L::kEpiWarps * (kPair ? 2 : 1));
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (kPair) ptx::tmem_alloc_pair<L::kTmemCols>(tmem_slot);
    else ptx::tmem_alloc<L::kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (kPair) ptx::cluster_sync();  // barrier inits + TMEM visible to the peer
  else __syncthreads();
  ptx::tc_fence_after();
  // everything above overlapped the previous kernel's tail (PDL)
  pdl::entry();
  const uint32_t tmem_base = *tmem_slot;
#ifdef PQLG_GEMM_TRACE
  if (threadIdx.x == 0) {
    PQLG_TRACE(0, gtimer());
    PQLG_TRACE(1, clock64());
    unsigned sm;
    asm("mov.u32 %0, %%smid;" : "=r"(sm));
    PQLG_TRACE(7, sm);
  }
#endif

  auto k_range = [&](int split, int& kt0, int& nkt) {
    kt0 = split * prob.k_tiles_per_split;
    int kt1 = kt0 + prob.k_tiles_per_split;
    if (kt1 > prob.k_tiles) kt1 = prob.k_tiles;
    nkt = kt1 - kt0;  // >= 1: make_problem never creates an empty split
  };

  if (warp == 0) {
    if (ptx::elect_one()) {
      constexpr int kBCols = kPair ? BN / 2 : BN;  // B columns staged by this CTA
      uint32_t it = 0;
      for (int u = unit0; u < n_units; u += unit_step) {
        const TileCoord tc = coord(u);
        int kt0, nkt;
        k_range(tc.split, kt0, nkt);
        const int m0 = tc.m_tile * kBM;
        const int n0 = tc.n_tile * BN + static_cast<int>(rank) * kBCols;
        for (int i = 0; i < nkt; ++i, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          ptx::mbar_wait(&empty[s], ph ^ 1);
          uint8_t* sa = smem + s * L::kStageBytes;
          uint8_t* sb = sa + L::kABytes;
          const int k0 = (kt0 + i) * kBK;
          if constexpr (kPair && !k3x) {
            // both CTAs' bytes complete on the leader's full barrier
            if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * L::kLoadBytes);
            const uint32_t fb = ptx::mapa(&full[s], 0);
            if constexpr (kAMN) {
#pragma unroll
              for (int j = 0; j < kBM / 32; ++j)
                ptx::tma_load_2d_pair(&ops.a[tc.group], fb, sa + j * (32 * kBK * 4), m0 + 32 * j, k0);
            } else {
              ptx::tma_load_2d_pair(&ops.a[tc.group], fb, sa, k0, m0);
            }
            if constexpr (kBMN) {
#pragma unroll
              for (int j = 0; j < kBCols / 32; ++j)
                ptx::tma_load_2d_pair(&ops.b[tc.group], fb, sb + j * (32 * kBK * 4), n0 + 32 * j, k0);
            } else {
              ptx::tma_load_2d_pair(&ops.b[tc.group], fb, sb, k0, n0);
            }
          } else {
            // (3xTF32 pairs: each CTA's bytes complete on its own barrier,
            // where its converter warps wait)
            ptx::mbar_arrive_expect_tx(&full[s], L::kLoadBytes);
            if constexpr (kAMN) {
#pragma unroll
              for (int j = 0; j < kBM / 32; ++j)
                ptx::tma_load_2d(&ops.a[tc.group], &full[s], sa + j * (32 * kBK * 4), m0 + 32 * j,
                                 k0);
            } else {
              ptx::tma_load_2d(&ops.a[tc.group], &full[s], sa, k0, m0);
            }
            if constexpr (kBMN) {
#pragma unroll
              for (int j = 0; j < kBCols / 32; ++j)
                ptx::tma_load_2d(&ops.b[tc.group], &full[s], sb + j * (32 * kBK * 4), n0 + 32 * j,
                                 k0);
            } else {
              ptx::tma_load_2d(&ops.b[tc.group], &full[s], sb, k0, n0);
            }
          }
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc<BN, kAMN, kBMN, kPair>();
    if (leader && ptx::elect_one()) {
      uint32_t it = 0, lt = 0;
      for (int u = unit0; u < n_units; u += unit_step, ++lt) {
        const TileCoord tc = coord(u);
        int kt0, nkt;
        k_range(tc.split, kt0, nkt);
        const uint32_t a = lt & 1;
        ptx::mbar_wait(&tmem_empty[a], ((lt >> 1) & 1) ^ 1);  // epilogue(s) drained this buffer
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + a * BN;
        for (int i = 0; i < nkt; ++i, ++it) {
          const int s = it % kStages;
          const uint32_t ph = (it / kStages) & 1;
          if constexpr (k3x && kPair) ptx::mbar_wait_cluster(&conv[s], ph);
          else if constexpr (k3x) ptx::mbar_wait(&conv[s], ph);
          else ptx::mbar_wait(&full[s], ph);
          ptx::tc_fence_after();
#ifdef PQLG_GEMM_TRACE
          if (it == 0) PQLG_TRACE(2, clock64());
#endif
          const uint32_t sa = ptx::smem_u32(smem + s * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
          auto mma = [&](uint64_t ad, uint64_t bd, uint32_t acc) {
            if constexpr (kPair) ptx::mma_tf32_pair(d_tmem, ad, bd, idesc, acc);
            else ptx::mma_tf32(d_tmem, ad, bd, idesc, acc);
          };
#pragma unroll
          for (int j = 0; j < kBK / kUmmaK; ++j) {
            const uint64_t ad = operand_desc<kAMN>(sa + j * k_step_bytes<kAMN>());
            const uint64_t bd = operand_desc<kBMN>(sb + j * k_step_bytes<kBMN>());
            const uint32_t acc = (i > 0 || j > 0) ? 1u : 0u;
            if constexpr (k3x) {
              const uint64_t al = operand_desc<kAMN>(sa + L::kLoadBytes + j * k_step_bytes<kAMN>());
              const uint64_t bl = operand_desc<kBMN>(sb + L::kLoadBytes + j * k_step_bytes<kBMN>());
              mma(al, bd, acc);  // small terms first
              mma(ad, bl, 1u);
              mma(ad, bd, 1u);
            } else {
              mma(ad, bd, acc);
            }
          }
          if constexpr (kPair) ptx::mma_commit_pair(&empty[s]);
          else ptx::mma_commit(&empty[s]);
        }
        if constexpr (kPair) ptx::mma_commit_pair(&tmem_full[a]);
        else ptx::mma_commit(&tmem_full[a]);
#ifdef PQLG_GEMM_TRACE
        if (lt == 0) PQLG_TRACE(14, clock64());
#endif
      }
#ifdef PQLG_GEMM_TRACE
      PQLG_TRACE(3, clock64());
#endif
    }
    __syncwarp();
  } else if (k3x && warp >= 2 + L::kEpiWarps) {
    // 3xTF32 converter warps: split each landed stage into hi / lo, make the
    // generic-proxy stores visible to the tensor core (async proxy), then
    // arrive on the MMA leader's conv barrier.
    const int ct = threadIdx.x - 32 * (2 + L::kEpiWarps);
    const int lane = threadIdx.x & 31;
    uint32_t it = 0;
    for (int u = unit0; u < n_units; u += unit_step) {
      const TileCoord tc = coord(u);
      int kt0, nkt;
      k_range(tc.split, kt0, nkt);
      for (int i = 0; i < nkt; ++i, ++it) {
        const int s = it % kStages;
        ptx::mbar_wait(&full[s], (it / kStages) & 1);
        split_stage<L::kLoadBytes>(smem + s * L::kStageBytes, ct);
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          if constexpr (kPair) ptx::mbar_arrive_cluster_release(ptx::mapa(&conv[s], 0));
          else ptx::mbar_arrive(&conv[s]);
        }
      }
    }
  } else {
    // Epilogue: warp w reads TMEM lane quadrant w % 4 (hardware rule) and
    // column half (w - 2) / 4 of the tile.
    constexpr int kHalves = L::kEpiWarps / 4;
    constexpr int kChunks = BN / 32;
    constexpr int kChunksPerWarp = kChunks / kHalves;
    const int ew = warp - 2;
    const int q = warp & 3;
    const int lane = threadIdx.x & 31;
    epi::Ctx ctx{};
    ctx.et = threadIdx.x - 64;
    ctx.ne = 32 * L::kEpiWarps;
    ctx.half = ew >> 2;
    ctx.halves = kHalves;
    uint8_t* stage = smem + L::kStagingOffset + ew * 4096;
    uint32_t nstore = 0;
    uint32_t lt = 0;
    for (int u = unit0; u < n_units; u += unit_step, ++lt) {
      const TileCoord tc = coord(u);
      ctx.group = tc.group;
      ctx.split = tc.split;
      ctx.n_tile = tc.n_tile;
      ctx.m_tile = tc.m_tile;
      ctx.row0 = tc.m_tile * kBM + q * 32;
      ctx.m = ctx.row0 + lane;
      const uint32_t a = lt & 1;
      if (lt > 0) ptx::named_bar_sync(1, 32 * L::kEpiWarps);  // previous tile done with scratch
      typename Epi::Row row;
      epi.prepare(row, ctx, scratch);
      ptx::named_bar_sync(1, 32 * L::kEpiWarps);
      ptx::mbar_wait(&tmem_full[a], (lt >> 1) & 1);
      ptx::tc_fence_after();
#ifdef PQLG_GEMM_TRACE
      if (threadIdx.x == 64 && lt == 0) PQLG_TRACE(4, clock64());
      if (threadIdx.x == 64 && lt == 1) PQLG_TRACE(13, clock64());
#endif
      const uint32_t t_addr = tmem_base + (static_cast<uint32_t>(q * 32) << 16) + a * BN;
      uint32_t r[32];
      const int c_begin = ctx.half * kChunksPerWarp;
      ptx::tmem_ld32(t_addr + c_begin * 32, r);
#pragma unroll 1
      for (int c = c_begin; c < c_begin + kChunksPerWarp; ++c) {
        ptx::tmem_ld_wait();
        float v[32];
#pragma unroll
        for (int uu = 0; uu < 32; ++uu) v[uu] = __uint_as_float(r[uu]);
        // next chunk's TMEM load overlaps this chunk's math and stores
        if (c + 1 < c_begin + kChunksPerWarp) ptx::tmem_ld32(t_addr + (c + 1) * 32, r);
        const int n0 = tc.n_tile * BN + c * 32;
        const bool st = epi.chunk(row, ctx, n0, v, scratch);
        if constexpr (Epi::kStoreRank > 0) {
          if (st) {
            uint8_t* buf = stage;
            // the previous store from this buffer has finished reading it
            if (lane == 0 && nstore > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; ++j) {
              float4* dst = reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
              *dst = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
            }
            asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
            __syncwarp();
            if (lane == 0) {
              if constexpr (Epi::kStoreRank == 2) {
                tma_store_2d(&ops.d[tc.group], buf, n0, ctx.row0);
              } else {
                tma_store_3d(&ops.d[0], buf, n0, ctx.row0, tc.group * prob.splits + tc.split);
              }
              asm volatile("cp.async.bulk.commit_group;" ::: "memory");
            }
            ++nstore;
          }
        }
#ifdef PQLG_GEMM_TRACE
        if (threadIdx.x == 64 && lt == 0 && c - c_begin < 4) PQLG_TRACE(8 + c - c_begin, clock64());
#endif
      }
      // every tcgen05.ld of this warp has completed: release the accumulator
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair) ptx::mbar_arrive_cluster(ptx::mapa(&tmem_empty[a], 0));
        else ptx::mbar_arrive(&tmem_empty[a]);
      }
      epi.end(row, ctx);
#ifdef PQLG_GEMM_TRACE
      if (threadIdx.x == 64 && lt == 0) PQLG_TRACE(12, clock64());
#endif
    }
    if constexpr (Epi::kStoreRank > 0) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
      __syncwarp();
    }
#ifdef PQLG_GEMM_TRACE
    if (threadIdx.x == 64) {
      PQLG_TRACE(5, clock64());
      PQLG_TRACE(6, gtimer());
    }
#endif
  }

  ptx::tc_fence_before();
  if constexpr (kPair) ptx::cluster_sync();  // no remote arrive may target an exited CTA
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (kPair) ptx::tmem_dealloc_pair<L::kTmemCols>(tmem_base);
    else ptx::tmem_dealloc<L::kTmemCols>(tmem_base);
  }
}

}  // namespace pqlg::gemm
