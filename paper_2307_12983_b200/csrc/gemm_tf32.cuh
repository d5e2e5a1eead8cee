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
// Structure (one 128 x BN output tile per CTA, 192 threads):
//   warp 0      TMA producer   (one elected lane, kStages-deep smem ring)
//   warp 1      TMEM allocator + MMA issuer (one elected lane)
//   warps 2..5  epilogue: Epi::prepare() preloads per-tile constants while the
//               mainloop runs; then tcgen05.ld 32 columns at a time ->
//               Epi::chunk() -> 128B-swizzled staging in the (now idle)
//               pipeline smem -> TMA bulk tensor store (coalesced, async).
// Split-K over blockIdx.z lets the K=8192 weight-gradient GEMMs fill 148 SMs;
// their epilogue stores partial tiles that a fixed-order reduction sums.
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "ptx.cuh"

namespace pqlg::gemm {

constexpr int kBM = 128;       // UMMA M (cta_group::1)
constexpr int kBK = 32;        // fp32 elements per 128-byte swizzle row
constexpr int kUmmaK = 8;      // K per tcgen05.mma.kind::tf32
constexpr int kThreads = 192;  // 6 warps
constexpr int kScratchBytes = 4096;  // per-tile epilogue constants

struct Operands {
  CUtensorMap a[2];  // one per group (twin critics share a launch)
  CUtensorMap b[2];
  CUtensorMap d[2];  // output maps (Epi::kStoreRank > 0)
};

struct Problem {
  int M, N, K;
  int k_tiles;          // ceil(K / kBK)
  int k_tiles_per_split;
  int splits;
};

template <int BN, int kStages>
struct SmemLayout {
  static constexpr int kABytes = kBM * kBK * 4;        // 16 KB
  static constexpr int kBBytes = BN * kBK * 4;
  static constexpr int kStageBytes = kABytes + kBBytes;
  static constexpr int kPipeBytes = kStages * kStageBytes;
  // epilogue staging reuses the pipeline ring: 4 warps x (BN/32) x 4 KB
  static constexpr int kStageOutBytes = 4 * (BN / 32) * 4096;
  static_assert(kStageOutBytes <= kPipeBytes, "staging must fit in the pipeline smem");
  static constexpr int kScratchOffset = kPipeBytes;
  static constexpr int kBarOffset = kScratchOffset + kScratchBytes;
  // full[kStages], empty[kStages], tmem_full, tmem pointer
  static constexpr int kTotal = kBarOffset + (2 * kStages + 1) * 8 + 16;
  static constexpr int kDynamic = kTotal + 1024;  // slack for 1024B alignment
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

template <int BN, bool kAMN, bool kBMN>
constexpr uint32_t make_idesc() {
  static_assert(BN % 16 == 0 && BN >= 16 && BN <= 256, "UMMA N for M=128");
  uint32_t d = 0;
  d |= 1u << 4;                      // D format f32
  d |= 2u << 7;                      // A format tf32
  d |= 2u << 10;                     // B format tf32
  d |= (kAMN ? 1u : 0u) << 15;       // A major
  d |= (kBMN ? 1u : 0u) << 16;       // B major
  d |= static_cast<uint32_t>(BN >> 3) << 17;
  d |= static_cast<uint32_t>(kBM >> 4) << 24;
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

// Epi concept:
//   static constexpr int kStoreRank;   // 0: Epi stores itself; 2/3: TMA store of v
//   struct Row;                        // per-thread row state
//   __device__ void prepare(Row&, int group, int split, int m, int n_tile, float* scratch) const;
//       called by all 128 epilogue threads before the accumulator is ready;
//       must end with ptx::named_bar_sync(1, 128) if it writes `scratch`.
//   __device__ bool chunk(Row&, int group, int split, int m, int n0, float (&v)[32],
//                         const float* scratch) const;  // transforms v; true = store v
//   __device__ void end(Row&, int group, int split, int m, int n_tile) const;
// `m` may be >= M (rows beyond the problem are zero-filled by TMA; TMA stores
// clip them); the epilogue masks its own direct stores.
template <int BN, int kStages, bool kAMN, bool kBMN, class Epi>
__global__ void __launch_bounds__(kThreads, 1)
    gemm_tf32_kernel(const __grid_constant__ Operands ops, const Problem prob, const Epi epi) {
  using L = SmemLayout<BN, kStages>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) &
                                             ~static_cast<uintptr_t>(1023));
  float* scratch = reinterpret_cast<float*>(smem + L::kScratchOffset);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_full + 1);

  const int warp = threadIdx.x >> 5;
  const int m_tile = blockIdx.x;
  const int n_tile = blockIdx.y;
  const int split = blockIdx.z % prob.splits;
  const int group = blockIdx.z / prob.splits;
  const int kt_begin = split * prob.k_tiles_per_split;
  int kt_end = kt_begin + prob.k_tiles_per_split;
  if (kt_end > prob.k_tiles) kt_end = prob.k_tiles;
  const int n_kt = kt_end > kt_begin ? kt_end - kt_begin : 0;

  constexpr uint32_t kTmemCols = BN < 32 ? 32 : BN;

  if (warp == 0 && ptx::elect_one()) {
    ptx::tma_prefetch(&ops.a[group]);
    ptx::tma_prefetch(&ops.b[group]);
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    ptx::mbar_init(tmem_full, 1);
    ptx::fence_barrier_init();
  }
  if (warp == 1) ptx::tmem_alloc<kTmemCols>(tmem_slot);
  ptx::tc_fence_before();
  __syncthreads();
  ptx::tc_fence_after();
  // everything above overlapped the previous kernel's tail (PDL)
  pdl::entry();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (ptx::elect_one()) {
      const int m0 = m_tile * kBM;
      const int n0 = n_tile * BN;
      for (int i = 0; i < n_kt; ++i) {
        const int s = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        ptx::mbar_wait(&empty[s], ph ^ 1);
        uint8_t* sa = smem + s * L::kStageBytes;
        uint8_t* sb = sa + L::kABytes;
        ptx::mbar_arrive_expect_tx(&full[s], L::kStageBytes);
        const int k0 = (kt_begin + i) * kBK;
        if constexpr (kAMN) {
#pragma unroll
          for (int j = 0; j < kBM / 32; ++j)
            ptx::tma_load_2d(&ops.a[group], &full[s], sa + j * (32 * kBK * 4), m0 + 32 * j, k0);
        } else {
          ptx::tma_load_2d(&ops.a[group], &full[s], sa, k0, m0);
        }
        if constexpr (kBMN) {
#pragma unroll
          for (int j = 0; j < BN / 32; ++j)
            ptx::tma_load_2d(&ops.b[group], &full[s], sb + j * (32 * kBK * 4), n0 + 32 * j, k0);
        } else {
          ptx::tma_load_2d(&ops.b[group], &full[s], sb, k0, n0);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc<BN, kAMN, kBMN>();
    if (ptx::elect_one()) {
      for (int i = 0; i < n_kt; ++i) {
        const int s = i % kStages;
        const uint32_t ph = (i / kStages) & 1;
        ptx::mbar_wait(&full[s], ph);
        ptx::tc_fence_after();
        const uint32_t sa = ptx::smem_u32(smem + s * L::kStageBytes);
        const uint32_t sb = sa + L::kABytes;
#pragma unroll
        for (int j = 0; j < kBK / kUmmaK; ++j) {
          const uint64_t ad = operand_desc<kAMN>(sa + j * k_step_bytes<kAMN>());
          const uint64_t bd = operand_desc<kBMN>(sb + j * k_step_bytes<kBMN>());
          ptx::mma_tf32(tmem_base, ad, bd, idesc, (i > 0 || j > 0) ? 1u : 0u);
        }
        ptx::mma_commit(&empty[s]);
      }
      ptx::mma_commit(tmem_full);
    }
    __syncwarp();
  } else {
    // Epilogue warps 2..5: TMEM lane quadrant = warp % 4.
    const int q = warp & 3;
    const int lane = threadIdx.x & 31;
    const int row0 = m_tile * kBM + q * 32;
    const int m = row0 + lane;
    typename Epi::Row row;
    epi.prepare(row, group, split, m, n_tile, scratch);
    if (n_kt > 0) {
      ptx::mbar_wait(tmem_full, 0);
      ptx::tc_fence_after();
    }
    // staging for this warp: (BN/32) buffers of 32 rows x 128 B (SW128)
    uint8_t* stage = smem + q * (BN / 32) * 4096;
#pragma unroll 1
    for (int c = 0; c < BN / 32; ++c) {
      float v[32];
      if (n_kt > 0) {
        uint32_t r[32];
        ptx::tmem_ld32(tmem_base + (static_cast<uint32_t>(q * 32) << 16) + c * 32, r);
        ptx::tmem_ld_wait();
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = __uint_as_float(r[t]);
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t) v[t] = 0.0f;
      }
      const int n0 = n_tile * BN + c * 32;
      const bool st = epi.chunk(row, group, split, m, n0, v, scratch);
      if constexpr (Epi::kStoreRank > 0) {
        if (st) {
          uint8_t* buf = stage + c * 4096;
#pragma unroll
          for (int j = 0; j < 8; ++j) {
            float4* dst = reinterpret_cast<float4*>(buf + lane * 128 + ((j ^ (lane & 7)) << 4));
            *dst = make_float4(v[4 * j], v[4 * j + 1], v[4 * j + 2], v[4 * j + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            if constexpr (Epi::kStoreRank == 2) {
              tma_store_2d(&ops.d[group], buf, n0, row0);
            } else {
              tma_store_3d(&ops.d[0], buf, n0, row0, group * prob.splits + split);
            }
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
        }
      }
    }
    epi.end(row, group, split, m, n_tile);
    if constexpr (Epi::kStoreRank > 0) {
      if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
      __syncwarp();
    }
  }

  ptx::tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    ptx::tmem_dealloc<kTmemCols>(tmem_base);
  }
}

}  // namespace pqlg::gemm
