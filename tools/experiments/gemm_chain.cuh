// Layer-chained persistent GEMM: the hidden layers of an MLP (and up to 4
// independent nets of the same shape) in ONE persistent launch.
//
//   layer l, group g:  D_l,g = epi_l( A_l,g * W_l,g )     A_0,g = input,
//                                                         A_l,g = D_(l-1),g
//
// Separate launches per layer pay, every layer, a pipeline fill, the last
// tile's exposed epilogue and the wave quantisation of the layer's tile
// count over 148 SMs (a 128-tile layer on 148 SMs is one partial wave).
// Here the tiles of all layers form one work list: a CTA claims the next
// unit (an atomic counter), so tiles of layer l+1 start as soon as the rows
// they read are complete, while other SMs still finish layer l.
//
// Dependencies: unit (l, g, m-block, n-tile) reads rows [128 m, 128 m + 128)
// of D_(l-1),g, all columns.  Every epilogue warp, after its TMA stores of a
// tile have fully completed (cp.async.bulk.wait_group 0), fences and adds 1
// to done[l][g][m]; the producer of a layer-(l+1) unit spins (acquire) until
// that count reaches n_tiles x epilogue warps, then issues its TMA loads.
// Units are claimed in increasing order and depend only on smaller units,
// which were claimed by running CTAs -- so the chain makes progress even
// when only part of the grid is resident (other streams' kernels on the SMs).
//
// Per CTA (same roles as gemm_tf32_kernel, one 128 x BN tile per unit):
//   warp 0      producer: claims units, hands them to the MMA / epilogue
//               warps through a 4-deep ring, waits for dependencies, TMA
//   warp 1      TMEM allocation + MMA issue (double-buffered accumulator)
//   warps 2..   epilogue (epi::Hidden of the unit's layer), TMA stores, done
// kPair: a unit is a 256 x BN tile computed by a CTA pair (cta_group::2, as
// gemm_tf32_kernel's pairs: each CTA stages its 128 A rows and half of B,
// halving the per-SM operand traffic the TF32 mainloop is bound by).  The
// leader's producer claims the unit and writes it into both CTAs' rings
// (st.shared::cluster + a cluster-scope release arrive); every consumer of
// both CTAs releases the slot on the leader's barrier.
// The last CTA to exit resets the claim counter and the done counters, so
// the launch can be replayed from a CUDA graph.
#pragma once

#include <cstdint>

#include "gemm_tf32.cuh"

namespace pqlg::gemm {

constexpr int kChainLayers = 3;  // max layers per chain
constexpr int kUnitRing = 4;

struct ChainOperands {
  CUtensorMap a[kChainLayers][kMaxGroups];
  CUtensorMap b[kChainLayers][kMaxGroups];
  CUtensorMap d[kChainLayers][kMaxGroups];
};

struct ChainProblem {
  int M, N;  // rows and output columns of every layer
  int layers, groups;
  int k_tiles[kChainLayers];
  // [0] claim counter, [1] exit ticket, then done[layers][groups][m_tiles]
  unsigned int* sync;
};

template <class Epi>
struct ChainEpi {
  Epi e[kChainLayers];
};

template <int BN, class Epi, bool kPair>
struct ChainLayout {
  using L = SmemLayout<BN, Epi, kPair, false>;
  // after L's barriers: unit slots [kUnitRing] (int), unit_full / unit_empty
  static constexpr int kRingOffset = (L::kTotal + 15) & ~15;
  static constexpr int kDynamic = kRingOffset + kUnitRing * 4 + 2 * kUnitRing * 8;
  static_assert(kDynamic <= kMaxDynSmem, "shared memory budget");
};

__device__ __forceinline__ unsigned int ld_acquire_u32(const unsigned int* p) {
  unsigned int v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

__device__ __forceinline__ void st_cluster_u32(uint32_t cluster_addr, int v) {
  asm volatile("st.shared::cluster.u32 [%0], %1;" ::"r"(cluster_addr), "r"(v) : "memory");
}

template <int BN, class Epi, bool kPair>
__global__ void __launch_bounds__(SmemLayout<BN, Epi, kPair, false>::kThreads, 1)
    chain_gemm_kernel(const __grid_constant__ ChainOperands ops, const ChainProblem prob,
                      const __grid_constant__ ChainEpi<Epi> epi) {
  using L = SmemLayout<BN, Epi, kPair, false>;
  using CL = ChainLayout<BN, Epi, kPair>;
  constexpr int kStages = L::kStages;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  uint8_t* smem = smem_raw;
  if ((ptx::smem_u32(smem) & 1023) != 0) __trap();
  float* scratch = reinterpret_cast<float*>(smem + L::kScratchOffset);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + L::kBarOffset);
  uint64_t* empty = full + kStages;
  uint64_t* tmem_full = empty + kStages;
  uint64_t* tmem_empty = tmem_full + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tmem_empty + 2);
  int* unit_slot = reinterpret_cast<int*>(smem + CL::kRingOffset);
  uint64_t* unit_full = reinterpret_cast<uint64_t*>(smem + CL::kRingOffset + kUnitRing * 4);
  uint64_t* unit_empty = unit_full + kUnitRing;

  const int warp = threadIdx.x >> 5;
  const int m_tiles = (prob.M + kBM - 1) / kBM;
  const int n_tiles = (prob.N + BN - 1) / BN;
  const uint32_t rank = kPair ? ptx::cluster_ctarank() : 0u;
  const bool leader = rank == 0;
  const int unit_m = kPair ? m_tiles / 2 : m_tiles;  // m-tile pairs (the host checks evenness)
  const int per_layer = unit_m * prob.groups * n_tiles;
  const int total = per_layer * prob.layers;
  unsigned int* claim = prob.sync;
  unsigned int* ticket = prob.sync + 1;
  unsigned int* done = prob.sync + 2;  // [layer][group][m_tile]
  const unsigned int done_target = static_cast<unsigned int>(n_tiles * L::kEpiWarps);

  if (warp == 0 && ptx::elect_one()) {
    for (int l = 0; l < prob.layers; ++l)
      for (int g = 0; g < prob.groups; ++g) {
        ptx::tma_prefetch(&ops.a[l][g]);
        ptx::tma_prefetch(&ops.b[l][g]);
      }
    for (int s = 0; s < kStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < 2; ++a) {
      ptx::mbar_init(&tmem_full[a], 1);
      ptx::mbar_init(&tmem_empty[a], L::kEpiWarps * (kPair ? 2 : 1));
    }
    for (int r = 0; r < kUnitRing; ++r) {
      ptx::mbar_init(&unit_full[r], 1);
      // the leader's slot is free once every consumer of the unit read it:
      // its MMA warp + epilogue warps (+ the peer's producer + epilogue warps)
      ptx::mbar_init(&unit_empty[r], kPair ? 2 * (1 + L::kEpiWarps) : 1 + L::kEpiWarps);
    }
    ptx::fence_barrier_init();
  }
  if (warp == 1) {
    if constexpr (kPair) ptx::tmem_alloc_pair<L::kTmemCols>(tmem_slot);
    else ptx::tmem_alloc<L::kTmemCols>(tmem_slot);
  }
  ptx::tc_fence_before();
  if constexpr (kPair) ptx::cluster_sync();
  else __syncthreads();
  ptx::tc_fence_after();
  pdl::entry();
  const uint32_t tmem_base = *tmem_slot;

  // unit -> (layer, group, m-tile, n-tile): layer-major, then m, group, n,
  // so a row block's tiles of one layer complete close together
  auto decode = [&](int u, int& l, int& g, int& m, int& t) {
    l = u / per_layer;
    int r = u - l * per_layer;
    m = r / (prob.groups * n_tiles);
    r -= m * prob.groups * n_tiles;
    g = r / n_tiles;
    t = r - g * n_tiles;
    if constexpr (kPair) m = 2 * m + static_cast<int>(rank);  // this CTA's 128-row block
  };
  // a consumer's next unit from the ring (-1: no more work); the slot is
  // released on the leader's barrier
  auto next_unit = [&](uint32_t& j) {
    const int slot = static_cast<int>(j % kUnitRing);
    if constexpr (kPair) ptx::mbar_wait_cluster(&unit_full[slot], (j / kUnitRing) & 1);
    else ptx::mbar_wait(&unit_full[slot], (j / kUnitRing) & 1);
    const int u = *reinterpret_cast<volatile int*>(&unit_slot[slot]);
    // (release at cluster scope: the read of the slot precedes the leader's
    // next remote write to it)
    if constexpr (kPair) ptx::mbar_arrive_cluster_release(ptx::mapa(&unit_empty[slot], 0));
    else ptx::mbar_arrive(&unit_empty[slot]);
    ++j;
    return u;
  };
  // producer: load unit u's operands (this CTA's A rows, its B columns)
  uint32_t it = 0;
  auto load_unit = [&](int u) {
    int l, g, m, t;
    decode(u, l, g, m, t);
    if (l > 0) {
      // rows [128 m, 128 m + 128) of the previous layer's output complete
      const unsigned int* dep = done + (static_cast<int64_t>(l - 1) * prob.groups + g) * m_tiles + m;
      while (ld_acquire_u32(dep) < done_target) __nanosleep(64);
      asm volatile("fence.proxy.async.global;" ::: "memory");
    }
    constexpr int kBCols = kPair ? BN / 2 : BN;
    const int m0 = m * kBM;
    const int n0 = t * BN + static_cast<int>(rank) * kBCols;
    for (int i = 0; i < prob.k_tiles[l]; ++i, ++it) {
      const int s = it % kStages;
      const uint32_t ph = (it / kStages) & 1;
      ptx::mbar_wait(&empty[s], ph ^ 1);
      uint8_t* sa = smem + s * L::kStageBytes;
      uint8_t* sb = sa + L::kABytes;
      const int k0 = i * kBK;
      if constexpr (kPair) {
        // both CTAs' bytes complete on the leader's full barrier
        if (leader) ptx::mbar_arrive_expect_tx(&full[s], 2 * L::kLoadBytes);
        const uint32_t fb = ptx::mapa(&full[s], 0);
        ptx::tma_load_2d_pair(&ops.a[l][g], fb, sa, k0, m0);
#pragma unroll
        for (int q = 0; q < kBCols / 32; ++q)
          ptx::tma_load_2d_pair(&ops.b[l][g], fb, sb + q * (32 * kBK * 4), n0 + 32 * q, k0);
      } else {
        ptx::mbar_arrive_expect_tx(&full[s], L::kLoadBytes);
        ptx::tma_load_2d(&ops.a[l][g], &full[s], sa, k0, m0);
#pragma unroll
        for (int q = 0; q < kBCols / 32; ++q)
          ptx::tma_load_2d(&ops.b[l][g], &full[s], sb + q * (32 * kBK * 4), n0 + 32 * q, k0);
      }
    }
  };

  if (warp == 0) {
    if (ptx::elect_one()) {
      uint32_t j = 0;
      if (leader) {
        while (true) {
          const int u = static_cast<int>(atomicAdd(claim, 1u));
          const int slot = static_cast<int>(j % kUnitRing);
          if constexpr (kPair) ptx::mbar_wait_cluster(&unit_empty[slot], ((j / kUnitRing) & 1) ^ 1);
          else ptx::mbar_wait(&unit_empty[slot], ((j / kUnitRing) & 1) ^ 1);
          const int v = u < total ? u : -1;
          unit_slot[slot] = v;
          if constexpr (kPair) {
            st_cluster_u32(ptx::mapa(&unit_slot[slot], 1), v);
            ptx::mbar_arrive_cluster_release(ptx::mapa(&unit_full[slot], 0));
            ptx::mbar_arrive_cluster_release(ptx::mapa(&unit_full[slot], 1));
          } else {
            ptx::mbar_arrive(&unit_full[slot]);
          }
          ++j;
          if (u >= total) break;
          load_unit(u);
        }
      } else {  // the pair's second CTA: same units, from its ring
        while (true) {
          const int u = next_unit(j);
          if (u < 0) break;
          load_unit(u);
        }
      }
    }
  } else if (warp == 1) {
    constexpr uint32_t idesc = make_idesc<BN, false, true, kPair>();
    if (leader && ptx::elect_one()) {
      uint32_t it = 0, lt = 0, j = 0;
      while (true) {
        const int u = next_unit(j);
        if (u < 0) break;
        int l, g, m, t;
        decode(u, l, g, m, t);
        const uint32_t a = lt & 1;
        ptx::mbar_wait(&tmem_empty[a], ((lt >> 1) & 1) ^ 1);
        ptx::tc_fence_after();
        const uint32_t d_tmem = tmem_base + a * BN;
        for (int i = 0; i < prob.k_tiles[l]; ++i, ++it) {
          const int s = it % kStages;
          ptx::mbar_wait(&full[s], (it / kStages) & 1);
          ptx::tc_fence_after();
          const uint32_t sa = ptx::smem_u32(smem + s * L::kStageBytes);
          const uint32_t sb = sa + L::kABytes;
#pragma unroll
          for (int q = 0; q < kBK / kUmmaK; ++q) {
            const uint64_t ad = operand_desc<false>(sa + q * k_step_bytes<false>());
            const uint64_t bd = operand_desc<true>(sb + q * k_step_bytes<true>());
            if constexpr (kPair) ptx::mma_tf32_pair(d_tmem, ad, bd, idesc, (i > 0 || q > 0) ? 1u : 0u);
            else ptx::mma_tf32(d_tmem, ad, bd, idesc, (i > 0 || q > 0) ? 1u : 0u);
          }
          if constexpr (kPair) ptx::mma_commit_pair(&empty[s]);
          else ptx::mma_commit(&empty[s]);
        }
        if constexpr (kPair) ptx::mma_commit_pair(&tmem_full[a]);
        else ptx::mma_commit(&tmem_full[a]);
        ++lt;
      }
    }
    __syncwarp();
  } else {
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
    uint32_t nstore = 0, lt = 0, j = 0;
    while (true) {
      int u = 0;
      if (lane == 0) u = next_unit(j);
      u = __shfl_sync(0xffffffffu, u, 0);
      j = __shfl_sync(0xffffffffu, j, 0);
      if (u < 0) break;
      int l, g, m, t;
      decode(u, l, g, m, t);
      const Epi& E = epi.e[l];
      ctx.group = g;
      ctx.split = 0;
      ctx.n_tile = t;
      ctx.m_tile = m;
      ctx.row0 = m * kBM + q * 32;
      ctx.m = ctx.row0 + lane;
      const uint32_t a = lt & 1;
      if (lt > 0) ptx::named_bar_sync(1, 32 * L::kEpiWarps);  // previous tile done with scratch
      typename Epi::Row row;
      E.prepare(row, ctx, scratch);
      ptx::named_bar_sync(1, 32 * L::kEpiWarps);
      ptx::mbar_wait(&tmem_full[a], (lt >> 1) & 1);
      ptx::tc_fence_after();
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
        if (c + 1 < c_begin + kChunksPerWarp) ptx::tmem_ld32(t_addr + (c + 1) * 32, r);
        const int n0 = t * BN + c * 32;
        if (E.chunk(row, ctx, n0, v, scratch)) {
          if (lane == 0 && nstore > 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
          __syncwarp();
#pragma unroll
          for (int jj = 0; jj < 8; ++jj) {
            float4* dst = reinterpret_cast<float4*>(stage + lane * 128 + ((jj ^ (lane & 7)) << 4));
            *dst = make_float4(v[4 * jj], v[4 * jj + 1], v[4 * jj + 2], v[4 * jj + 3]);
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&ops.d[l][g], stage, n0, ctx.row0);
            asm volatile("cp.async.bulk.commit_group;" ::: "memory");
          }
          ++nstore;
        }
      }
      ptx::tc_fence_before();
      __syncwarp();
      if (lane == 0) {
        if constexpr (kPair) ptx::mbar_arrive_cluster(ptx::mapa(&tmem_empty[a], 0));
        else ptx::mbar_arrive(&tmem_empty[a]);
      }
      E.end(row, ctx);
      // this warp's rows of the tile are in global memory: count them done
      if (lane == 0) {
        asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
        asm volatile("fence.proxy.async.global;" ::: "memory");
        __threadfence();
        atomicAdd(done + (static_cast<int64_t>(l) * prob.groups + g) * m_tiles + m, 1u);
      }
      __syncwarp();
      ++lt;
    }
  }

  ptx::tc_fence_before();
  if constexpr (kPair) ptx::cluster_sync();  // no remote arrive may target an exited CTA
  else __syncthreads();
  if (warp == 1) {
    ptx::tc_fence_after();
    if constexpr (kPair) ptx::tmem_dealloc_pair<L::kTmemCols>(tmem_base);
    else ptx::tmem_dealloc<L::kTmemCols>(tmem_base);
  }
  // the last CTA out resets the counters for the next launch (graph replay)
  if (threadIdx.x == 0) {
    __threadfence();
    if (atomicAdd(ticket, 1u) == gridDim.x - 1) {
      const int n_done = prob.layers * prob.groups * m_tiles;
      for (int i = 0; i < n_done; ++i) done[i] = 0u;
      *claim = 0u;
      __threadfence();
      *ticket = 0u;
    }
  }
}

}  // namespace pqlg::gemm
