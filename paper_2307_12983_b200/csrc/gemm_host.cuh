// Host-side helpers for the tcgen05 GEMM: tensor maps per operand role and a
// launcher that sizes the grid (m tiles x n tiles x splits*groups).
#pragma once

#include <cstdio>
#include <cstdlib>

#include "common.h"
#include "gemm_tf32.cuh"

namespace pqlg::gemm {

// GEMM precision of the closures built on this thread: the cores' constructors
// set it from pqlg_config::precision for the duration of their plan building.
//   TF32   operand maps typed TFLOAT32 (TMA rounds to nearest), one MMA per K step
//   3xTF32 operand maps FLOAT32, hi/lo split in shared memory, three MMAs per K
//          step (fp32-faithful parity mode; gemm_tf32.cuh)
inline thread_local bool t_build_x3 = false;
struct PrecisionScope {
  bool prev;
  explicit PrecisionScope(bool x3) : prev(t_build_x3) { t_build_x3 = x3; }
  ~PrecisionScope() { t_build_x3 = prev; }
  PrecisionScope(const PrecisionScope&) = delete;
  PrecisionScope& operator=(const PrecisionScope&) = delete;
};
inline bool build_x3() { return t_build_x3; }
// Operand maps of the current build precision (TFLOAT32 unless 3xTF32).
inline bool tf32_maps() { return !t_build_x3; }

// A operand. mn = false: A is [M x K] row-major (stride lda >= K).
//            mn = true:  A is stored [K x M] row-major (stride lda >= M).
inline CUtensorMap map_a(const float* A, int M, int K, int lda, bool mn, bool tf32 = false) {
  if (mn) return make_tmap_2d(A, M, K, lda, 32, kBK, Swz::k128a32, tf32);
  return make_tmap_2d(A, K, M, lda, kBK, kBM, Swz::k128, tf32);
}

// B operand. mn = false: B is [N x K] row-major; mn = true: B is [K x N].
inline CUtensorMap map_b(const float* B, int N, int K, int ldb, bool mn, int BN,
                         bool tf32 = false) {
  if (mn) return make_tmap_2d(B, N, K, ldb, 32, kBK, Swz::k128a32, tf32);
  return make_tmap_2d(B, K, N, ldb, kBK, BN, Swz::k128, tf32);
}

inline Problem make_problem(int M, int N, int K, int splits) {
  require(M > 0 && N > 0 && K > 0, "gemm: empty problem");
  Problem p{};
  p.M = M;
  p.N = N;
  p.K = K;
  p.k_tiles = (K + kBK - 1) / kBK;
  if (splits < 1) splits = 1;
  if (splits > p.k_tiles) splits = p.k_tiles;
  p.k_tiles_per_split = (p.k_tiles + splits - 1) / splits;
  p.splits = (p.k_tiles + p.k_tiles_per_split - 1) / p.k_tiles_per_split;  // none empty
  p.groups = 1;
  return p;
}

inline int sm_count() {
  static int n = [] {
    int dev = 0, c = 0;
    PQLG_CUDA(cudaGetDevice(&dev));
    PQLG_CUDA(cudaDeviceGetAttribute(&c, cudaDevAttrMultiProcessorCount, dev));
    return c;
  }();
  return n;
}

// CTA pairs (cta_group::2) for wide tiles when the m-tiles pair up evenly;
// PQLG_PAIR=0 keeps one CTA per tile (A/B switch).
inline bool pair_enabled() {
  static const bool on = [] {
    const char* e = std::getenv("PQLG_PAIR");
    return !(e && e[0] == '0');
  }();
  return on;
}
template <int BN>
inline bool use_pair(int M) {
  return BN >= 128 && ((M + kBM - 1) / kBM) % 2 == 0 && pair_enabled();
}
// Box of a K-major B operand: a pair's CTA stages half of the BN columns.
template <int BN>
inline int b_box(int M) {
  return use_pair<BN>(M) ? BN / 2 : BN;
}

template <int BN, bool kAMN, bool kBMN, class Epi, bool kPair, bool k3x>
void launch_impl(const Operands& ops, Problem p, int groups, const Epi& epi, cudaStream_t st) {
  using L = SmemLayout<BN, Epi, kPair, k3x>;
  auto kern = gemm_tf32_kernel<BN, kAMN, kBMN, Epi, kPair, k3x>;
  static bool configured = false;
  if (!configured) {
    PQLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   L::kDynamic));
    if (kPair)
      PQLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 0));
    configured = true;
  }
  p.groups = groups;
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.N + BN - 1) / BN) * p.splits * groups;
  int grid = tiles < sm_count() ? tiles : sm_count();
  if (kPair) grid &= ~1;  // whole clusters of 2 (tiles are even here)
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(grid);
  cfg.blockDim = dim3(L::kThreads);
  cfg.dynamicSmemBytes = L::kDynamic;
  cfg.stream = st;
  cudaLaunchAttribute attr[2];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = pdl_enabled() ? 1 : 0;
  int na = 1;
  if (kPair) {
    attr[1].id = cudaLaunchAttributeClusterDimension;
    attr[1].val.clusterDim.x = 2;
    attr[1].val.clusterDim.y = 1;
    attr[1].val.clusterDim.z = 1;
    na = 2;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  const bool prof = profiling_active();
  if (prof) {
    char shape[96];
    std::snprintf(shape, sizeof(shape), "groups=%d M=%d N=%d K=%d splits=%d%s%s", groups, p.M,
                  p.N, p.K, p.splits, kPair ? " pair" : "", k3x ? " 3xtf32" : "");
    profile_before(st, reinterpret_cast<const void*>(kern), shape);
  }
  PQLG_CUDA(cudaLaunchKernelEx(&cfg, kern, ops, p, epi));
  count_launch();
  if (prof) profile_after(st);
}

// Persistent launch: min(tiles, SMs) CTAs, one per SM, walking the tiles
// (or, for CTA pairs, clusters of 2 walking m-tile pairs).  x3: the 3xTF32
// variant (the operand maps must then be FLOAT32-typed).
template <int BN, bool kAMN, bool kBMN, class Epi>
void launch(const Operands& ops, Problem p, int groups, const Epi& epi, cudaStream_t st,
            bool x3 = false) {
  if (x3) {
    if constexpr (BN >= 128) {
      if (use_pair<BN>(p.M))
        return launch_impl<BN, kAMN, kBMN, Epi, true, true>(ops, p, groups, epi, st);
    }
    return launch_impl<BN, kAMN, kBMN, Epi, false, true>(ops, p, groups, epi, st);
  }
  if constexpr (BN >= 128) {
    if (use_pair<BN>(p.M))
      return launch_impl<BN, kAMN, kBMN, Epi, true, false>(ops, p, groups, epi, st);
  }
  launch_impl<BN, kAMN, kBMN, Epi, false, false>(ops, p, groups, epi, st);
}

}  // namespace pqlg::gemm
