// Host-side helpers for the tcgen05 GEMM: tensor maps per operand role and a
// launcher that sizes the grid (m tiles x n tiles x splits*groups).
#pragma once

#include "common.h"
#include "gemm_tf32.cuh"

namespace pqlg::gemm {

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

// Persistent launch: min(tiles, SMs) CTAs, one per SM, walking the tiles.
template <int BN, bool kAMN, bool kBMN, class Epi>
void launch(const Operands& ops, Problem p, int groups, const Epi& epi, cudaStream_t st) {
  using L = SmemLayout<BN, Epi>;
  auto kern = gemm_tf32_kernel<BN, kAMN, kBMN, Epi>;
  static bool configured = false;
  if (!configured) {
    PQLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                   L::kDynamic));
    configured = true;
  }
  p.groups = groups;
  const int tiles = ((p.M + kBM - 1) / kBM) * ((p.N + BN - 1) / BN) * p.splits * groups;
  const int grid = tiles < sm_count() ? tiles : sm_count();
  ::pqlg::launch(kern, dim3(grid), dim3(L::kThreads), L::kDynamic, st, ops, p, epi);
}

}  // namespace pqlg::gemm
