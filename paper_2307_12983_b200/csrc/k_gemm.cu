// Operator-level GEMM entry points (pqlg_k_gemm_tf32*): the affine kernels of
// pql::kernels (kernels.hpp:25-43) restated as one tcgen05 TF32 GEMM with the
// learners' epilogue path (bias + ReLU, TMA store, split-K partials + a
// fixed-order reduction).  Used by the per-op parity tests and the bench's
// roofline measurement.
#include <cstring>

#include "pdl.cuh"
#include "epilogues.cuh"
#include "gemm_host.cuh"

namespace pqlg {
namespace {

__global__ void reduce_splits(const float* W, int splits, int M, int N, float* D, int ldd,
                              const float* bias, int relu) {
  pdl::entry();
  const size_t total = static_cast<size_t>(M) * N;
  for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < total;
       i += static_cast<size_t>(gridDim.x) * blockDim.x) {
    float acc = W[i];
    for (int s = 1; s < splits; ++s) acc = __fadd_rn(acc, W[s * total + i]);
    const int m = static_cast<int>(i / N), n = static_cast<int>(i % N);
    if (bias) acc = __fadd_rn(acc, bias[n]);
    if (relu) acc = acc > 0.0f ? acc : 0.0f;
    D[static_cast<size_t>(m) * ldd + n] = acc;
  }
}

template <int BN, bool AMN, bool BMN>
void run(const float* A, const float* B, float* D, const float* bias, int M, int N, int K,
         int lda, int ldb, int ldd, int relu, int splits, int round_mode, cudaStream_t st) {
  const bool tf32 = round_mode == 1;
  const bool x3 = round_mode == 2;
  gemm::Operands ops;
  ops.a[0] = ops.a[1] = gemm::map_a(A, M, K, lda, AMN, tf32);
  ops.b[0] = ops.b[1] = gemm::map_b(B, N, K, ldb, BMN, BMN ? BN : gemm::b_box<BN>(M), tf32);
  gemm::Problem p = gemm::make_problem(M, N, K, splits);
  if (p.splits == 1) {
    ops.d[0] = ops.d[1] = make_store_map(D, M, N, ldd);
    gemm::launch<BN, AMN, BMN>(ops, p, 1, epi::Linear{bias, relu, BN, N}, st, x3);
    return;
  }
  require(N % 4 == 0, "split-K partials need N % 4 == 0");
  float* W = nullptr;
  PQLG_CUDA(cudaMallocAsync(&W, sizeof(float) * p.splits * M * N, st));
  ops.d[0] = ops.d[1] = make_tmap_3d(W, N, M, p.splits, N, static_cast<uint64_t>(M) * N, 32, 32,
                                     Swz::k128);
  gemm::launch<BN, AMN, BMN>(ops, p, 1, epi::Partial{}, st, x3);
  launch(reduce_splits, dim3(296), dim3(256), 0, st, W, p.splits, M, N, D, ldd, bias, relu);
  PQLG_CUDA(cudaFreeAsync(W, st));
}

// Back-to-back launches of the hidden-layer forward GEMM with the learners'
// Hidden epilogue (bias + ReLU + bitmask + TMA store) and pre-encoded maps.
template <int BN>
void run_repeat(const float* A, const float* B, float* D, const float* bias, int M, int N, int K,
                int lda, int ldb, int ldd, int relu, int iters, cudaStream_t st) {
  gemm::Operands ops;
  ops.a[0] = ops.a[1] = gemm::map_a(A, M, K, lda, false, true);
  ops.b[0] = ops.b[1] = gemm::map_b(B, N, K, ldb, true, BN, true);
  ops.d[0] = ops.d[1] = make_store_map(D, M, N, ldd);
  const gemm::Problem p = gemm::make_problem(M, N, K, 1);
  const epi::Linear e{bias, relu, BN, N};
  for (int i = 0; i < iters; ++i) gemm::launch<BN, false, true>(ops, p, 1, e, st);
}

// The update's dominant launch: `groups` independent hidden layers in one
// persistent launch (the twin target + twin online critics, 4 groups).  Group
// g reads its own A + g*M*lda, W = B + g*K*ldb, bias + g*N and writes its own
// D + g*M*ldd, as the four critics of an update do (distinct operands, so
// the timing sees the in-update DRAM/L2 traffic, not one L2-resident set).
void run_repeat_groups(const float* A, const float* B, float* D, const float* bias, int M, int N,
                       int K, int lda, int ldb, int ldd, int groups, int iters, cudaStream_t st) {
  require(groups >= 1 && groups <= gemm::kMaxGroups, "repeat_groups: 1..4 groups");
  require(N > 128, "repeat_groups: hidden-layer widths (N > 128)");
  gemm::Operands ops;
  std::memset(&ops, 0, sizeof(ops));
  epi::Hidden e{};
  for (int g = 0; g < groups; ++g) {
    ops.a[g] = gemm::map_a(A + static_cast<size_t>(g) * M * lda, M, K, lda, false, true);
    ops.b[g] = gemm::map_b(B + static_cast<size_t>(g) * K * ldb, N, K, ldb, true, 256, true);
    ops.d[g] = make_store_map(D + static_cast<size_t>(g) * M * ldd, M, N, ldd);
    e.bias[g] = bias + static_cast<size_t>(g) * N;
  }
  const gemm::Problem p = gemm::make_problem(M, N, K, 1);
  e.bn = 256;
  e.M = M;
  e.N = N;
  e.store = 0xF;
  for (int i = 0; i < iters; ++i) gemm::launch<256, false, true>(ops, p, groups, e, st);
}

template <int BN>
void dispatch_major(int a_mn, int b_mn, const float* A, const float* B, float* D,
                    const float* bias, int M, int N, int K, int lda, int ldb, int ldd, int relu,
                    int splits, int tf32, cudaStream_t st) {
  if (!a_mn && !b_mn) run<BN, false, false>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
  else if (!a_mn && b_mn) run<BN, false, true>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
  else if (a_mn && !b_mn) run<BN, true, false>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
  else run<BN, true, true>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
}

}  // namespace
}  // namespace pqlg

extern "C" int pqlg_k_gemm_tf32_repeat(const float* A, const float* B, float* D,
                                       const float* bias, int M, int N, int K, int lda, int ldb,
                                       int ldd, int relu, int iters, void* stream) {
  return pqlg::guarded([&] {
    auto st = static_cast<cudaStream_t>(stream);
    if (N > 128) pqlg::run_repeat<256>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, iters, st);
    else if (N > 64) pqlg::run_repeat<128>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, iters, st);
    else if (N > 32) pqlg::run_repeat<64>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, iters, st);
    else pqlg::run_repeat<32>(A, B, D, bias, M, N, K, lda, ldb, ldd, relu, iters, st);
  });
}

extern "C" int pqlg_k_gemm_tf32_repeat_groups(const float* A, const float* B, float* D,
                                              const float* bias, int M, int N, int K, int lda,
                                              int ldb, int ldd, int groups, int iters,
                                              void* stream) {
  return pqlg::guarded([&] {
    pqlg::run_repeat_groups(A, B, D, bias, M, N, K, lda, ldb, ldd, groups, iters,
                            static_cast<cudaStream_t>(stream));
  });
}

extern "C" int pqlg_k_gemm_tf32(const float* A, const float* B, float* D, const float* bias, int M,
                                int N, int K, int a_mn, int b_mn, int lda, int ldb, int ldd,
                                int relu, int splits, int round_mode, void* stream) {
  return pqlg::guarded([&] {
    pqlg::require(M > 0 && N > 0 && K > 0, "gemm: empty shape");
    auto st = static_cast<cudaStream_t>(stream);
    pqlg::require(round_mode >= 0 && round_mode <= 2, "gemm: round_mode 0, 1 or 2");
    const int tf32 = round_mode;
    if (N > 128)
      pqlg::dispatch_major<256>(a_mn, b_mn, A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
    else if (N > 64)
      pqlg::dispatch_major<128>(a_mn, b_mn, A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
    else if (N > 32)
      pqlg::dispatch_major<64>(a_mn, b_mn, A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
    else
      pqlg::dispatch_major<32>(a_mn, b_mn, A, B, D, bias, M, N, K, lda, ldb, ldd, relu, splits, tf32, st);
  });
}
