// Host-side builders for the MLP GEMMs of the learners: every GEMM of an
// update is turned into a closure with its tensor maps pre-encoded at handle
// construction, so an update is a fixed list of launches (CUDA-graph ready).
//
//   fwd    out = A * W        A = activations [M x K] (K-major),
//                             W = [K x N] row-major (fa::Mlp layout, N-major)
//   dgrad  din = G * W^T      G = [M x N_out] (K-major), W = [N_in x N_out] (K-major)
//   wgrad  dW = H^T * G       H = [K=B x M=in] (M-major), G = [B x N] (N-major)
#pragma once

#include <algorithm>

#include <cmath>
#include <cstring>
#include <functional>
#include <type_traits>
#include <vector>

#include "epilogues.cuh"
#include "gemm_host.cuh"
#include "head_kernels.cuh"

namespace pqlg::mlp {

using Step = std::function<void(cudaStream_t)>;

inline int bn_for(int N) { return N > 128 ? 256 : N > 64 ? 128 : N > 32 ? 64 : 32; }
inline int n_tiles(int N) { return (N + bn_for(N) - 1) / bn_for(N); }
// Head-dot partial slots of a Hidden epilogue over N columns: one per
// min(64, bn)-column block (epi::Hidden).
inline int hidden_slots(int N) {
  const int unit = bn_for(N) < 64 ? bn_for(N) : 64;
  return (N + unit - 1) / unit;
}
constexpr int kSMs = 148;

// Small launches: when twice the 128-row x 256-column tiles (all groups)
// still fit in one wave on the SMs, 128-column tiles fill twice as many of
// them (c2 actor step 41.1 -> 36.9 us, c1 25.8 -> 22.6 us).  At B = 8192 the
// doubled count would need a second wave (c3 critic +1.5 us, 3xTF32 +35 us
// measured), so 256 stays: c2 / c3 learners are unchanged.  Applies to the
// epilogues whose tile width is a run-time field (`bn`).  PQLG_BN_FILL=0
// disables (A/B knob, read once).
inline bool bn_fill() {
  static const bool on = [] {
    const char* e = std::getenv("PQLG_BN_FILL");
    return !(e && e[0] == '0');
  }();
  return on;
}
inline int fill_bn(int M, int N, int groups) {
  const int bn = bn_for(N);
  if (bn == 256 && bn_fill() && 2 * ((M + 127) / 128) * ((N + 255) / 256) * groups <= kSMs)
    return 128;
  return bn;
}
template <class E, class = void>
struct has_bn : std::false_type {};
template <class E>
struct has_bn<E, std::void_t<decltype(std::declval<E&>().bn)>> : std::true_type {};
// The tile width of a launch over [M x N] x groups; sets epi.bn to match.
template <class Epi>
int pick_bn(int M, int N, int groups, Epi& epi) {
  if constexpr (has_bn<Epi>::value) {
    epi.bn = fill_bn(M, N, groups);
    return epi.bn;
  }
  return bn_for(N);
}

template <class F>
void with_bn_value(int bn, F&& f) {
  switch (bn) {
    case 256: f(std::integral_constant<int, 256>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    default: f(std::integral_constant<int, 32>{}); break;
  }
}
template <class F>
void with_bn(int N, F&& f) {
  switch (bn_for(N)) {
    case 256: f(std::integral_constant<int, 256>{}); break;
    case 128: f(std::integral_constant<int, 128>{}); break;
    case 64: f(std::integral_constant<int, 64>{}); break;
    default: f(std::integral_constant<int, 32>{}); break;
  }
}

// Split factor so that (tiles * splits) roughly fills the 148 SMs once.
inline int wgrad_splits(int M, int N, int K, int groups) {
  const int tiles = ((M + 127) / 128) * n_tiles(N) * groups;
  const int k_tiles = (K + gemm::kBK - 1) / gemm::kBK;
  int s = kSMs / tiles;
  if (s < 1) s = 1;
  if (s > k_tiles) s = k_tiles;
  const int per = (k_tiles + s - 1) / s;  // effective count after even chunking
  return (k_tiles + per - 1) / per;
}

// ldw: row stride of W (N unless W is read from a padded WeightMirror).
// Output maps: D0/D1 [M x N] with row stride ldd (null: the epilogue stores
// directly and no map is built).
inline void set_out(gemm::Operands& ops, const float* D0, const float* D1, int M, int N,
                    int64_t ldd, int groups) {
  std::memset(&ops.d, 0, sizeof(ops.d));
  if (!D0) return;
  ops.d[0] = make_store_map(D0, M, N, ldd);
  ops.d[1] = groups > 1 ? make_store_map(D1, M, N, ldd) : ops.d[0];
}

template <class Epi>
Step fwd(const float* A0, const float* A1, int64_t lda, const float* W0, const float* W1, int M,
         int N, int K, int groups, Epi epi, int64_t ldw = 0, const float* D0 = nullptr,
         const float* D1 = nullptr, int64_t ldd = 0) {
  Step step;
  if (ldw == 0) ldw = N;
  if (ldd == 0) ldd = N;
  with_bn_value(pick_bn(M, N, groups, epi), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    gemm::Operands ops;
    ops.a[0] = gemm::map_a(A0, M, K, lda, false, gemm::tf32_maps());
    ops.a[1] = groups > 1 ? gemm::map_a(A1, M, K, lda, false, gemm::tf32_maps()) : ops.a[0];
    ops.b[0] = gemm::map_b(W0, N, K, ldw, true, BN, gemm::tf32_maps());
    ops.b[1] = groups > 1 ? gemm::map_b(W1, N, K, ldw, true, BN, gemm::tf32_maps()) : ops.b[0];
    set_out(ops, D0, D1, M, N, ldd, groups);
    const gemm::Problem p = gemm::make_problem(M, N, K, 1);
    const bool x3 = gemm::build_x3();
    step = [ops, p, groups, epi, x3](cudaStream_t st) {
      gemm::launch<BN, false, true>(ops, p, groups, epi, st, x3);
    };
  });
  return step;
}

// Forward layer over `groups` (<= gemm::kMaxGroups) independent nets sharing
// one launch: A[g] [M x K] (stride lda), W[g] [K x N] (stride ldw), outputs
// D[g] [M x N] (stride ldd; null: the epilogue stores nothing / itself).
template <class Epi>
Step fwd_groups(const float* const* A, int64_t lda, const float* const* W, int M, int N, int K,
                int groups, Epi epi, int64_t ldw, const float* const* D, int64_t ldd) {
  require(groups >= 1 && groups <= gemm::kMaxGroups, "fwd_groups: 1..4 groups");
  Step step;
  if (ldw == 0) ldw = N;
  if (ldd == 0) ldd = N;
  with_bn_value(pick_bn(M, N, groups, epi), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    gemm::Operands ops;
    std::memset(&ops, 0, sizeof(ops));
    for (int g = 0; g < groups; ++g) {
      ops.a[g] = gemm::map_a(A[g], M, K, lda, false, gemm::tf32_maps());
      ops.b[g] = gemm::map_b(W[g], N, K, ldw, true, BN, gemm::tf32_maps());
      if (D && D[g]) ops.d[g] = make_store_map(D[g], M, N, ldd);
    }
    const gemm::Problem p = gemm::make_problem(M, N, K, 1);
    const bool x3 = gemm::build_x3();
    step = [ops, p, groups, epi, x3](cudaStream_t st) {
      gemm::launch<BN, false, true>(ops, p, groups, epi, st, x3);
    };
  });
  return step;
}

// din[M x N_in] = G[M x N_out] * W^T, W = [N_in x N_out] row-major (ld = ldw).
template <class Epi>
Step dgrad(const float* G0, const float* G1, int64_t ldg, const float* W0, const float* W1,
           int64_t ldw, int M, int N_in, int N_out, int groups, Epi epi,
           const float* D0 = nullptr, const float* D1 = nullptr, int64_t ldd = 0) {
  if (ldd == 0) ldd = N_in;
  Step step;
  with_bn_value(pick_bn(M, N_in, groups, epi), [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    gemm::Operands ops;
    ops.a[0] = gemm::map_a(G0, M, N_out, ldg, false, gemm::tf32_maps());
    ops.a[1] = groups > 1 ? gemm::map_a(G1, M, N_out, ldg, false, gemm::tf32_maps()) : ops.a[0];
    const int box = gemm::b_box<BN>(M);  // K-major B: a CTA pair splits the columns
    ops.b[0] = gemm::map_b(W0, N_in, N_out, ldw, false, box, gemm::tf32_maps());
    ops.b[1] = groups > 1 ? gemm::map_b(W1, N_in, N_out, ldw, false, box, gemm::tf32_maps()) : ops.b[0];
    set_out(ops, D0, D1, M, N_in, ldd, groups);
    const gemm::Problem p = gemm::make_problem(M, N_in, N_out, 1);
    const bool x3 = gemm::build_x3();
    step = [ops, p, groups, epi, x3](cudaStream_t st) {
      gemm::launch<BN, false, false>(ops, p, groups, epi, st, x3);
    };
  });
  return step;
}

// dW[M=in x N=out] = H^T G over K = batch rows; split-K partial tiles are
// TMA-stored to W[(group*splits + split)][M][N] (N % 4 == 0).
template <class Epi>
Step wgrad(const float* H0, const float* H1, int64_t ldh, const float* G0, const float* G1,
           int64_t ldg, int M, int N, int K, int groups, int splits, Epi epi, float* W,
           int64_t ldw_part = 0) {
  if (ldw_part == 0) ldw_part = N;
  Step step;
  with_bn(N, [&](auto bn) {
    constexpr int BN = decltype(bn)::value;
    gemm::Operands ops;
    ops.a[0] = gemm::map_a(H0, M, K, ldh, true, gemm::tf32_maps());
    ops.a[1] = groups > 1 ? gemm::map_a(H1, M, K, ldh, true, gemm::tf32_maps()) : ops.a[0];
    ops.b[0] = gemm::map_b(G0, N, K, ldg, true, BN, gemm::tf32_maps());
    ops.b[1] = groups > 1 ? gemm::map_b(G1, N, K, ldg, true, BN, gemm::tf32_maps()) : ops.b[0];
    const gemm::Problem p = gemm::make_problem(M, N, K, splits);
    require(p.splits == splits, "wgrad: split count must divide the k tiles evenly");
    ops.d[0] = ops.d[1] = make_tmap_3d(W, N, M, static_cast<uint64_t>(groups) * splits,
                                       ldw_part, static_cast<uint64_t>(M) * ldw_part, 32, 32,
                                       Swz::k128);
    const bool x3 = gemm::build_x3();
    step = [ops, p, groups, epi, x3](cudaStream_t st) {
      gemm::launch<BN, true, true>(ops, p, groups, epi, st, x3);
    };
  });
  return step;
}

// Narrow policy head H -> A (A <= 32) as split-K partial tiles + the
// finishing kernel (head_kernels.cuh).  `fin` carries everything but the
// partial buffer, which is allocated here; returns the two steps.
struct HeadSplit {
  DevBuf<float> part;
  int splits = 1;
  int64_t ld_part = 0;
  void plan(int M, int A, int K) {
    const int tiles = (M + gemm::kBM - 1) / gemm::kBM;
    const int k_tiles = (K + gemm::kBK - 1) / gemm::kBK;
    int s = (2 * kSMs + tiles - 1) / tiles;
    const int max_s = k_tiles / 4 > 1 ? k_tiles / 4 : 1;  // >= 4 k-tiles per split
    if (s > max_s) s = max_s;
    splits = gemm::make_problem(M, A, K, s).splits;
    ld_part = (A + 3) / 4 * 4;
    part.alloc(static_cast<size_t>(splits) * M * ld_part);
  }
};

// The head GEMM: split-K partial tiles into hs.part (plans hs).  N <= 32
// (act_dim) or <= 64 (the SAC head's [mean | log_std]).
inline Step head_gemm_step(HeadSplit& hs, const float* A0, int64_t lda, const float* W,
                           int64_t ldw, int M, int N, int K) {
  require(N <= 64, "policy head: at most 64 head outputs");
  hs.plan(M, N, K);
  gemm::Operands ops;
  std::memset(&ops, 0, sizeof(ops));
  ops.a[0] = gemm::map_a(A0, M, K, lda, false, gemm::tf32_maps());
  const int bn = N <= 32 ? 32 : 64;
  ops.b[0] = gemm::map_b(W, N, K, ldw, true, bn, gemm::tf32_maps());
  ops.d[0] = make_tmap_3d(hs.part.p, N, M, hs.splits, hs.ld_part,
                          static_cast<uint64_t>(M) * hs.ld_part, 32, 32, Swz::k128);
  const gemm::Problem p = gemm::make_problem(M, N, K, hs.splits);
  const bool x3 = gemm::build_x3();
  if (bn == 32)
    return [ops, p, x3](cudaStream_t st) {
      gemm::launch<32, false, true>(ops, p, 1, epi::Partial{}, st, x3);
    };
  return [ops, p, x3](cudaStream_t st) {
    gemm::launch<64, false, true>(ops, p, 1, epi::Partial{}, st, x3);
  };
}

// The finish (bias, squash, noise, stores) of a planned head.
inline Step head_finish_step(const HeadSplit& hs, head::FinishArgs fin, int M, int N) {
  fin.part = hs.part.p;
  fin.S = hs.splits;
  fin.ld_part = hs.ld_part;
  fin.M = M;
  fin.A = N;
  const int rows_blocks = (M + head::kFinishWarps - 1) / head::kFinishWarps;
  const int blocks = rows_blocks < 4 * kSMs ? rows_blocks : 4 * kSMs;
  return [fin, blocks](cudaStream_t st) {
    launch(head::policy_head_finish_kernel, dim3(blocks), dim3(32 * head::kFinishWarps), 0, st,
           fin);
  };
}

// The narrow head (head::head_mma_kernel): one launch computes x * W and,
// in squash mode, the finish.  `r` carries the mode and output fields;
// x/w/M/K/N are set here.
template <int kNT, bool k3x, int kMT>
inline void launch_head_mt(const head::RowsArgs& r, cudaStream_t st) {
  auto kern = head::head_mma_kernel<kNT, k3x, kMT>;
  const size_t smem = head::head_smem<kNT, k3x, kMT>(r.K);
  static bool configured = false;
  if (!configured) {
    PQLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
    configured = true;
  }
  const int fin = r.fin.partial ? r.fin.nblk : 0;
  // finish blocks reuse the dynamic shared memory for their [16][32] double2
  const size_t smem_all = fin ? std::max<size_t>(smem, actor::kNormFinishWarps * 32 * 16) : smem;
  constexpr int rows = head::head_rows<kMT>();
  launch(kern, dim3((r.M + rows - 1) / rows + fin), dim3(32 * head::kHeadWarps), smem_all, st, r);
}
template <int kNT, bool k3x>
inline void launch_head(const head::RowsArgs& r, cudaStream_t st) {
  if (head::head_mt(r.M) == 4) launch_head_mt<kNT, k3x, 4>(r, st);
  else launch_head_mt<kNT, k3x, 2>(r, st);
}

template <int kNT>
inline void pick_head(bool x3, void (*&fn)(const head::RowsArgs&, cudaStream_t)) {
  fn = x3 ? launch_head<kNT, true> : launch_head<kNT, false>;
}

inline Step head_rows_step(head::RowsArgs r, const float* x, int64_t ldx, const float* W, int M,
                           int N, int K) {
  require(N >= 1 && N <= 8 * head::kHeadMaxNT, "policy head: at most 72 head outputs");
  require(K % 4 == 0 && ldx % 4 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0,
          "policy head: activation rows must be 16-byte aligned");
  r.x = x;
  r.ldx = ldx;
  r.w = W;
  if (r.ldw == 0) r.ldw = N;
  r.M = M;
  r.K = K;
  r.N = N;
  const bool x3 = gemm::build_x3();
  const int nt = (N + 7) / 8;
  void (*fn)(const head::RowsArgs&, cudaStream_t) = nullptr;
  switch (nt) {
    case 1: pick_head<1>(x3, fn); break;
    case 2: pick_head<2>(x3, fn); break;
    case 3: pick_head<3>(x3, fn); break;
    case 4: pick_head<4>(x3, fn); break;
    case 5: pick_head<5>(x3, fn); break;
    case 6: pick_head<6>(x3, fn); break;
    case 7: pick_head<7>(x3, fn); break;
    case 8: pick_head<8>(x3, fn); break;
    default: pick_head<9>(x3, fn); break;
  }
  require(head::head_smem<9, false, 4>(K) <= 200 * 1024 || nt < 9,
          "policy head: hidden width too large for the head kernel");
  return [r, fn](cudaStream_t st) { fn(r, st); };
}

// Packs W [K x ldw] (columns [0, N)) into the head kernel's fragment order
// (RowsArgs::wpack; head_pack_elems float4).
inline int64_t head_pack_elems(int N, int K) {
  return static_cast<int64_t>((K + 15) / 16) * ((N + 7) / 8) * 32;
}
template <int kNT>
inline void launch_head_pack(const float* W, int64_t ldw, int K, int N, float4* out, bool x3,
                             cudaStream_t st) {
  const int n = static_cast<int>(head_pack_elems(N, K));
  if (x3) launch(head::head_pack_kernel<kNT, true>, dim3((n + 255) / 256), dim3(256), 0, st, W, ldw, K, N, out);
  else launch(head::head_pack_kernel<kNT, false>, dim3((n + 255) / 256), dim3(256), 0, st, W, ldw, K, N, out);
}
inline void head_pack(const float* W, int64_t ldw, int K, int N, float4* out, bool x3,
                      cudaStream_t st) {
  switch ((N + 7) / 8) {
    case 1: launch_head_pack<1>(W, ldw, K, N, out, x3, st); break;
    case 2: launch_head_pack<2>(W, ldw, K, N, out, x3, st); break;
    case 3: launch_head_pack<3>(W, ldw, K, N, out, x3, st); break;
    case 4: launch_head_pack<4>(W, ldw, K, N, out, x3, st); break;
    case 5: launch_head_pack<5>(W, ldw, K, N, out, x3, st); break;
    case 6: launch_head_pack<6>(W, ldw, K, N, out, x3, st); break;
    case 7: launch_head_pack<7>(W, ldw, K, N, out, x3, st); break;
    case 8: launch_head_pack<8>(W, ldw, K, N, out, x3, st); break;
    default: launch_head_pack<9>(W, ldw, K, N, out, x3, st); break;
  }
}

// Raw head sums into hs.part (one "split", row stride round_up(N, 4)) for a
// finish kernel that adds the bias itself (the SAC Gaussian finish).
// `base` may carry wpack / fin (the actor's packed weights and normalizer finish).
inline Step head_raw_step(HeadSplit& hs, const float* x, int64_t ldx, const float* W, int M,
                          int N, int K, const head::RowsArgs& base = head::RowsArgs{}) {
  hs.splits = 1;
  hs.ld_part = (N + 3) / 4 * 4;
  hs.part.alloc(static_cast<size_t>(M) * hs.ld_part);
  head::RowsArgs r = base;
  r.mode = 0;
  r.out = hs.part.p;
  r.ld_out = hs.ld_part;
  return head_rows_step(r, x, ldx, W, M, N, K);
}

// DeterministicPolicy::act in one launch: act = mid + half*tanh(x W + b),
// optional tanh_out and (actor) mixed exploration noise + clamp.
inline Step head_squash_step(head::RowsArgs r, const float* x, int64_t ldx, const float* W, int M,
                             int N, int K) {
  r.mode = 1;
  return head_rows_step(r, x, ldx, W, M, N, K);
}

// Bias-correction table bc[t] = (float(1/(1-0.9^t)), float(1/(1-0.999^t)))
// computed on the host with the same libm pow the reference uses
// (optim.hpp:35-39).  Beyond t = 32767 both are exactly 1.0f.
inline std::vector<float2> adam_bias_table(double beta1, double beta2, int len = 32768) {
  std::vector<float2> t(len);
  t[0] = make_float2(1.0f, 1.0f);
  for (int i = 1; i < len; ++i) {
    const double b1t = std::pow(beta1, static_cast<double>(i));
    const double b2t = std::pow(beta2, static_cast<double>(i));
    t[i] = make_float2(static_cast<float>(1.0 / (1.0 - b1t)), static_cast<float>(1.0 / (1.0 - b2t)));
  }
  return t;
}

}  // namespace pqlg::mlp
