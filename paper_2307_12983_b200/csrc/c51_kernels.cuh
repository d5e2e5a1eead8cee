// Row kernels of the PQL-D categorical critic (proj/include/pql/agents/c51.hpp)
// between the tensor-core GEMMs.  The head GEMMs' C51Head epilogue already
// produced softmax probabilities and expected values per row; these kernels
// finish the losses:
//
//   c51_critic_loss_kernel  c51_critic_loss (c51.hpp:104-156): per row pick
//                           the target head with the lower E (tie -> q1),
//                           c51_project (c51.hpp:62-98: fp64 positions, snap
//                           within 1e-5, float mass split, j ascending), then
//                           the cross-entropy of both online heads and their
//                           upstream (s - proj)/B, plus per-block column sums
//                           of the upstream (the head bias gradient).
//   c51_actor_pick_kernel   c51_actor_loss (c51.hpp:159-205): loss -= min E,
//                           upstream -s_k (z_k - E)/B of the picked head only.
//
// One thread per row (the projection's float accumulation order is the
// reference's); the projected distribution / upstream rows live in shared
// memory as [atom][thread] so a warp's accesses hit distinct banks.
#pragma once

#include <cstdint>

#include "critic_kernels.cuh"
#include "pdl.cuh"

namespace pqlg::c51 {

constexpr int kThreads = 128;
constexpr int kMaxAtoms = 64;
constexpr int kSmemStride = kThreads + 1;
constexpr size_t kLossSmem = 2ull * kMaxAtoms * kSmemStride * sizeof(float);

struct CriticLossArgs {
  const float* pt[2];   // target probs [B x ld]
  const float* evt[2];  // target expected values [B]
  const float* po[2];   // online probs [B x ld]
  int64_t ld;
  const float* ret;
  const float* eff;
  const float* atoms;  // [L]
  double vmin, vmax, dz;
  int L;
  float* up;       // [2][B x ld] dLoss/dlogits
  float* db_part;  // [2][gridDim.x][L] per-block column sums of up
  int64_t* step;   // Adam step, advanced once per update
  double* block_loss;
  unsigned int* counter;
  float* loss_out;
  uint32_t* status;  // bit2: non-finite loss, bit3: projection input not normalized
  int B;
  int Bg;  // mean divisor (global batch when data-parallel)
};

static __global__ void __launch_bounds__(kThreads)
    c51_critic_loss_kernel(const __grid_constant__ CriticLossArgs a) {
  extern __shared__ float sm[];
  float* q1 = sm;                             // [atom][thread]: proj, then up of q1
  float* q2 = sm + kMaxAtoms * kSmemStride;   // up of q2
  pdl::entry();
  const int tid = threadIdx.x;
  const int b = blockIdx.x * kThreads + tid;
  if (b == 0) *a.step += 1;
  const int L = a.L;
  for (int j = 0; j < kMaxAtoms; ++j) {
    q1[j * kSmemStride + tid] = 0.0f;
    q2[j * kSmemStride + tid] = 0.0f;
  }
  double l = 0.0;
  if (b < a.B) {
    // target distribution: the head with the lower expected value (c51.hpp:123-124)
    const int pick = a.evt[0][b] <= a.evt[1][b] ? 0 : 1;
    const float* p = a.pt[pick] + static_cast<int64_t>(b) * a.ld;
    double mass = 0.0;
    for (int j = 0; j < L; ++j) mass = __dadd_rn(mass, static_cast<double>(p[j]));
    if (fabs(mass - 1.0) > 1e-5) atomicOr(a.status, 8u);
    const double g = a.ret[b], e = a.eff[b];
    for (int j = 0; j < L; ++j) {
      double tz = __dadd_rn(g, __dmul_rn(e, static_cast<double>(a.atoms[j])));
      if (tz < a.vmin) tz = a.vmin;
      if (tz > a.vmax) tz = a.vmax;
      double pos = __ddiv_rn(__dsub_rn(tz, a.vmin), a.dz);
      const double snapped = rint(pos);  // std::nearbyint, round-to-nearest-even
      if (fabs(__dsub_rn(pos, snapped)) < 1e-5) pos = snapped;
      const int lo = static_cast<int>(pos);
      const double frac = __dsub_rn(pos, static_cast<double>(lo));
      const float pj = p[j];
      float* ql = q1 + lo * kSmemStride + tid;
      if (frac == 0.0) {
        *ql = __fadd_rn(*ql, pj);
      } else {
        *ql = __fadd_rn(*ql, static_cast<float>(__dmul_rn(pj, __dsub_rn(1.0, frac))));
        ql[kSmemStride] = __fadd_rn(ql[kSmemStride], static_cast<float>(__dmul_rn(pj, frac)));
      }
    }
    // cross-entropy of both online heads against the projection (c51.hpp:138-150)
    const float* s1 = a.po[0] + static_cast<int64_t>(b) * a.ld;
    const float* s2 = a.po[1] + static_cast<int64_t>(b) * a.ld;
    float* u1 = a.up + static_cast<int64_t>(b) * a.ld;
    float* u2 = u1 + static_cast<int64_t>(a.B) * a.ld;
    const float Bf = static_cast<float>(a.Bg);
    float lr = 0.0f;
    for (int j = 0; j < L; ++j) {
      const float pj = q1[j * kSmemStride + tid];
      const float x1 = s1[j], x2 = s2[j];
      if (pj > 0.0f) {
        lr = __fsub_rn(lr, __fmul_rn(pj, logf(x1 > 1e-30f ? x1 : 1e-30f)));
        lr = __fsub_rn(lr, __fmul_rn(pj, logf(x2 > 1e-30f ? x2 : 1e-30f)));
      }
      const float g1 = __fdiv_rn(__fsub_rn(x1, pj), Bf);
      const float g2 = __fdiv_rn(__fsub_rn(x2, pj), Bf);
      u1[j] = g1;
      u2[j] = g2;
      q1[j * kSmemStride + tid] = g1;
      q2[j * kSmemStride + tid] = g2;
    }
    l = static_cast<double>(lr);
  }
  __syncthreads();
  // head bias gradient partials: column sums of the block's upstream rows
  for (int c = tid; c < 2 * L; c += kThreads) {
    const int k = c / L, j = c % L;
    const float* col = (k ? q2 : q1) + j * kSmemStride;
    float s = 0.0f;
    for (int r = 0; r < kThreads; ++r) s = __fadd_rn(s, col[r]);
    a.db_part[(static_cast<int64_t>(k) * gridDim.x + blockIdx.x) * L + j] = s;
  }
  critic::block_mean_finish<kThreads>(l, a.block_loss, a.counter, a.Bg, a.loss_out, a.status,
                                      4u);
}

struct ActorPickArgs {
  const float* po[2];   // online probs [B x ld] at (s, pi(s))
  const float* ev[2];   // expected values [B]
  int64_t ld;
  const float* atoms;
  int L;
  float* up;  // [2][B x ld]
  int64_t* step;
  double* block_loss;
  unsigned int* counter;
  float* loss_out;
  uint32_t* status;
  int B, Bg;
};

static __global__ void __launch_bounds__(kThreads)
    c51_actor_pick_kernel(const __grid_constant__ ActorPickArgs a) {
  pdl::entry();
  const int b = blockIdx.x * kThreads + threadIdx.x;
  if (b == 0) *a.step += 1;
  double l = 0.0;
  if (b < a.B) {
    const float e1 = a.ev[0][b], e2 = a.ev[1][b];
    const bool pick1 = e1 <= e2;
    l = -static_cast<double>(pick1 ? e1 : e2);
    const int k = pick1 ? 0 : 1;
    const float e = pick1 ? e1 : e2;
    const float* s = a.po[k] + static_cast<int64_t>(b) * a.ld;
    float* upk = a.up + (static_cast<int64_t>(k) * a.B + b) * a.ld;
    float* upo = a.up + (static_cast<int64_t>(1 - k) * a.B + b) * a.ld;
    const float Bf = static_cast<float>(a.Bg);
    for (int j = 0; j < a.L; ++j) {
      // -s_j * (z_j - E) / B  (c51.hpp:192-197)
      upk[j] = __fdiv_rn(__fmul_rn(-s[j], __fsub_rn(a.atoms[j], e)), Bf);
      upo[j] = 0.0f;
    }
  }
  critic::block_mean_finish<kThreads>(l, a.block_loss, a.counter, a.Bg, a.loss_out, a.status,
                                      4u);
}

}  // namespace pqlg::c51
