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
#pragma once

#include <cstdint>

#include "critic_kernels.cuh"
#include "pdl.cuh"

namespace pqlg::c51 {

constexpr int kThreads = 128;    // actor-pick kernel: one thread per row
constexpr int kMaxAtoms = 64;
constexpr int kLossWarps = 8;    // critic-loss kernel: one warp per row
constexpr int kLossBlocks = 296; // 2 x 148 SMs; warps stride over the rows

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
  float* db_part;  // [2][kLossBlocks * kLossWarps][L] per-warp column sums of up
  int64_t* step;   // Adam step, advanced once per update
  double* block_loss;
  unsigned int* counter;
  float* loss_out;
  uint32_t* status;  // bit2: non-finite loss, bit3: projection input not normalized
  int B;
  int Bg;  // mean divisor (global batch when data-parallel)
};

// One warp per row, lane j owning atoms j and j + 32.  The projection's
// float accumulation into each atom keeps the reference's order, source
// atoms j ascending (c51.hpp:79-95): every lane first computes its sources'
// (lo, mass-to-lo, mass-to-lo+1); since Tz_j = G + eff*z_j is nondecreasing
// in j (eff >= 0), lo_j is sorted, so the sources of target atom i are one
// contiguous run -- those with lo_j == i-1 (split mass) followed by those
// with lo_j == i -- found by binary search and folded left to right.
static __global__ void __launch_bounds__(kLossWarps * 32)
    c51_critic_loss_kernel(const __grid_constant__ CriticLossArgs a) {
  __shared__ int s_lo[kLossWarps][kMaxAtoms];
  __shared__ float s_cl[kLossWarps][kMaxAtoms];
  __shared__ float s_ch[kLossWarps][kMaxAtoms];
  pdl::entry();
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  const int warp = blockIdx.x * kLossWarps + wib;
  const int n_warps = gridDim.x * kLossWarps;
  if (blockIdx.x == 0 && threadIdx.x == 0) *a.step += 1;
  const int L = a.L;
  const float Bf = static_cast<float>(a.Bg);
  int* lo_s = s_lo[wib];
  float* cl_s = s_cl[wib];
  float* ch_s = s_ch[wib];
  float db[2][2] = {{0.0f, 0.0f}, {0.0f, 0.0f}};  // [critic][atom lane / lane+32]
  double l = 0.0;
  for (int b = warp; b < a.B; b += n_warps) {
    const int pick = a.evt[0][b] <= a.evt[1][b] ? 0 : 1;  // c51.hpp:123-124
    const float* p = a.pt[pick] + static_cast<int64_t>(b) * a.ld;
    const double g = a.ret[b], e = a.eff[b];
    double mass = 0.0;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int j = lane + 32 * h;
      float cl = 0.0f, ch = 0.0f;
      int lo = 1 << 20;  // beyond every target (j >= L)
      if (j < L) {
        const float pj = p[j];
        mass += static_cast<double>(pj);
        double tz = __dadd_rn(g, __dmul_rn(e, static_cast<double>(a.atoms[j])));
        if (tz < a.vmin) tz = a.vmin;
        if (tz > a.vmax) tz = a.vmax;
        double pos = __ddiv_rn(__dsub_rn(tz, a.vmin), a.dz);
        const double snapped = rint(pos);  // std::nearbyint (round-half-even)
        if (fabs(__dsub_rn(pos, snapped)) < 1e-5) pos = snapped;
        lo = static_cast<int>(pos);
        const double frac = __dsub_rn(pos, static_cast<double>(lo));
        if (frac == 0.0) {
          cl = pj;  // whole mass to lo, nothing to lo + 1
        } else {
          cl = static_cast<float>(__dmul_rn(pj, __dsub_rn(1.0, frac)));
          ch = static_cast<float>(__dmul_rn(pj, frac));
        }
      }
      lo_s[j] = lo;
      cl_s[j] = cl;
      ch_s[j] = ch;
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) mass += __shfl_xor_sync(0xffffffffu, mass, o);
    if (lane == 0 && fabs(mass - 1.0) > 1e-5) atomicOr(a.status, 8u);
    __syncwarp();
    const float* s1 = a.po[0] + static_cast<int64_t>(b) * a.ld;
    const float* s2 = a.po[1] + static_cast<int64_t>(b) * a.ld;
    float* u1 = a.up + static_cast<int64_t>(b) * a.ld;
    float* u2 = u1 + static_cast<int64_t>(a.B) * a.ld;
    float lr = 0.0f;
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i < L) {
        // first source with lo >= i - 1, then fold while lo <= i
        int lo_idx = 0, hi_idx = L;
        while (lo_idx < hi_idx) {
          const int mid = (lo_idx + hi_idx) >> 1;
          if (lo_s[mid] < i - 1) lo_idx = mid + 1;
          else hi_idx = mid;
        }
        float q = 0.0f;
        for (int j = lo_idx; j < L; ++j) {
          const int lj = lo_s[j];
          if (lj > i) break;
          q = __fadd_rn(q, lj == i ? cl_s[j] : ch_s[j]);  // lj == i-1: the split remainder
        }
        // cross-entropy of both online heads (c51.hpp:138-150)
        const float x1 = s1[i], x2 = s2[i];
        if (q > 0.0f) {
          lr = __fsub_rn(lr, __fmul_rn(q, logf(x1 > 1e-30f ? x1 : 1e-30f)));
          lr = __fsub_rn(lr, __fmul_rn(q, logf(x2 > 1e-30f ? x2 : 1e-30f)));
        }
        const float g1 = __fdiv_rn(__fsub_rn(x1, q), Bf);
        const float g2 = __fdiv_rn(__fsub_rn(x2, q), Bf);
        u1[i] = g1;
        u2[i] = g2;
        db[0][h] = __fadd_rn(db[0][h], g1);
        db[1][h] = __fadd_rn(db[1][h], g2);
      }
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) lr += __shfl_xor_sync(0xffffffffu, lr, o);
    if (lane == 0) l += static_cast<double>(lr);
    __syncwarp();
  }
  // head bias gradient partials: this warp's column sums (rows in its order)
#pragma unroll
  for (int k = 0; k < 2; ++k)
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int i = lane + 32 * h;
      if (i < L) a.db_part[(static_cast<int64_t>(k) * n_warps + warp) * L + i] = db[k][h];
    }
  critic::block_mean_finish<kLossWarps * 32>(l, a.block_loss, a.counter, a.Bg, a.loss_out,
                                             a.status, 4u);
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
