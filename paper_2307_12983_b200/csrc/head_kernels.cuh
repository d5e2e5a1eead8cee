// The learners' narrow policy head (H -> act_dim, DeterministicPolicy::act,
// policy.hpp:33-38) as split-K GEMM partials + one finishing kernel.  With
// only M/128 row tiles of 32 columns the head GEMM alone would stream its
// [M x H] input through a fraction of the SMs; split over K it uses all of
// them, and the finish sums the splits in fixed order, adds the bias and
// squashes.
#pragma once

#include <cstdint>

#include "pdl.cuh"

namespace pqlg::head {

constexpr int kFinishWarps = 8;

struct FinishArgs {
  const float* part;     // [S][M][ld_part] head-GEMM partial sums
  int S;
  int64_t ld_part;
  const float* bias;     // [A]
  float* act;            // [M x ld_act]
  int64_t ld_act;
  float* tanh_out;       // nullable [M x ld_tanh] (policy backward)
  int64_t ld_tanh;
  int M, A;
  float mid, half;
};

// Warp per row (grid-stride), lane = action column: y = sum_s part[s]
// (s ascending) + b, a = mid + half*tanh(y); coalesced loads and stores.
// (The actor's head, which also draws exploration noise, keeps the fused
// GEMM epilogue: its per-row draws overlap the mainloop there.)
static __global__ void __launch_bounds__(32 * kFinishWarps)
    policy_head_finish_kernel(const __grid_constant__ FinishArgs a) {
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warps = gridDim.x * kFinishWarps;
  const int64_t split_stride = static_cast<int64_t>(a.M) * a.ld_part;
  if (lane >= a.A) return;
  const float bc = a.bias[lane];
  for (int m = blockIdx.x * kFinishWarps + w; m < a.M; m += warps) {
    const float* p = a.part + static_cast<int64_t>(m) * a.ld_part + lane;
    float acc = p[0];
    for (int s = 1; s < a.S; ++s) acc = __fadd_rn(acc, p[s * split_stride]);
    const float y = __fadd_rn(acc, bc);
    const float th = tanhf(y);
    if (a.tanh_out) a.tanh_out[static_cast<int64_t>(m) * a.ld_tanh + lane] = th;
    a.act[static_cast<int64_t>(m) * a.ld_act + lane] = __fadd_rn(a.mid, __fmul_rn(a.half, th));
  }
}

}  // namespace pqlg::head
