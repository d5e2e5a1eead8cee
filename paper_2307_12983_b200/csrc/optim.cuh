// Gradient finalisation and the fused clip + Adam + Polyak optimizer.
//
//   finalize: fixed-order sums of split-K / per-tile partials into the flat
//             Mlp-layout gradient, fp64 sum of squares per block, and (last
//             block) the clip scale of fa::clip_global_norm (optim.hpp:54-69)
//   adam:     g *= s (scalar.hpp:88-91), Adam (scalar.hpp:69-80) with the
//             fp64 bias corrections of optim.hpp:35-39 from a host table, then
//             soft_update (scalar.hpp:82-86) -- one pass, bit-exact per element
//             (explicit __fmul_rn/__fadd_rn: no FMA contraction, matching the
//             reference's -ffp-contract=off).
// All are HBM-bound streaming kernels (grid = multiple of 148 SMs x 4).
#pragma once

#include "pdl.cuh"
#include <cstdint>

namespace pqlg::optim {

constexpr int kMaxSegments = 16;
constexpr int kFinalizeThreads = 256;

// dst[i] = sum_{t < n_terms} src[t*stride + i]  for i < count  (t ascending)
struct Segment {
  int64_t dst;
  int64_t count;
  const float* src;
  int64_t group_stride;  // src advance per group
  int n_terms;
  int64_t stride;
  int64_t cols = 0;      // > 0: src rows are padded, src = (j / cols) * ld_src + j % cols
  int64_t ld_src = 0;
};

struct FinalizeArgs {
  Segment seg[kMaxSegments];
  int n_seg;
  int64_t total;    // elements per group (== params)
  int64_t gstride;  // group stride of grads (16-byte aligned groups)
  float* grads;     // [groups x gstride]
  double* block_sq;         // [groups x gridDim.x]
  unsigned int* counter;    // [groups], self-resetting
  float* scale;             // [groups] clip scale (1 if not clipped)
  uint32_t* status;         // bit0: non-finite gradient norm
  float max_norm;
};

// __grid_constant__: the segment table is indexed dynamically; without it
// every thread would copy the whole argument block to local memory.
static __global__ void __launch_bounds__(kFinalizeThreads)
    finalize_kernel(const __grid_constant__ FinalizeArgs a) {
  pdl::entry();
  const int group = blockIdx.y;
  double sq = 0.0;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.total;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    int s = 0;
    while (s + 1 < a.n_seg && i >= a.seg[s + 1].dst) ++s;
    const Segment& sg = a.seg[s];
    const int64_t j = i - sg.dst;
    const int64_t js = sg.cols > 0 ? (j / sg.cols) * sg.ld_src + j % sg.cols : j;
    const float* src = sg.src + group * sg.group_stride + js;
    // terms summed in ascending order; loads issued 8 at a time so the
    // latency of the (L2-resident) partials overlaps
    float acc = src[0];
    int t = 1;
    for (; t + 8 <= sg.n_terms; t += 8) {
      float v[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) v[u] = src[(t + u) * sg.stride];
#pragma unroll
      for (int u = 0; u < 8; ++u) acc = __fadd_rn(acc, v[u]);
    }
    for (; t < sg.n_terms; ++t) acc = __fadd_rn(acc, src[t * sg.stride]);
    a.grads[group * a.gstride + i] = acc;
    const double d = static_cast<double>(acc);
    sq += d * d;
  }
  // block reduction in fixed order (fp64)
  __shared__ double red[kFinalizeThreads / 32];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) sq += __shfl_down_sync(0xffffffffu, sq, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = sq;
  __syncthreads();
  __shared__ bool last;
  if (threadIdx.x == 0) {
    double b = 0.0;
    for (int w = 0; w < kFinalizeThreads / 32; ++w) b += red[w];
    a.block_sq[group * gridDim.x + blockIdx.x] = b;
    __threadfence();
    const unsigned prev = atomicAdd(&a.counter[group], 1u);
    last = prev == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  // Last block: fixed-order tree over the block partials (all threads load,
  // so the L2 latency is paid once, not gridDim.x times).
  __threadfence();
  const volatile double* bs = a.block_sq + group * gridDim.x;
  double part = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += blockDim.x) part += bs[b];
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) part += __shfl_down_sync(0xffffffffu, part, d);
  __syncthreads();
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = part;
  __syncthreads();
  if (threadIdx.x != 0) return;
  double tot = 0.0;
  for (int w = 0; w < kFinalizeThreads / 32; ++w) tot += red[w];
  a.counter[group] = 0;
  const double norm = sqrt(tot);
  float s = 1.0f;
  if (!isfinite(norm)) {
    atomicOr(a.status, 1u);
    s = __int_as_float(0x7fc00000);
  } else if (norm > static_cast<double>(a.max_norm)) {
    s = static_cast<float>(static_cast<double>(a.max_norm) / norm * (1.0 - 1e-6));
  }
  a.scale[group] = s;
}

struct AdamArgs {
  float* p;        // [groups x n]
  const float* g;  // [groups x n]
  float* m;
  float* v;
  float* target;   // nullable: Polyak target [groups x n]
  int64_t n;
  int64_t gstride;      // group stride of p/g/m/v/target
  const float* scale;   // [groups], clip scale
  const uint32_t* status;
  const int64_t* step;  // device Adam step t (already incremented for this update)
  const float2* bc;     // bias-correction table, index t (clamped)
  int64_t bc_len;
  float lr, beta1, beta2, eps, tau;
};

static __global__ void adam_polyak_kernel(AdamArgs a) {
  pdl::entry();
  // A non-finite target / loss / gradient makes the reference throw before
  // adam_step modifies anything (ddpg.hpp:37,72; optim.hpp:33-34).
  if (*a.status) return;
  const int group = blockIdx.y;
  int64_t t = *a.step;
  if (t >= a.bc_len) t = a.bc_len - 1;
  const float2 bc = a.bc[t];
  const float s = a.scale[group];
  const bool clipped = s != 1.0f;
  const float ob1 = __fsub_rn(1.0f, a.beta1), ob2 = __fsub_rn(1.0f, a.beta2);
  const float keep = __fsub_rn(1.0f, a.tau);
  const int64_t off = group * a.gstride;
  for (int64_t i = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.n;
       i += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    float gi = a.g[off + i];
    if (clipped) gi = __fmul_rn(gi, s);
    float m = __fadd_rn(__fmul_rn(a.beta1, a.m[off + i]), __fmul_rn(ob1, gi));
    float v = __fadd_rn(__fmul_rn(a.beta2, a.v[off + i]), __fmul_rn(ob2, __fmul_rn(gi, gi)));
    a.m[off + i] = m;
    a.v[off + i] = v;
    const float mhat = __fmul_rn(m, bc.x);
    const float vhat = __fmul_rn(v, bc.y);
    const float upd = __fmul_rn(a.lr, __fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), a.eps)));
    const float p = __fsub_rn(a.p[off + i], upd);
    a.p[off + i] = p;
    if (a.target)
      a.target[off + i] = __fadd_rn(__fmul_rn(a.tau, p), __fmul_rn(keep, a.target[off + i]));
  }
}

}  // namespace pqlg::optim
