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
  // filled by plan_finalize
  int64_t blk0 = 0;      // first block of this segment
  int mode = 0;          // 0: thread per element, 1: float4 per thread, 2: warp per element
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
  int skip_norm;            // 1: reduction only (a data-parallel all-reduce follows)
  const float* check;       // nullable: a scalar (the all-reduced loss) whose
                            // non-finiteness sets status bit 2
};

// Host: give every segment its own block range (no per-element segment
// search) and pick the float4 path where the layout allows; returns the
// number of blocks per group.
inline int plan_finalize(FinalizeArgs& f) {
  int64_t blocks = 0;
  for (int i = 0; i < f.n_seg; ++i) {
    Segment& sg = f.seg[i];
    const bool v = sg.cols == 0 && sg.count % 4 == 0 && sg.dst % 4 == 0 && sg.stride % 4 == 0 &&
                   sg.group_stride % 4 == 0 && f.gstride % 4 == 0 &&
                   (reinterpret_cast<uintptr_t>(sg.src) & 15) == 0 &&
                   (reinterpret_cast<uintptr_t>(f.grads) & 15) == 0;
    // long sums (per-row-tile bias partials: 64-128 terms) get a warp each so
    // the kernel's critical path is not one thread's chain of dependent loads
    // (a warp per element only pays for short segments: on a weight segment
    // its strided reads waste 28 of every 32 bytes fetched)
    sg.mode = (sg.n_terms > 16 && sg.count <= 4096) ? 2 : (v ? 1 : 0);
    sg.blk0 = blocks;
    const int64_t per_block = sg.mode == 2 ? kFinalizeThreads / 32
                                           : static_cast<int64_t>(kFinalizeThreads) * (v ? 4 : 1);
    blocks += (sg.count + per_block - 1) / per_block;
  }
  return static_cast<int>(blocks);
}

// __grid_constant__: the segment table is indexed dynamically; without it
// every thread would copy the whole argument block to local memory.
static __global__ void __launch_bounds__(kFinalizeThreads)
    finalize_kernel(const __grid_constant__ FinalizeArgs a) {
  pdl::entry();
  const int group = blockIdx.y;
  int si = 0;
  while (si + 1 < a.n_seg && static_cast<int64_t>(blockIdx.x) >= a.seg[si + 1].blk0) ++si;
  const Segment& sg = a.seg[si];
  const int64_t lb = static_cast<int64_t>(blockIdx.x) - sg.blk0;
  double sq = 0.0;
  // terms summed in ascending order, 8 loads in flight
  if (sg.mode == 2) {
    // lane l sums terms l, l+32, ... in order; lanes combine by a fixed xor tree
    const int lane = threadIdx.x & 31;
    const int64_t j = lb * (blockDim.x / 32) + (threadIdx.x >> 5);
    if (j < sg.count) {
      const int64_t js = sg.cols > 0 ? (j / sg.cols) * sg.ld_src + j % sg.cols : j;
      const float* src = sg.src + group * sg.group_stride + js;
      float acc = 0.0f;
      for (int t0 = lane; t0 < sg.n_terms; t0 += 128) {
        float v[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int t = t0 + 32 * u;
          v[u] = t < sg.n_terms ? src[t * sg.stride] : 0.0f;
        }
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (t0 + 32 * u < sg.n_terms) acc = __fadd_rn(acc, v[u]);
      }
#pragma unroll
      for (int o = 16; o >= 1; o >>= 1) acc = __fadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, o));
      if (lane == 0) {
        a.grads[group * a.gstride + sg.dst + j] = acc;
        const double d = static_cast<double>(acc);
        sq = d * d;
      }
    }
  } else if (sg.mode == 1) {
    const int64_t j = (lb * blockDim.x + threadIdx.x) * 4;
    if (j < sg.count) {
      const float* src = sg.src + group * sg.group_stride + j;
      float4 acc = *reinterpret_cast<const float4*>(src);
      int t = 1;
      for (; t < sg.n_terms; t += 8) {
        float4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t + u < sg.n_terms) v[u] = *reinterpret_cast<const float4*>(src + (t + u) * sg.stride);
#pragma unroll
        for (int u = 0; u < 8; ++u) {
          if (t + u < sg.n_terms) {
            acc.x = __fadd_rn(acc.x, v[u].x);
            acc.y = __fadd_rn(acc.y, v[u].y);
            acc.z = __fadd_rn(acc.z, v[u].z);
            acc.w = __fadd_rn(acc.w, v[u].w);
          }
        }
      }
      *reinterpret_cast<float4*>(a.grads + group * a.gstride + sg.dst + j) = acc;
      const double d0 = acc.x, d1 = acc.y, d2 = acc.z, d3 = acc.w;
      sq = ((d0 * d0 + d1 * d1) + d2 * d2) + d3 * d3;
    }
  } else {
    const int64_t j = lb * blockDim.x + threadIdx.x;
    if (j < sg.count) {
      const int64_t js = sg.cols > 0 ? (j / sg.cols) * sg.ld_src + j % sg.cols : j;
      const float* src = sg.src + group * sg.group_stride + js;
      float acc = src[0];
      for (int t = 1; t < sg.n_terms; t += 8) {
        float v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t + u < sg.n_terms) v[u] = src[(t + u) * sg.stride];
#pragma unroll
        for (int u = 0; u < 8; ++u)
          if (t + u < sg.n_terms) acc = __fadd_rn(acc, v[u]);
      }
      a.grads[group * a.gstride + sg.dst + j] = acc;
      const double d = static_cast<double>(acc);
      sq = d * d;
    }
  }
  if (a.skip_norm) return;
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
  if (a.check && !isfinite(*a.check)) atomicOr(a.status, 4u);
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

// pql_sac: sac_alpha_loss + adam_step on log alpha (sac.hpp:117-125,
// learners.cpp:254-256), done by one thread of the policy's Adam launch.
struct AlphaStep {
  float* log_alpha;        // null: no alpha update
  float* m;
  float* v;
  const float* mean_logp;  // this update's mean log-prob (detached)
  float target_entropy;    // -act_dim (learners.cpp:217)
  float lr;                // lr_actor
};

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
  AlphaStep alpha;
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
  if (a.alpha.log_alpha && blockIdx.x == 0 && group == 0 && threadIdx.x == 0) {
    const float drift = __fadd_rn(*a.alpha.mean_logp, a.alpha.target_entropy);
    const float gi = -drift;  // dloss/dlog_alpha
    const float mo = __fadd_rn(__fmul_rn(a.beta1, *a.alpha.m), __fmul_rn(ob1, gi));
    const float vo = __fadd_rn(__fmul_rn(a.beta2, *a.alpha.v), __fmul_rn(ob2, __fmul_rn(gi, gi)));
    const float upd = __fmul_rn(
        a.alpha.lr, __fdiv_rn(__fmul_rn(mo, bc.x), __fadd_rn(__fsqrt_rn(__fmul_rn(vo, bc.y)), a.eps)));
    *a.alpha.m = mo;
    *a.alpha.v = vo;
    *a.alpha.log_alpha = __fsub_rn(*a.alpha.log_alpha, upd);
  }
  const int64_t off = group * a.gstride;
  float* __restrict__ P = a.p + off;
  const float* __restrict__ G = a.g + off;
  float* __restrict__ M = a.m + off;
  float* __restrict__ V = a.v + off;
  float* __restrict__ T = a.target ? a.target + off : nullptr;
  auto step = [&](float p, float gi, float m, float v, float tg, float& po, float& mo, float& vo,
                  float& to) {
    if (clipped) gi = __fmul_rn(gi, s);
    mo = __fadd_rn(__fmul_rn(a.beta1, m), __fmul_rn(ob1, gi));
    vo = __fadd_rn(__fmul_rn(a.beta2, v), __fmul_rn(ob2, __fmul_rn(gi, gi)));
    const float mhat = __fmul_rn(mo, bc.x);
    const float vhat = __fmul_rn(vo, bc.y);
    const float upd = __fmul_rn(a.lr, __fdiv_rn(mhat, __fadd_rn(__fsqrt_rn(vhat), a.eps)));
    po = __fsub_rn(p, upd);
    to = __fadd_rn(__fmul_rn(a.tau, po), __fmul_rn(keep, tg));
  };
  // float4 body (group bases are 16-byte aligned), scalar tail
  const int64_t n4 = a.n / 4;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t q = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; q < n4;
       q += stride) {
    const float4 p4 = reinterpret_cast<const float4*>(P)[q];
    const float4 g4 = reinterpret_cast<const float4*>(G)[q];
    const float4 m4 = reinterpret_cast<const float4*>(M)[q];
    const float4 v4 = reinterpret_cast<const float4*>(V)[q];
    const float4 t4 = T ? reinterpret_cast<const float4*>(T)[q] : make_float4(0, 0, 0, 0);
    float4 po, mo, vo, to;
    step(p4.x, g4.x, m4.x, v4.x, t4.x, po.x, mo.x, vo.x, to.x);
    step(p4.y, g4.y, m4.y, v4.y, t4.y, po.y, mo.y, vo.y, to.y);
    step(p4.z, g4.z, m4.z, v4.z, t4.z, po.z, mo.z, vo.z, to.z);
    step(p4.w, g4.w, m4.w, v4.w, t4.w, po.w, mo.w, vo.w, to.w);
    reinterpret_cast<float4*>(P)[q] = po;
    reinterpret_cast<float4*>(M)[q] = mo;
    reinterpret_cast<float4*>(V)[q] = vo;
    if (T) reinterpret_cast<float4*>(T)[q] = to;
  }
  for (int64_t i = 4 * n4 + blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; i < a.n;
       i += stride) {
    float po, mo, vo, to;
    step(P[i], G[i], M[i], V[i], T ? T[i] : 0.0f, po, mo, vo, to);
    P[i] = po;
    M[i] = mo;
    V[i] = vo;
    if (T) T[i] = to;
  }
}

}  // namespace pqlg::optim
