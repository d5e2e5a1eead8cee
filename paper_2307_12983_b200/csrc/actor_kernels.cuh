// Actor-side kernels: the synthetic vectorised environment, observation
// normalisation, the running-normalizer update and (for the op-level hook)
// standalone mixed exploration noise.
//
//   env step       EnvBatch::step contract (vecenv.cpp:84-106) with the
//                  synthetic task of SURVEY 8(d); float mul/add only, in the
//                  d-ascending order, so states/rewards are bit-exact
//   normalize      RunningNormalizer::apply_stats (normalizer.hpp:56-70)
//   norm update    RunningNormalizer::update + merge (normalizer.hpp:33-50,
//                  :73-83): Welford per 128-row chunk (row order), chunks
//                  merged with Chan's formula in fixed tree order, fp64
//   noise          explore::apply_noise (noise.hpp:56-72), bit-exact
#pragma once

#include "pdl.cuh"
#include <cstdint>
#include <vector>

#include "ptx.cuh"
#include "norm_finish.cuh"
#include "rng.cuh"
#include "common.h"

namespace pqlg::actor {

constexpr int kEnvWarps = 8;
constexpr int kEnvPer = 4;                         // envs per warp per tile
constexpr int kEnvTile = kEnvWarps * kEnvPer;      // 32 envs per block iteration
constexpr int kMaxA = 32;
constexpr int kMaxD = 256;                         // 64 float4 quads: two per lane

struct EnvState {
  float* s;                // [N x ld] state (= observation); null: the caller keeps the
  int64_t ld;              //   state in its obs buffers (s_in = this step's obs)
  const float* s_in;       // state read by the step (= s unless aliased); rows 16-byte
  int64_t ld_in;           //   aligned, ld_in % 4 == 0
  const float* M;          // [D x A] coupling
  const float4* MT;        // [round_up(A, 4)][kMaxD / 4] M^T, zero padded (env_transpose_M)
  int64_t* episode_step;   // [N]
  uint64_t* rng;           // [N] SplitMix state per env
  int N, D, A;
  int max_len;
  float low, high;
  float one = 1.0f;        // a runtime 1.0f (see add2 below)
};

struct StepOut {
  float* next_obs;   // [N x ld_obs] (auto-reset rows hold the fresh observation)
  float* boot;       // [N x ld_obs] next obs, or the terminal observation on done
  float* rew;        // [N]
  uint8_t* term;     // [N] done && !truncated
  uint8_t* trunc;    // [N]
  uint8_t* done;     // [N] (nullable)
  int64_t ld_obs;
  uint32_t* status;  // bit3: non-finite action
};

// Optional fused observation normalisation of the next observation (the
// actor's next policy input): the running stats are updated from this
// step's observations before the env step, exactly the stats the reference
// applies at the next rollout_step (learners.cpp:89, :113).
struct NextNorm {
  float* out;         // [N x ld_out] (null: not fused)
  int64_t ld_out;
  const float* mean;  // fp32 apply constants
  const float* inv;
  const int* identity;
};

// ---- paired fp32 arithmetic (sm_100 FMUL2 / FFMA2), rounding like the scalar ops.
// ptxas contracts a paired mul feeding a paired add into one FFMA2 (even
// with explicit .rn), which would skip the product's rounding.  The sum is
// therefore formed as fma(p, one, acc) with `one` a kernel argument equal to
// 1.0f: p * 1 is exact, so the result is round(p + acc), the reference's
// separately rounded add, and there is no multiply left to contract.
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(uint64_t r, float& a, float& b) {
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r));
}
__device__ __forceinline__ uint64_t mul2(uint64_t a, uint64_t b) {
  uint64_t r;
  asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
  return r;
}
__device__ __forceinline__ uint64_t add2(uint64_t p, uint64_t acc, uint64_t one2) {
  uint64_t r;
  asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(r) : "l"(p), "l"(one2), "l"(acc));
  return r;
}

__device__ __forceinline__ float clamp10(float v) {
  return v < -10.0f ? -10.0f : (v > 10.0f ? 10.0f : v);
}

// Synthetic EnvBatch::step (vecenv.cpp:84-106 contract, SURVEY 8(d) task).
// A warp owns kEnvPer envs of a 32-env block tile; lane l owns observation
// quads l and l + 32 (d = 4q..4q+3), so rows move as float4.
//   1  s' = clamp(0.95 s + 0.05 M a): M^T (pre-transposed at env creation)
//      copied into shared memory; for every k the lane's quad of M^T[k] (one
//      LDS.128) feeds kEnvPer envs with paired mul / add (k ascending, no
//      FMA: bit-exact; the k >= A padding adds +0 products, which leave the
//      +0-started sums unchanged)
//   2  done flags from s'_0 and the episode counter (prefetched with the
//      state), boot / next obs (fresh reset draws on done) / next-obs
//      normalisation stored by the owning warp straight away
//   3  the order-sensitive d-ascending sum of s'^2 (the reward) runs one
//      thread per env over the block's 32 rows in shared memory (double
//      buffered: one warp per tile, while the others start the next tile)
template <int kSlots>
static __global__ void __launch_bounds__(32 * kEnvWarps)
    env_step_kernel(EnvState e, const float* __restrict__ act, int64_t ld_act, StepOut o,
                    NextNorm nn) {
  extern __shared__ float4 sh4[];
  constexpr int kQT = 32 * kSlots;                       // M^T row stride (float4)
  const int D = e.D, A = e.A, Q = (D + 3) >> 2;
  const int Ap = (A + 3) & ~3;
  const int ldv = D | 1;                                 // odd: conflict-free chain reads
  float4* sMT = sh4;                                     // [Ap][kQT]
  float* sv = reinterpret_cast<float*>(sMT + Ap * kQT);  // [2][kEnvTile][ldv]   s'
  float* sa = sv + 2 * kEnvTile * ldv;                   // [kEnvTile][32]       clamped a
  float* saa = sa + kEnvTile * 32;                       // [2][kEnvTile]        sum a^2
  int* sflag = reinterpret_cast<int*>(saa + 2 * kEnvTile);  // [2][kEnvTile] done | trunc<<1
  // M^T (constant since env creation) before the PDL wait
  for (int idx = threadIdx.x; idx < Ap * kQT; idx += blockDim.x) {
    const int k = idx / kQT, q = idx - k * kQT;
    sMT[idx] = __ldg(e.MT + k * (kMaxD / 4) + q);
  }
  __syncthreads();
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint64_t one2 = pk(e.one, e.one);
  const uint64_t c095 = pk(0.95f, 0.95f), c005 = pk(0.05f, 0.05f);
  const bool id = nn.out ? (*nn.identity != 0) : true;
  const bool xnorm = nn.out != nullptr && !id;
  const bool vec = ((o.ld_obs & 3) == 0) &&
                   ((reinterpret_cast<uintptr_t>(o.next_obs) | reinterpret_cast<uintptr_t>(o.boot)) & 15) == 0 &&
                   (!nn.out || (((nn.ld_out & 3) == 0) && (reinterpret_cast<uintptr_t>(nn.out) & 15) == 0)) &&
                   (!e.s || (((e.ld & 3) == 0) && (reinterpret_cast<uintptr_t>(e.s) & 15) == 0));
  // this lane's normalisation constants
  float nm[kSlots][4], ni[kSlots][4];
#pragma unroll
  for (int sl = 0; sl < kSlots; ++sl)
#pragma unroll
    for (int c = 0; c < 4; ++c) {
      const int d = 4 * (lane + 32 * sl) + c;
      nm[sl][c] = (xnorm && d < D) ? nn.mean[d] : 0.0f;
      ni[sl][c] = (xnorm && d < D) ? nn.inv[d] : 1.0f;
    }
  const int n_tiles = (e.N + kEnvTile - 1) / kEnvTile;
  float* sa_w = sa + w * kEnvPer * 32;
  int it = 0;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++it) {
    const int buf = it & 1;
    const int i0 = tile * kEnvTile;
    const int base = i0 + w * kEnvPer;
    const int nv = e.N - base;  // valid envs of this warp (may be <= 0)
    // ---- loads: state quads, actions and episode counters of the warp's envs
    float4 s4[kEnvPer][kSlots];
#pragma unroll
    for (int p = 0; p < kEnvPer; ++p) {
      const float* srow = e.s_in + static_cast<int64_t>(base + p) * e.ld_in;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int q = lane + 32 * sl;
        s4[p][sl] = (p < nv && q < Q) ? __ldg(reinterpret_cast<const float4*>(srow) + q)
                                      : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float up[kEnvPer];
#pragma unroll
    for (int p = 0; p < kEnvPer; ++p)
      up[p] = (lane < A && p < nv) ? __ldg(act + static_cast<int64_t>(base + p) * ld_act + lane) : 0.0f;
    const int64_t ep_prev = (lane < kEnvPer && lane < nv) ? e.episode_step[base + lane] : 0;
    {
      bool bad = false;
#pragma unroll
      for (int p = 0; p < kEnvPer; ++p) {
        float u = up[p];
        if (lane < A && p < nv) {
          bad |= !isfinite(u);
          u = u < e.low ? e.low : (u > e.high ? e.high : u);
        }
        sa_w[p * 32 + lane] = u;
      }
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(o.status, 8u);
    }
    __syncwarp();
    if (lane < kEnvPer) {  // sum a^2, k ascending
      const float* ap = sa_w + lane * 32;
      float aa = 0.0f;
      for (int k = 0; k < A; ++k) aa = __fadd_rn(aa, __fmul_rn(ap[k], ap[k]));
      saa[buf * kEnvTile + w * kEnvPer + lane] = aa;
    }
    // ---- 1: M a, k ascending (sums start at +0 like the reference's loop)
    uint64_t acc[kEnvPer][kSlots][2];
#pragma unroll
    for (int p = 0; p < kEnvPer; ++p)
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) acc[p][sl][0] = acc[p][sl][1] = 0ull;
#pragma unroll 1
    for (int k4 = 0; k4 < Ap; k4 += 4) {
      float4 u4[kEnvPer];
#pragma unroll
      for (int p = 0; p < kEnvPer; ++p) u4[p] = *reinterpret_cast<const float4*>(sa_w + p * 32 + k4);
#pragma unroll
      for (int kk = 0; kk < 4; ++kk) {
        uint64_t m2[kSlots][2];
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          const float4 m = sMT[(k4 + kk) * kQT + lane + 32 * sl];
          m2[sl][0] = pk(m.x, m.y);
          m2[sl][1] = pk(m.z, m.w);
        }
#pragma unroll
        for (int p = 0; p < kEnvPer; ++p) {
          const float u = kk == 0 ? u4[p].x : (kk == 1 ? u4[p].y : (kk == 2 ? u4[p].z : u4[p].w));
          const uint64_t uu = pk(u, u);
#pragma unroll
          for (int sl = 0; sl < kSlots; ++sl) {
            acc[p][sl][0] = add2(mul2(m2[sl][0], uu), acc[p][sl][0], one2);
            acc[p][sl][1] = add2(mul2(m2[sl][1], uu), acc[p][sl][1], one2);
          }
        }
      }
    }
    // s' = clamp(0.95 s + 0.05 acc) -> registers (s4) and the chain buffer
    float* svb = sv + buf * kEnvTile * ldv;
#pragma unroll
    for (int p = 0; p < kEnvPer; ++p)
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        float4& v = s4[p][sl];
        const uint64_t t01 = mul2(pk(v.x, v.y), c095), t23 = mul2(pk(v.z, v.w), c095);
        const uint64_t r01 = add2(mul2(acc[p][sl][0], c005), t01, one2);
        const uint64_t r23 = add2(mul2(acc[p][sl][1], c005), t23, one2);
        upk(r01, v.x, v.y);
        upk(r23, v.z, v.w);
        v.x = clamp10(v.x);
        v.y = clamp10(v.y);
        v.z = clamp10(v.z);
        v.w = clamp10(v.w);
        const int d0 = 4 * (lane + 32 * sl);
        float* row = svb + (w * kEnvPer + p) * ldv;
        if (d0 + 3 < D) {
          row[d0] = v.x;
          row[d0 + 1] = v.y;
          row[d0 + 2] = v.z;
          row[d0 + 3] = v.w;
        } else {
          if (d0 < D) row[d0] = v.x;
          if (d0 + 1 < D) row[d0 + 1] = v.y;
          if (d0 + 2 < D) row[d0 + 2] = v.z;
        }
      }
    // ---- 2: flags (lane p: env base + p), then the rows
    int flag = 0;
    {
      float mine = 0.0f;
#pragma unroll
      for (int p = 0; p < kEnvPer; ++p) {
        const float v0 = __shfl_sync(0xffffffffu, s4[p][0].x, 0);
        if (lane == p) mine = v0;
      }
      if (lane < kEnvPer && lane < nv) {
        const int i = base + lane;
        const bool terminal = fabsf(mine) > 9.0f;
        const int64_t ep = ep_prev + 1;
        const bool timeout = ep >= e.max_len;
        const bool done = terminal || timeout;
        const bool trunc = !terminal && timeout;
        e.episode_step[i] = done ? 0 : ep;
        flag = (done ? 1 : 0) | (trunc ? 2 : 0);
        sflag[buf * kEnvTile + w * kEnvPer + lane] = flag;
      }
    }
#pragma unroll
    for (int p = 0; p < kEnvPer; ++p) {
      if (p >= nv) break;
      const int i = base + p;
      const bool done = (__shfl_sync(0xffffffffu, flag, p) & 1) != 0;
      const uint64_t st0 = done ? e.rng[i] : 0ull;
      const int64_t ro = static_cast<int64_t>(i) * o.ld_obs;
      float* bt = o.boot + ro;
      float* nx = o.next_obs + ro;
      float* sr = e.s ? e.s + static_cast<int64_t>(i) * e.ld : nullptr;
      float* xn = nn.out ? nn.out + static_cast<int64_t>(i) * nn.ld_out : nullptr;
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl) {
        const int q = lane + 32 * sl;
        if (q >= Q) continue;
        const int d0 = 4 * q;
        const float4 v = s4[p][sl];
        float4 nv4 = v;
        if (done) {  // auto-reset: draw d of the reset sequence (vecenv.cpp:100-103)
          uint64_t t0 = st0 + static_cast<uint64_t>(d0);
          nv4.x = rng::env_uniform(t0, -1.0f, 1.0f);
          uint64_t t1 = st0 + static_cast<uint64_t>(d0 + 1);
          nv4.y = rng::env_uniform(t1, -1.0f, 1.0f);
          uint64_t t2 = st0 + static_cast<uint64_t>(d0 + 2);
          nv4.z = rng::env_uniform(t2, -1.0f, 1.0f);
          uint64_t t3 = st0 + static_cast<uint64_t>(d0 + 3);
          nv4.w = rng::env_uniform(t3, -1.0f, 1.0f);
        }
        float4 z = nv4;
        if (xnorm) {
          float zz[4] = {nv4.x, nv4.y, nv4.z, nv4.w};
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            float t = __fmul_rn(__fsub_rn(zz[c], nm[sl][c]), ni[sl][c]);
            if (t > 5.0f) t = 5.0f;
            if (t < -5.0f) t = -5.0f;
            zz[c] = t;
          }
          z = make_float4(zz[0], zz[1], zz[2], zz[3]);
        }
        if (vec && d0 + 3 < D) {
          *reinterpret_cast<float4*>(bt + d0) = v;
          *reinterpret_cast<float4*>(nx + d0) = nv4;
          if (sr) *reinterpret_cast<float4*>(sr + d0) = nv4;
          if (xn) *reinterpret_cast<float4*>(xn + d0) = z;
        } else {
          const float vv[4] = {v.x, v.y, v.z, v.w}, nn4[4] = {nv4.x, nv4.y, nv4.z, nv4.w},
                      z4[4] = {z.x, z.y, z.z, z.w};
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (d0 + c < D) {
              bt[d0 + c] = vv[c];
              nx[d0 + c] = nn4[c];
              if (sr) sr[d0 + c] = nn4[c];
              if (xn) xn[d0 + c] = z4[c];
            }
        }
      }
      if (done && lane == 0) e.rng[i] = st0 + static_cast<uint64_t>(D);
    }
    // ---- 3: the reward chains of this tile (one warp, lane = env)
    __syncthreads();
    if (w == (it & (kEnvWarps - 1))) {
      const int i = i0 + lane;
      if (i < e.N) {
        const float* row = svb + lane * ldv;
        float ss = 0.0f;
        int d = 0;
        for (; d + 8 <= D; d += 8) {
          float q8[8];
#pragma unroll
          for (int t = 0; t < 8; ++t) q8[t] = row[d + t];
#pragma unroll
          for (int t = 0; t < 8; ++t) ss = __fadd_rn(ss, __fmul_rn(q8[t], q8[t]));
        }
        for (; d < D; ++d) ss = __fadd_rn(ss, __fmul_rn(row[d], row[d]));
        const float reward =
            -__fadd_rn(__fdiv_rn(ss, static_cast<float>(D)),
                       __fmul_rn(0.01f, __fdiv_rn(saa[buf * kEnvTile + lane], static_cast<float>(A))));
        const int f = sflag[buf * kEnvTile + lane];
        const bool done = (f & 1) != 0, trunc = (f & 2) != 0;
        o.rew[i] = reward;
        o.term[i] = static_cast<uint8_t>(done && !trunc);
        o.trunc[i] = static_cast<uint8_t>(trunc);
        if (o.done) o.done[i] = static_cast<uint8_t>(done);
      }
    }
    // sv / saa / sflag [buf] are rewritten two tiles later, after the next
    // barrier, which this tile's chain warp reaches only when it is done
  }
}

// ---------------------------------------------------------------------------
// TMA-fed persistent env step (the actor's path; same arithmetic as
// env_step_kernel above, so states / rewards / flags stay bit-exact).
//
// One CTA per SM walks the 32-env tiles blockIdx.x, +gridDim.x, ...; every
// tile moves through shared memory in whole contiguous row blocks, in and
// out by 1-D bulk copies (cp.async.bulk), and the warps specialise:
//   producer warp    bulk loads of the tile's observation and action rows
//                    into a kEnvStages-deep ring (full / ready / empty
//                    mbarriers per stage)
//   8 step warps     4 envs each (lane = observation quads): clamped actions,
//                    sum a^2, M a, s' (written back into the stage rows) and
//                    the done / truncation flags
//   1 chain warp     lane = env: the d-ascending s'^2 reward
//                    sum read as float4 from the stage (row stride 212 floats
//                    puts 8 lanes on 8 distinct bank quads: conflict-free),
//                    rewards and flags out
//   6 writer warps   rows w, w+6, ... (lane = quads): next obs (fresh reset
//                    draws on done rows) and its normalisation, float4 stores
//                    straight from registers, and optionally the fp64
//                    running-normalizer partial sums of the next observations
//                    (shifted by the running mean), so the next step's
//                    normalizer update needs no second pass over them; the
//                    first writer lane bulk-stores boot (= s') straight from
//                    the stage rows and releases the stage once that store
//                    has read it
// ---------------------------------------------------------------------------
constexpr int kEnvStages = 4;
#ifndef PQLG_ENV_STEP_WARPS
#define PQLG_ENV_STEP_WARPS 8
#endif
constexpr int kTStepWarps = PQLG_ENV_STEP_WARPS;   // step warps ...
constexpr int kTPer = kEnvTile / kTStepWarps;       // ... of kTPer envs each
#ifndef PQLG_ENV_CHAIN
#define PQLG_ENV_CHAIN 1
#endif
constexpr int kEnvChainWarps = PQLG_ENV_CHAIN;
#ifndef PQLG_ENV_WRITERS
#define PQLG_ENV_WRITERS 6
#endif
constexpr int kEnvWriterWarps = PQLG_ENV_WRITERS;
constexpr int kEnvTmaWarps = kTStepWarps + kEnvChainWarps + kEnvWriterWarps + 1;
constexpr int kEnvTmaThreads = 32 * kEnvTmaWarps;

// Running-normalizer partials of the step's next observations (null: off).
struct NormPartialOut {
  double2* partial;     // [gridDim.x][D]: (sum (x - shift), sum (x - shift)^2) per column
  double* shift_out;    // [D] the shift used (block 0 writes it)
  const double* mean;   // running mean (fp64) = the shift
};

// Stage: [rows 32 x ld][act rows 32 x ld_act][aa 32][flags 32]
__host__ __device__ inline int64_t env_tma_stage_bytes(int64_t ld, int64_t ld_act) {
  return (static_cast<int64_t>(kEnvTile) * (ld + ld_act) * 4 + 2 * kEnvTile * 4 + 127) / 128 * 128;
}
inline size_t env_tma_smem(int A, int slots, int64_t ld, int64_t ld_act) {
  const int Ap = (A + 3) & ~3;
  return static_cast<size_t>(Ap) * 32 * slots * 16 + kTStepWarps * kTPer * 32 * 4 +
         kEnvStages * env_tma_stage_bytes(ld, ld_act) + 3 * kEnvStages * 8;
}
// The bulk path needs one row stride for the state, boot, next obs and
// normalised next obs (the actor's Dp-wide buffers) and 16-byte rows.
inline bool env_tma_ok(const float* act, int64_t ld_act, int D, int A, int64_t ld) {
  const int64_t red = static_cast<int64_t>(kEnvWriterWarps) * 4 * ((D + 3) / 4) * 16;
  const int slots = (D + 3) / 4 <= 32 ? 1 : 2;
  return (ld_act % 4) == 0 && (ld % 4) == 0 && (reinterpret_cast<uintptr_t>(act) & 15) == 0 &&
         D <= kMaxD && kEnvStages * env_tma_stage_bytes(ld, ld_act) >= red &&
         env_tma_smem(A, slots, ld, ld_act) <= 227 * 1024;
}

// Phase timestamps (%globaltimer, ns) of the TMA env step, per CTA [32 slots]
// (tools/env_trace.py builds a variant with -DPQLG_ENV_TRACE; the product never does).
#ifdef PQLG_ENV_TRACE
__device__ unsigned long long* g_env_trace;
__device__ __forceinline__ void env_trace(int slot) {
  if (g_env_trace && slot < 32) {
    unsigned long long t;
    asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
    g_env_trace[blockIdx.x * 32 + slot] = t;
  }
}
#else
__device__ __forceinline__ void env_trace(int) {}
#endif

#ifdef PQLG_ENV_SPIN
#define PQLG_ENV_WAIT ptx::mbar_wait_spin
#else
#define PQLG_ENV_WAIT ptx::mbar_wait
#endif

__device__ __forceinline__ void bulk_store_1d(void* gmem, const void* smem, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(
                   reinterpret_cast<uint64_t>(gmem)),
               "r"(ptx::smem_u32(smem)), "r"(bytes)
               : "memory");
}

template <int kSlots>
static __global__ void __launch_bounds__(kEnvTmaThreads, 1)
    env_step_tma_kernel(EnvState e, const float* __restrict__ act, int64_t ld_act, StepOut o,
                        NextNorm nn, NormPartialOut np) {
  extern __shared__ __align__(128) float4 sh4[];
  constexpr int kQT = 32 * kSlots;
  const int D = e.D, A = e.A, Q = (D + 3) >> 2;
  const int Ap = (A + 3) & ~3;
  const int64_t ld = e.ld_in;  // = o.ld_obs = nn.ld_out (= e.ld): checked by the host
  const int64_t stage_bytes = env_tma_stage_bytes(ld, ld_act);
  float4* sMT = sh4;                                                // [Ap][kQT]
  float* sa = reinterpret_cast<float*>(sMT + Ap * kQT);             // [warp][kTPer][32]
  uint8_t* ring = reinterpret_cast<uint8_t*>(sa + kTStepWarps * kTPer * 32);
  uint64_t* full = reinterpret_cast<uint64_t*>(ring + kEnvStages * stage_bytes);
  uint64_t* ready = full + kEnvStages;
  uint64_t* empty = ready + kEnvStages;
  auto st_obs = [&](int s) { return reinterpret_cast<float*>(ring + s * stage_bytes); };
  auto st_act = [&](int s) { return st_obs(s) + kEnvTile * ld; };
  auto st_aa = [&](int s) { return st_act(s) + kEnvTile * ld_act; };
  auto st_flag = [&](int s) { return reinterpret_cast<int*>(st_aa(s) + kEnvTile); };

  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) env_trace(0);
  constexpr int kChain0 = kTStepWarps, kWriter0 = kTStepWarps + kEnvChainWarps;
  constexpr int kProducer = kWriter0 + kEnvWriterWarps;
  // M^T (constant since env creation) and the barriers before the PDL wait
  for (int idx = threadIdx.x; idx < Ap * kQT; idx += blockDim.x) {
    const int k = idx / kQT, q = idx - k * kQT;
    sMT[idx] = __ldg(e.MT + k * (kMaxD / 4) + q);
  }
  if (threadIdx.x == 0) {
    for (int s = 0; s < kEnvStages; ++s) {
      ptx::mbar_init(&full[s], 1);
      ptx::mbar_init(&ready[s], 32 * kTStepWarps);
      ptx::mbar_init(&empty[s], 2);  // the tile's chain warp + the store-issuing writer
    }
    ptx::fence_barrier_init();
  }
  __syncthreads();
  pdl::entry();
  if (threadIdx.x == 0) env_trace(1);
  const int n_tiles = (e.N + kEnvTile - 1) / kEnvTile;

  double s1[kSlots][4], s2[kSlots][4];
#pragma unroll
  for (int sl = 0; sl < kSlots; ++sl)
#pragma unroll
    for (int c = 0; c < 4; ++c) s1[sl][c] = s2[sl][c] = 0.0;

  if (w == kProducer) {
    if (lane == 0) {
      int k = 0;
      for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
        const int s = k % kEnvStages;
        PQLG_ENV_WAIT(&empty[s], ((k / kEnvStages) & 1) ^ 1);
        const int i0 = tile * kEnvTile;
        const int nv = min(kEnvTile, e.N - i0);
        const uint32_t ob = static_cast<uint32_t>(nv * ld * 4);
        const uint32_t ab = static_cast<uint32_t>(nv * ld_act * 4);
        ptx::mbar_arrive_expect_tx(&full[s], ob + ab);
        ptx::bulk_load_1d(st_obs(s), e.s_in + static_cast<int64_t>(i0) * ld, ob, &full[s]);
        ptx::bulk_load_1d(st_act(s), act + static_cast<int64_t>(i0) * ld_act, ab, &full[s]);
      }
    }
  } else if (w >= kWriter0) {
    // ---- writers: rows ww, ww + kEnvWriterWarps, ... of each tile (lane = quads)
    const int ww = w - kWriter0;
    const bool xnorm = nn.out != nullptr && *nn.identity == 0;
    float nm[kSlots][4], ni[kSlots][4];
    double shf[kSlots][4];
#pragma unroll
    for (int sl = 0; sl < kSlots; ++sl)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int d = 4 * (lane + 32 * sl) + c;
        nm[sl][c] = (xnorm && d < D) ? nn.mean[d] : 0.0f;
        ni[sl][c] = (xnorm && d < D) ? nn.inv[d] : 1.0f;
        // padding columns: zero values minus a zero shift add nothing
        shf[sl][c] = (np.partial && d < D) ? np.mean[d] : 0.0;
      }
    int k = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
      const int s = k % kEnvStages;
      PQLG_ENV_WAIT(&ready[s], (k / kEnvStages) & 1);
      if (threadIdx.x == 32 * kWriter0 && k == 0) env_trace(16);
      const int i0 = tile * kEnvTile;
      const int nrow = min(kEnvTile, e.N - i0);
      if (threadIdx.x == 32 * kWriter0)  // boot = s', straight from the stage rows
        bulk_store_1d(o.boot + static_cast<int64_t>(i0) * ld, st_obs(s),
                      static_cast<uint32_t>(nrow * ld * 4));
#pragma unroll 1
      for (int r = ww; r < nrow; r += kEnvWriterWarps) {
        const int i = i0 + r;
        const bool done = (st_flag(s)[r] & 1) != 0;
        const uint64_t st0 = done ? e.rng[i] : 0ull;
        const float* srow = st_obs(s) + static_cast<int64_t>(r) * ld;
        const int64_t ro = static_cast<int64_t>(i) * ld;
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          const int q = lane + 32 * sl;
          if (q >= Q) continue;
          const int d0 = 4 * q;
          float4 nv4 = *reinterpret_cast<const float4*>(srow + d0);
          if (done) {  // auto-reset: draw d of the reset sequence (vecenv.cpp:100-103)
            uint64_t t0 = st0 + static_cast<uint64_t>(d0);
            nv4.x = rng::env_uniform(t0, -1.0f, 1.0f);
            uint64_t t1 = st0 + static_cast<uint64_t>(d0 + 1);
            nv4.y = rng::env_uniform(t1, -1.0f, 1.0f);
            uint64_t t2 = st0 + static_cast<uint64_t>(d0 + 2);
            nv4.z = rng::env_uniform(t2, -1.0f, 1.0f);
            uint64_t t3 = st0 + static_cast<uint64_t>(d0 + 3);
            nv4.w = rng::env_uniform(t3, -1.0f, 1.0f);
            if (d0 + 3 >= D) {  // padding columns stay zero
              if (d0 + 1 >= D) nv4.y = 0.0f;
              if (d0 + 2 >= D) nv4.z = 0.0f;
              nv4.w = 0.0f;
            }
          }
          const float x4[4] = {nv4.x, nv4.y, nv4.z, nv4.w};
          if (np.partial) {
#pragma unroll
            for (int c = 0; c < 4; ++c) {
              const double dd = static_cast<double>(x4[c]) - shf[sl][c];
              s1[sl][c] += dd;
              s2[sl][c] = fma(dd, dd, s2[sl][c]);
            }
          }
          // the padding columns d >= D of the last quad are zero (M^T is zero padded)
          *reinterpret_cast<float4*>(o.next_obs + ro + d0) = nv4;
          if (e.s) *reinterpret_cast<float4*>(e.s + ro + d0) = nv4;
          if (nn.out) {
            float4 z = nv4;
            if (xnorm) {
              float zz[4];
#pragma unroll
              for (int c = 0; c < 4; ++c) {
                float t = __fmul_rn(__fsub_rn(x4[c], nm[sl][c]), ni[sl][c]);
                if (t > 5.0f) t = 5.0f;
                if (t < -5.0f) t = -5.0f;
                zz[c] = t;
              }
              z = make_float4(zz[0], zz[1], zz[2], zz[3]);
            }
            *reinterpret_cast<float4*>(nn.out + ro + d0) = z;
          }
        }
        if (done && lane == 0) e.rng[i] = st0 + static_cast<uint64_t>(D);
      }
      // every writer is done reading the stage; the boot store has read it
      ptx::named_bar_sync(1, 32 * kEnvWriterWarps);
      if (threadIdx.x == 32 * kWriter0) {
        asm volatile("cp.async.bulk.commit_group;" ::: "memory");
        if (k < 4) env_trace(28 + k);
        asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        ptx::mbar_arrive(&empty[s]);
        if (k < 4) env_trace(20 + k);
      }
    }
    if (threadIdx.x == 32 * kWriter0)  // global writes complete before the kernel ends
      asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  } else if (w >= kChain0) {
    // ---- reward chains (lane = env), alternate tiles
    const int cw = w - kChain0;
    int k = cw;
    for (int tile = blockIdx.x + cw * gridDim.x; tile < n_tiles;
         tile += kEnvChainWarps * gridDim.x, k += kEnvChainWarps) {
      const int s = k % kEnvStages;
      PQLG_ENV_WAIT(&ready[s], (k / kEnvStages) & 1);
      const int i = tile * kEnvTile + lane;
      if (i < e.N) {
        const float* row = st_obs(s) + lane * ld;
        float ss = 0.0f;
        int d = 0;
        for (; d + 16 <= D; d += 16) {
          float4 q4[4];
#pragma unroll
          for (int t = 0; t < 4; ++t) q4[t] = *reinterpret_cast<const float4*>(row + d + 4 * t);
#pragma unroll
          for (int t = 0; t < 4; ++t) {
            ss = __fadd_rn(ss, __fmul_rn(q4[t].x, q4[t].x));
            ss = __fadd_rn(ss, __fmul_rn(q4[t].y, q4[t].y));
            ss = __fadd_rn(ss, __fmul_rn(q4[t].z, q4[t].z));
            ss = __fadd_rn(ss, __fmul_rn(q4[t].w, q4[t].w));
          }
        }
        for (; d < D; ++d) ss = __fadd_rn(ss, __fmul_rn(row[d], row[d]));
        const float reward =
            -__fadd_rn(__fdiv_rn(ss, static_cast<float>(D)),
                       __fmul_rn(0.01f, __fdiv_rn(st_aa(s)[lane], static_cast<float>(A))));
        const int f = st_flag(s)[lane];
        const bool done = (f & 1) != 0, trunc = (f & 2) != 0;
        o.rew[i] = reward;
        o.term[i] = static_cast<uint8_t>(done && !trunc);
        o.trunc[i] = static_cast<uint8_t>(trunc);
        if (o.done) o.done[i] = static_cast<uint8_t>(done);
      }
      __syncwarp();
      if (lane == 0) ptx::mbar_arrive(&empty[s]);
      if (lane == 0 && k < 4) env_trace(24 + k);
    }
  } else {
    // ---- step warps: s' = clamp(0.95 s + 0.05 M clamp(a)) and the flags
    const uint64_t one2 = pk(e.one, e.one);
    const uint64_t c095 = pk(0.95f, 0.95f), c005 = pk(0.05f, 0.05f);
    float* sa_w = sa + w * kTPer * 32;
    int k = 0;
    for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x, ++k) {
      const int s = k % kEnvStages;
      const int i0 = tile * kEnvTile;
      const int base = i0 + w * kTPer;
      const int nv = e.N - base;  // valid envs of this warp (may be <= 0)
      const int64_t ep_prev = (lane < kTPer && lane < nv) ? e.episode_step[base + lane] : 0;
      PQLG_ENV_WAIT(&full[s], (k / kEnvStages) & 1);
      if (threadIdx.x == 0 && k < 4) env_trace(4 + k);
      float* srow0 = st_obs(s) + static_cast<int64_t>(w * kTPer) * ld;
      const float* arow0 = st_act(s) + static_cast<int64_t>(w * kTPer) * ld_act;
      {
        bool bad = false;
#pragma unroll
        for (int p = 0; p < kTPer; ++p) {
          float u = (lane < A && p < nv) ? arow0[p * ld_act + lane] : 0.0f;
          if (lane < A && p < nv) {
            bad |= !isfinite(u);
            u = u < e.low ? e.low : (u > e.high ? e.high : u);
          }
          sa_w[p * 32 + lane] = u;
        }
        if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(o.status, 8u);
      }
      __syncwarp();
      if (lane < kTPer) {  // sum a^2, k ascending
        const float* ap = sa_w + lane * 32;
        float aa = 0.0f;
        for (int kk = 0; kk < A; ++kk) aa = __fadd_rn(aa, __fmul_rn(ap[kk], ap[kk]));
        st_aa(s)[w * kTPer + lane] = aa;
      }
      if (threadIdx.x == 0 && k == 0) env_trace(17);
      // ---- M a, k ascending (sums start at +0 like the reference's loop)
      uint64_t acc[kTPer][kSlots][2];
#pragma unroll
      for (int p = 0; p < kTPer; ++p)
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) acc[p][sl][0] = acc[p][sl][1] = 0ull;
#pragma unroll 1
      for (int k4 = 0; k4 < Ap; k4 += 4) {
        float4 u4[kTPer];
#pragma unroll
        for (int p = 0; p < kTPer; ++p) u4[p] = *reinterpret_cast<const float4*>(sa_w + p * 32 + k4);
#pragma unroll
        for (int kk = 0; kk < 4; ++kk) {
          uint64_t m2[kSlots][2];
#pragma unroll
          for (int sl = 0; sl < kSlots; ++sl) {
            const float4 m = sMT[(k4 + kk) * kQT + lane + 32 * sl];
            m2[sl][0] = pk(m.x, m.y);
            m2[sl][1] = pk(m.z, m.w);
          }
#pragma unroll
          for (int p = 0; p < kTPer; ++p) {
            const float u = kk == 0 ? u4[p].x : (kk == 1 ? u4[p].y : (kk == 2 ? u4[p].z : u4[p].w));
            const uint64_t uu = pk(u, u);
#pragma unroll
            for (int sl = 0; sl < kSlots; ++sl) {
              acc[p][sl][0] = add2(mul2(m2[sl][0], uu), acc[p][sl][0], one2);
              acc[p][sl][1] = add2(mul2(m2[sl][1], uu), acc[p][sl][1], one2);
            }
          }
        }
      }
      // s' back into the stage rows (for the chain, the writers and the boot
      // store); s is read only now, so it does not occupy registers during M a
      if (threadIdx.x == 0 && k == 0) env_trace(18);
      float s0[kTPer];  // s'_0 of each env (the terminal test)
#pragma unroll
      for (int p = 0; p < kTPer; ++p)
#pragma unroll
        for (int sl = 0; sl < kSlots; ++sl) {
          const int q = lane + 32 * sl;
          float4 v = (p < nv && q < Q) ? *reinterpret_cast<const float4*>(srow0 + p * ld + 4 * q)
                                       : make_float4(0.f, 0.f, 0.f, 0.f);
          const uint64_t t01 = mul2(pk(v.x, v.y), c095), t23 = mul2(pk(v.z, v.w), c095);
          const uint64_t r01 = add2(mul2(acc[p][sl][0], c005), t01, one2);
          const uint64_t r23 = add2(mul2(acc[p][sl][1], c005), t23, one2);
          upk(r01, v.x, v.y);
          upk(r23, v.z, v.w);
          v.x = clamp10(v.x);
          v.y = clamp10(v.y);
          v.z = clamp10(v.z);
          v.w = clamp10(v.w);
          if (sl == 0) s0[p] = v.x;
          if (p < nv && q < Q) *reinterpret_cast<float4*>(srow0 + p * ld + 4 * q) = v;
        }
      if (threadIdx.x == 0 && k == 0) env_trace(19);
      // flags (lane p: env base + p)
      {
        float mine = 0.0f;
#pragma unroll
        for (int p = 0; p < kTPer; ++p) {
          const float v0 = __shfl_sync(0xffffffffu, s0[p], 0);
          if (lane == p) mine = v0;
        }
        if (lane < kTPer && lane < nv) {
          const int i = base + lane;
          const bool terminal = fabsf(mine) > 9.0f;
          const int64_t ep = ep_prev + 1;
          const bool timeout = ep >= e.max_len;
          const bool done = terminal || timeout;
          const bool trunc = !terminal && timeout;
          e.episode_step[i] = done ? 0 : ep;
          st_flag(s)[w * kTPer + lane] = (done ? 1 : 0) | (trunc ? 2 : 0);
        }
      }
      // s', aa and the flags are complete in the stage
      ptx::fence_proxy_async_smem();  // the boot bulk store reads the s' rows
      ptx::mbar_arrive(&ready[s]);
      if (threadIdx.x == 0 && k < 4) env_trace(8 + k);
    }
  }
  if (lane == 0) env_trace(12 + (w < kTStepWarps ? 0 : (w < kWriter0 ? 1 : (w < kProducer ? 2 : 3))));
  // ---- the block's normalizer partials, writer warps added in fixed order
  if (np.partial) {
    __syncthreads();  // every stage consumed: the ring is free
    double2* red = reinterpret_cast<double2*>(ring);  // [kEnvWriterWarps][4 Q]
    if (w >= kWriter0 && w < kProducer) {
#pragma unroll
      for (int sl = 0; sl < kSlots; ++sl)
#pragma unroll
        for (int c = 0; c < 4; ++c)
          if (lane + 32 * sl < Q)
            red[(w - kWriter0) * (4 * Q) + 4 * (lane + 32 * sl) + c] = make_double2(s1[sl][c], s2[sl][c]);
    }
    __syncthreads();
    for (int c = threadIdx.x; c < D; c += blockDim.x) {
      double a = 0.0, b = 0.0;
#pragma unroll
      for (int ww = 0; ww < kEnvWriterWarps; ++ww) {
        const double2 t = red[ww * (4 * Q) + c];
        a += t.x;
        b += t.y;
      }
      np.partial[static_cast<int64_t>(blockIdx.x) * D + c] = make_double2(a, b);
      if (blockIdx.x == 0) np.shift_out[c] = np.mean[c];
    }
  }
  if (threadIdx.x == 0) env_trace(2);
}

// Host: M^T zero padded to [round_up(A, 4)][kMaxD] for the kernel's copy.
inline std::vector<float> env_transpose_M(const std::vector<float>& M, int D, int A) {
  const int Ap = (A + 3) & ~3;
  std::vector<float> t(static_cast<size_t>(Ap) * kMaxD, 0.0f);
  for (int d = 0; d < D; ++d)
    for (int k = 0; k < A; ++k) t[static_cast<size_t>(k) * kMaxD + d] = M[static_cast<size_t>(d) * A + k];
  return t;
}

inline size_t env_step_smem(int D, int A, int slots) {
  const int Ap = (A + 3) & ~3;
  return (static_cast<size_t>(Ap) * 128 * slots + 2ull * kEnvTile * (D | 1) + kEnvTile * 32 +
          4ull * kEnvTile) *
         sizeof(float);
}

// reset_all (vecenv.cpp:53-60) + staggered episode_step = i % max_len.
static __global__ void env_reset_kernel(EnvState e, float* obs, int64_t ld_obs, int env_offset) {
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * kEnvWarps + w;
  if (i >= e.N) return;
  const uint64_t st0 = e.rng[i];
  float* s = e.s + static_cast<int64_t>(i) * e.ld;
  for (int d = lane; d < e.D; d += 32) {
    uint64_t st = st0 + static_cast<uint64_t>(d);
    const float v = rng::env_uniform(st, -1.0f, 1.0f);
    s[d] = v;
    obs[static_cast<int64_t>(i) * ld_obs + d] = v;
  }
  if (lane == 0) {
    e.rng[i] = st0 + static_cast<uint64_t>(e.D);
    e.episode_step[i] = (static_cast<int64_t>(env_offset) + i) % e.max_len;
  }
}

// out = apply_stats(obs) with fp32 constants (identity if count <= 1).
static __global__ void normalize_kernel(const float* __restrict__ x, int64_t ldx, float* out,
                                        int64_t ldo, const float* mean, const float* inv,
                                        const int* identity, int N, int D) {
  pdl::entry();
  const int64_t n = static_cast<int64_t>(N) * D;
  const bool id = *identity != 0;
  for (int64_t e = blockIdx.x * static_cast<int64_t>(blockDim.x) + threadIdx.x; e < n;
       e += static_cast<int64_t>(gridDim.x) * blockDim.x) {
    const int64_t r = e / D;
    const int d = static_cast<int>(e % D);
    float z = x[r * ldx + d];
    if (!id) {
      z = __fmul_rn(__fsub_rn(z, mean[d]), inv[d]);
      if (z > 5.0f) z = 5.0f;
      if (z < -5.0f) z = -5.0f;
    }
    out[r * ldo + d] = z;
  }
}

// RunningNormalizer::update (normalizer.hpp:33-50, :73-83) in two launches,
// parallel and deterministic:
//   norm_partial_kernel  one wave of row blocks (kNormBlocks): block g takes a
//                        contiguous row range; its threads are (row lane,
//                        column quad) -- float4 loads of whole rows, fp64
//                        sums of (x - shift) and (x - shift)^2 per column,
//                        shift = the batch's first row (no cancellation for
//                        offset data); the row lanes are added in fixed order
//                        -> partial[g][c] = (s1, s2)
//   norm_finish_kernel   a block per 32 columns: warp w sums blocks w, w+16,
//                        ... in order, the 16 warp sums in order; the batch
//                        (mean, M2) is merged into the running stats with
//                        Chan's formula and the fp32 apply constants refreshed
//                        (normalizer.hpp:62-66); the last block advances the
//                        count (every block read the old one first).
constexpr int kNormBlocks = 148;      // partial rows (one wave, upper bound)
constexpr int kNormThreads = 512;     // partial kernel: 8 row lanes x 64 quads
constexpr int kNormQuads = 64;
constexpr int kNormLanes = kNormThreads / kNormQuads;
inline int norm_blocks(int N) {
  // at least ~32 rows per block so the fixed cost amortises
  int g = (N + 31) / 32;
  return g < 1 ? 1 : (g > kNormBlocks ? kNormBlocks : g);
}
inline int norm_tickets(int) { return 1; }

// vec: x rows are 16-byte aligned (ldx % 4 == 0, 16-byte base); otherwise
// scalar loads.
template <bool kVec>
static __global__ void __launch_bounds__(kNormThreads)
    norm_partial_kernel(const float* __restrict__ x, int64_t ldx, int N, int D,
                        double2* __restrict__ partial, double* shift_out) {
  pdl::entry();
  if (blockIdx.x == 0)  // the shift: the batch's first row
    for (int c = threadIdx.x; c < D; c += blockDim.x) shift_out[c] = static_cast<double>(x[c]);
  __shared__ double2 red[kNormLanes][kNormQuads][4];  // 32 KB
  const int lane_r = threadIdx.x / kNormQuads, q0 = threadIdx.x % kNormQuads;
  const int g = blockIdx.x;
  const int per = (N + gridDim.x - 1) / gridDim.x;
  const int r0 = g * per, r1 = min(r0 + per, N);
  const int Q = (D + 3) >> 2;
  for (int qb = 0; qb < Q; qb += kNormQuads) {
    const int q = qb + q0;
    double s1[4] = {0.0, 0.0, 0.0, 0.0}, s2[4] = {0.0, 0.0, 0.0, 0.0};
    if (q < Q) {
      float sh[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) sh[u] = 4 * q + u < D ? x[4 * q + u] : 0.0f;
      constexpr int kU = 8;  // rows in flight per thread
      for (int rb = r0 + lane_r; rb < r1; rb += kNormLanes * kU) {
        float4 v[kU];
#pragma unroll
        for (int t = 0; t < kU; ++t) {
          const int r = rb + kNormLanes * t;
          v[t] = make_float4(0.f, 0.f, 0.f, 0.f);
          if (r < r1) {
            const float* row = x + static_cast<int64_t>(r) * ldx + 4 * q;
            if constexpr (kVec) {
              v[t] = __ldg(reinterpret_cast<const float4*>(row));
            } else {
              v[t].x = row[0];
              if (4 * q + 1 < D) v[t].y = row[1];
              if (4 * q + 2 < D) v[t].z = row[2];
              if (4 * q + 3 < D) v[t].w = row[3];
            }
          }
        }
#pragma unroll
        for (int t = 0; t < kU; ++t) {
          if (rb + kNormLanes * t < r1) {
            const float e[4] = {v[t].x, v[t].y, v[t].z, v[t].w};
#pragma unroll
            for (int u = 0; u < 4; ++u) {
              const double d = static_cast<double>(e[u]) - static_cast<double>(sh[u]);
              s1[u] += d;
              s2[u] += d * d;
            }
          }
        }
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) red[lane_r][q0][u] = make_double2(s1[u], s2[u]);
    __syncthreads();
    // fixed-order sum of the row lanes; thread (c within this quad block)
    for (int cc = threadIdx.x; cc < 4 * kNormQuads; cc += blockDim.x) {
      const int c = 4 * qb + cc;
      if (c < D) {
        double a = 0.0, b = 0.0;
#pragma unroll
        for (int l = 0; l < kNormLanes; ++l) {
          const double2 t = red[l][cc >> 2][cc & 3];
          a += t.x;
          b += t.y;
        }
        partial[static_cast<int64_t>(g) * D + c] = make_double2(a, b);
      }
    }
    __syncthreads();
  }
}

static __global__ void __launch_bounds__(32 * kNormFinishWarps)
    norm_finish_kernel(const NormFinishArgs f) {
  pdl::entry();
  __shared__ double2 red[kNormFinishWarps * 32];
  norm_finish_block(f, blockIdx.x, red);
}

// Host: the update's two launches (partial buffer: kNormBlocks x D double2,
// shift: D doubles).  The actor splits them: the partials of step t+1's
// observations come out of step t's env kernel (NormPartialOut), so a step
// only runs the finish (norm_finish); norm_partial covers the first step.
inline void norm_partial(const float* x, int64_t ldx, int N, int D, int blocks, double* partial,
                         double* shift, cudaStream_t st) {
  const bool vec = (ldx % 4) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  double2* part = reinterpret_cast<double2*>(partial);
  if (vec)
    launch(norm_partial_kernel<true>, dim3(blocks), dim3(kNormThreads), 0, st, x, ldx, N, D, part,
           shift);
  else
    launch(norm_partial_kernel<false>, dim3(blocks), dim3(kNormThreads), 0, st, x, ldx, N, D, part,
           shift);
}
inline NormFinishArgs norm_finish_args(const double* shift, int N, int D, int blocks,
                                       const double* partial, unsigned int* ticket,
                                       const NormState& ns) {
  return NormFinishArgs{shift, N, D, blocks, reinterpret_cast<const double2*>(partial), ticket, ns,
                        norm_finish_blocks(D)};
}
inline void norm_finish(const double* shift, int N, int D, int blocks, const double* partial,
                        unsigned int* ticket, const NormState& ns, cudaStream_t st) {
  launch(norm_finish_kernel, dim3(norm_finish_blocks(D)), dim3(32 * kNormFinishWarps), 0, st,
         norm_finish_args(shift, N, D, blocks, partial, ticket, ns));
}
inline void norm_update(const float* x, int64_t ldx, int N, int D, double* partial, double* shift,
                        unsigned int* ticket, const NormState& ns, cudaStream_t st) {
  const int g = norm_blocks(N);
  norm_partial(x, ldx, N, D, g, partial, shift, st);
  norm_finish(shift, N, D, g, partial, ticket, ns, st);
}

// Sharded actor: after an all-gather of every shard's batch
// statistics ([world][2D + 1]: mean, M2, n), each rank combines them in rank
// order (Chan) and merges the result into its running stats, so all shards
// keep identical normalizers -- the statistics of the concatenated batch up
// to fp64 rounding.  With one shard this is the unsharded update bit for bit.
// One block, a thread per column (D <= 1024).
static __global__ void norm_merge_kernel(const double* __restrict__ gathered, int world, int D,
                                         NormState s) {
  pdl::entry();
  const int c = threadIdx.x;
  const int64_t stride = 2 * static_cast<int64_t>(D) + 1;
  const int64_t n0i = *s.count;
  int64_t nsum = 0;
  for (int k = 0; k < world; ++k) nsum += static_cast<int64_t>(gathered[k * stride + 2 * D]);
  if (c < D) {
    double nb = gathered[2 * D];
    double bmean = gathered[c], bm2 = gathered[D + c];
    for (int k = 1; k < world; ++k) {
      const double* g = gathered + k * stride;
      chan_merge(nb, bmean, bm2, g[2 * D], g[c], g[D + c]);
      nb += g[2 * D];
    }
    double mean = s.mean[c], m2 = s.m2[c];
    chan_merge(static_cast<double>(n0i), mean, m2, nb, bmean, bm2);
    s.mean[c] = mean;
    s.m2[c] = m2;
    s.mean_f[c] = static_cast<float>(mean);
    s.inv_f[c] = static_cast<float>(1.0 / sqrt(m2 / static_cast<double>(n0i + nsum) + 1e-8));
  }
  __syncthreads();  // every thread has read the old count
  if (c == 0) {
    *s.count = n0i + nsum;
    *s.identity = n0i + nsum <= 1 ? 1 : 0;
  }
}


// Standalone apply_noise (op-level hook): one thread per env row.
static __global__ void noise_kernel(float* act, int64_t ld, int N, int A, const float* sigma,
                                    float low, float high, uint64_t* states) {
  pdl::entry();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  float* row = act + static_cast<int64_t>(i) * ld;
  const float sig = sigma[i];
  uint64_t st = states[i];
  if (sig > 0.0f) {
    float saved = 0.0f;
    bool has = false;
    for (int d = 0; d < A; ++d) {
      float z;
      if (has) {
        has = false;
        z = saved;
      } else {
        z = rng::polar_pair(st, saved);
        has = true;
      }
      row[d] = __fadd_rn(row[d], __fadd_rn(__fmul_rn(z, sig), 0.0f));
    }
  }
  for (int d = 0; d < A; ++d) {
    float v = row[d];
    if (v < low) v = low;
    if (v > high) v = high;
    row[d] = v;
  }
  states[i] = st;
}

}  // namespace pqlg::actor
