// Actor-side kernels: the synthetic vectorised environment, observation
// normalisation, the running-normalizer update and (for the op-level hook)
// standalone mixed exploration noise.
//
//   env step       EnvBatch::step contract (vecenv.cpp:84-106) with the
//                  synthetic task of SURVEY 8(d); float mul/add only, in the
//                  oracle's order, so states/rewards are bit-exact
//   normalize      RunningNormalizer::apply_stats (normalizer.hpp:56-70)
//   norm update    RunningNormalizer::update + merge (normalizer.hpp:33-50,
//                  :73-83): Welford per 128-row chunk (row order), chunks
//                  merged with Chan's formula in fixed tree order, fp64
//   noise          explore::apply_noise (noise.hpp:56-72), bit-exact
#pragma once

#include <cstdint>

#include "rng.cuh"

namespace pqlg::actor {

constexpr int kEnvWarps = 8;
constexpr int kNormChunk = 128;

struct EnvState {
  float* s;                // [N x ld] state (= observation)
  int64_t ld;
  const float* M;          // [D x A] coupling
  int64_t* episode_step;   // [N]
  uint64_t* rng;           // [N] SplitMix state per env
  int N, D, A;
  int max_len;
  float low, high;
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

// One warp per env.  Lane-parallel over state dims; the order-sensitive sums
// (sum a^2, sum s'^2, the per-dim M a dot) are evaluated in the oracle's
// ascending order.  M is staged in shared memory (padded rows, float4
// loads) and the clamped action kept in registers.
constexpr int kMaxA = 32;
static __global__ void __launch_bounds__(32 * kEnvWarps)
    env_step_kernel(EnvState e, const float* __restrict__ act, int64_t ld_act, StepOut o,
                    NextNorm nn) {
  extern __shared__ float4 sh4[];
  const int Ap = (e.A + 3) & ~3;
  float* sM = reinterpret_cast<float*>(sh4);             // [D x Ap]
  float* sv_all = sM + static_cast<int64_t>(e.D) * Ap;  // [kEnvWarps][D]
  for (int j = threadIdx.x; j < e.D * Ap; j += blockDim.x) {
    const int d = j / Ap, k = j % Ap;
    sM[j] = k < e.A ? e.M[static_cast<int64_t>(d) * e.A + k] : 0.0f;
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * kEnvWarps + w;
  if (i >= e.N) return;
  float* sv = sv_all + w * e.D;
  const float* a_in = act + static_cast<int64_t>(i) * ld_act;
  float a[kMaxA];
  bool bad = false;
#pragma unroll
  for (int k = 0; k < kMaxA; ++k) {
    float u = 0.0f;
    if (k < e.A) {
      u = a_in[k];  // broadcast load (all lanes, same address)
      if (!isfinite(u)) bad = true;
      u = u < e.low ? e.low : (u > e.high ? e.high : u);
    }
    a[k] = u;
  }
  if (bad && lane == 0) atomicOr(o.status, 8u);
  float* s = e.s + static_cast<int64_t>(i) * e.ld;
  for (int d = lane; d < e.D; d += 32) {
    float ma = 0.0f;
    const float4* Mr = reinterpret_cast<const float4*>(sM + static_cast<int64_t>(d) * Ap);
#pragma unroll
    for (int k4 = 0; k4 < kMaxA / 4; ++k4) {
      if (4 * k4 < e.A) {
        const float4 m4 = Mr[k4];
        const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (4 * k4 + u < e.A) ma = __fadd_rn(ma, __fmul_rn(mm[u], a[4 * k4 + u]));
      }
    }
    float v = __fadd_rn(__fmul_rn(0.95f, s[d]), __fmul_rn(0.05f, ma));
    v = v < -10.0f ? -10.0f : (v > 10.0f ? 10.0f : v);
    sv[d] = v;
  }
  __syncwarp();
  // reward / termination / time limit (lane 0, ascending sums)
  int done_i = 0, trunc_i = 0;
  if (lane == 0) {
    float aa = 0.0f, ss = 0.0f;
#pragma unroll
    for (int k = 0; k < kMaxA; ++k)
      if (k < e.A) aa = __fadd_rn(aa, __fmul_rn(a[k], a[k]));
    int d = 0;
    for (; d + 8 <= e.D; d += 8) {
      float q[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) q[u] = sv[d + u];
#pragma unroll
      for (int u = 0; u < 8; ++u) ss = __fadd_rn(ss, __fmul_rn(q[u], q[u]));
    }
    for (; d < e.D; ++d) ss = __fadd_rn(ss, __fmul_rn(sv[d], sv[d]));
    const float reward = -__fadd_rn(__fdiv_rn(ss, static_cast<float>(e.D)),
                                    __fmul_rn(0.01f, __fdiv_rn(aa, static_cast<float>(e.A))));
    const bool terminal = fabsf(sv[0]) > 9.0f;
    const int64_t ep = e.episode_step[i] + 1;
    const bool timeout = ep >= e.max_len;
    done_i = terminal || timeout;
    trunc_i = !terminal && timeout;
    e.episode_step[i] = done_i ? 0 : ep;
    o.rew[i] = reward;
    o.term[i] = static_cast<uint8_t>(done_i && !trunc_i);
    o.trunc[i] = static_cast<uint8_t>(trunc_i);
    if (o.done) o.done[i] = static_cast<uint8_t>(done_i);
  }
  done_i = __shfl_sync(0xffffffffu, done_i, 0);
  const uint64_t st0 = e.rng[i];
  float* nxt = o.next_obs + static_cast<int64_t>(i) * o.ld_obs;
  float* bt = o.boot + static_cast<int64_t>(i) * o.ld_obs;
  const bool id = nn.out ? (*nn.identity != 0) : true;
  float* xn = nn.out ? nn.out + static_cast<int64_t>(i) * nn.ld_out : nullptr;
  for (int d = lane; d < e.D; d += 32) {
    const float v = sv[d];
    bt[d] = v;  // terminal observation on done, next observation otherwise
    float ns = v;
    if (done_i) {
      uint64_t st = st0 + static_cast<uint64_t>(d);  // draw d of the reset sequence
      ns = rng::env_uniform(st, -1.0f, 1.0f);
    }
    s[d] = ns;
    nxt[d] = ns;
    if (xn) {
      float z = ns;
      if (!id) {
        z = __fmul_rn(__fsub_rn(ns, nn.mean[d]), nn.inv[d]);
        if (z > 5.0f) z = 5.0f;
        if (z < -5.0f) z = -5.0f;
      }
      xn[d] = z;
    }
  }
  if (done_i && lane == 0) e.rng[i] = st0 + static_cast<uint64_t>(e.D);
}

inline size_t env_step_smem(int D, int A) {
  const int Ap = (A + 3) & ~3;
  return (static_cast<size_t>(D) * Ap + static_cast<size_t>(kEnvWarps) * D) * sizeof(float);
}

// reset_all (vecenv.cpp:53-60) + staggered episode_step = i % max_len.
static __global__ void env_reset_kernel(EnvState e, float* obs, int64_t ld_obs, int env_offset) {
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

// Batch moments, parallel and deterministic: warp lanes own columns, warps
// stride rows; sums are shifted by the batch's first row (no cancellation
// for offset data) and reduced in fixed order.  partial[(g*D + c)*2 + {0,1}]
// = (sum (x - x0), sum (x - x0)^2) over row group g.
constexpr int kNormGroups = 64;
static __global__ void __launch_bounds__(256)
    norm_partial_kernel(const float* __restrict__ x, int64_t ldx, int N, int D, double* partial) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int g = blockIdx.y;
  const int per = (N + gridDim.y - 1) / gridDim.y;
  const int r0 = g * per, r1 = min(r0 + per, N);
  double s1 = 0.0, s2 = 0.0;
  if (c < D) {
    const double shift = x[c];
    for (int r = r0 + w; r < r1; r += 8) {
      const double v = static_cast<double>(x[static_cast<int64_t>(r) * ldx + c]) - shift;
      s1 += v;
      s2 += v * v;
    }
  }
  __shared__ double red[8][32][2];
  red[w][lane][0] = s1;
  red[w][lane][1] = s2;
  __syncthreads();
  if (w == 0 && c < D) {
    double a = 0.0, b = 0.0;
    for (int k = 0; k < 8; ++k) {
      a += red[k][lane][0];
      b += red[k][lane][1];
    }
    partial[(static_cast<int64_t>(g) * D + c) * 2] = a;
    partial[(static_cast<int64_t>(g) * D + c) * 2 + 1] = b;
  }
}

struct NormState {
  int64_t* count;
  double* mean;
  double* m2;
  float* mean_f;
  float* inv_f;
  int* identity;
};

// Batch (mean, M2) from the partials (groups summed in order), then
// merge(bcount, bmean, bm2) into the running stats (normalizer.hpp:73-83)
// and the fp32 apply constants (normalizer.hpp:62-66).  One block, so the
// count update follows every column's read of it.
static __global__ void norm_finish_kernel(const float* __restrict__ x, const double* partial,
                                          int groups, int D, int64_t rows, NormState s) {
  const int64_t n0i = *s.count;
  const int64_t cnt = n0i + rows;
  const double nb = static_cast<double>(rows);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double s1 = 0.0, s2 = 0.0;
    for (int g = 0; g < groups; ++g) {
      s1 += partial[(static_cast<int64_t>(g) * D + d) * 2];
      s2 += partial[(static_cast<int64_t>(g) * D + d) * 2 + 1];
    }
    const double bmean = static_cast<double>(x[d]) + s1 / nb;
    double bm2 = s2 - s1 * s1 / nb;
    if (bm2 < 0.0) bm2 = 0.0;
    const double na = static_cast<double>(n0i);
    const double nab = na + nb;
    const double delta = bmean - s.mean[d];
    const double mean = s.mean[d] + delta * (nb / nab);
    const double m2 = s.m2[d] + (bm2 + delta * delta * (na * nb / nab));
    s.mean[d] = mean;
    s.m2[d] = m2;
    s.mean_f[d] = static_cast<float>(mean);
    s.inv_f[d] = static_cast<float>(1.0 / sqrt(m2 / static_cast<double>(cnt) + 1e-8));
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *s.count = cnt;
    *s.identity = cnt <= 1 ? 1 : 0;
  }
}

// Standalone apply_noise (op-level hook): one thread per env row.
static __global__ void noise_kernel(float* act, int64_t ld, int N, int A, const float* sigma,
                                    float low, float high, uint64_t* states) {
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
