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

// One warp per env.  Lane-parallel over state dims; the order-sensitive sums
// (sum a^2, sum s'^2, the per-dim M a dot) are evaluated in the oracle's
// ascending order.
static __global__ void env_step_kernel(EnvState e, const float* __restrict__ act, int64_t ld_act,
                                       StepOut o) {
  extern __shared__ float sh[];  // [kEnvWarps][D + A]
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int i = blockIdx.x * kEnvWarps + w;
  if (i >= e.N) return;
  float* sa = sh + w * (e.D + e.A);
  float* sv = sa + e.A;
  const float* a_in = act + static_cast<int64_t>(i) * ld_act;
  bool bad = false;
  for (int k = lane; k < e.A; k += 32) {
    float u = a_in[k];
    if (!isfinite(u)) bad = true;
    u = u < e.low ? e.low : (u > e.high ? e.high : u);
    sa[k] = u;
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(o.status, 8u);
  __syncwarp();
  float* s = e.s + static_cast<int64_t>(i) * e.ld;
  for (int d = lane; d < e.D; d += 32) {
    float ma = 0.0f;
    const float* Mr = e.M + static_cast<int64_t>(d) * e.A;
    for (int k = 0; k < e.A; ++k) ma = __fadd_rn(ma, __fmul_rn(Mr[k], sa[k]));
    float v = __fadd_rn(__fmul_rn(0.95f, s[d]), __fmul_rn(0.05f, ma));
    v = v < -10.0f ? -10.0f : (v > 10.0f ? 10.0f : v);
    sv[d] = v;
  }
  __syncwarp();
  // reward / termination / time limit (lane 0, ascending sums)
  int done_i = 0, trunc_i = 0;
  if (lane == 0) {
    float aa = 0.0f, ss = 0.0f;
    for (int k = 0; k < e.A; ++k) aa = __fadd_rn(aa, __fmul_rn(sa[k], sa[k]));
    for (int d = 0; d < e.D; ++d) ss = __fadd_rn(ss, __fmul_rn(sv[d], sv[d]));
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
  }
  if (done_i && lane == 0) e.rng[i] = st0 + static_cast<uint64_t>(e.D);
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

// Welford over one chunk of rows (row order) for all columns: thread = column.
static __global__ void norm_chunk_kernel(const float* __restrict__ x, int64_t ldx, int N, int D,
                                         double* cmean, double* cm2, double* ccount) {
  const int chunk = blockIdx.x;
  const int r0 = chunk * kNormChunk, r1 = min(r0 + kNormChunk, N);
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double mean = 0.0, m2 = 0.0, n = 0.0;
    for (int r = r0; r < r1; ++r) {
      n += 1.0;
      const double v = x[static_cast<int64_t>(r) * ldx + d];
      const double delta = v - mean;
      mean += delta / n;
      m2 += delta * (v - mean);
    }
    cmean[static_cast<int64_t>(chunk) * D + d] = mean;
    cm2[static_cast<int64_t>(chunk) * D + d] = m2;
    if (d == 0) ccount[chunk] = n;
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

// Chan merge of the chunk statistics (left fold in chunk order) and of the
// batch into the running stats; then the fp32 apply constants.  Launched as
// one block so the count update follows every column's read of it.
static __global__ void norm_merge_kernel(const double* cmean, const double* cm2,
                                         const double* ccount, int chunks, int D, int64_t rows,
                                         NormState s) {
  const int64_t n0i = *s.count;
  const int64_t cnt = n0i + rows;
  for (int d = threadIdx.x; d < D; d += blockDim.x) {
    double na = ccount[0], ma = cmean[d], m2a = cm2[d];
    for (int c = 1; c < chunks; ++c) {
      const double nb = ccount[c], mb = cmean[static_cast<int64_t>(c) * D + d],
                   m2b = cm2[static_cast<int64_t>(c) * D + d];
      const double nab = na + nb;
      const double delta = mb - ma;
      ma += delta * (nb / nab);
      m2a += m2b + delta * delta * (na * nb / nab);
      na = nab;
    }
    // merge(bcount, bmean, bm2) into the running stats (normalizer.hpp:73-83)
    const double n0 = static_cast<double>(n0i);
    const double nab = n0 + na;
    const double delta = ma - s.mean[d];
    const double mean = s.mean[d] + delta * (na / nab);
    const double m2 = s.m2[d] + (m2a + delta * delta * (n0 * na / nab));
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
