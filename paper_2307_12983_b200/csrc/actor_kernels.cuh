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

// Tiles of 32 envs per block iteration (persistent grid, M staged once per
// block in shared memory):
//   phase 1  warp per env: s' = clamp(0.95 s + 0.05 M a) lane-parallel over d,
//            up to 8 independent k-ascending chains per lane; s' -> smem tile
//   phase 2  thread per env (warp 0): the d-ascending sum of s'^2, reward,
//            termination, time limit -- the order-sensitive serial sums run
//            32 envs at a time instead of on one lane of a warp
//   phase 3  warp per env: boot obs, auto-reset draws, next obs, state and
//            the fused next-obs normalisation
// All sums are float mul/add in d-ascending order, so states, rewards and
// flags are bit-exact.
constexpr int kMaxA = 32;
constexpr int kEnvTile = 32;
constexpr int kMaxDChunks = 8;  // obs_dim <= 256

__device__ __forceinline__ int env_tile_ld(int D) { return D | 1; }  // odd: conflict-free rows

static __global__ void __launch_bounds__(32 * kEnvWarps)
    env_step_kernel(EnvState e, const float* __restrict__ act, int64_t ld_act, StepOut o,
                    NextNorm nn) {
  extern __shared__ float4 sh4[];
  const int D = e.D, A = e.A;
  const int Ap = (A + 3) & ~3;
  const int ldv = env_tile_ld(D);
  float* sM = reinterpret_cast<float*>(sh4);             // [D x Ap]
  float* sv = sM + static_cast<int64_t>(D) * Ap;        // [kEnvTile x ldv]  s'
  float* saa = sv + kEnvTile * ldv;                      // [kEnvTile]        sum a^2
  int* sdone = reinterpret_cast<int*>(saa + kEnvTile);   // [kEnvTile]
  for (int idx = threadIdx.x; idx < D * Ap; idx += blockDim.x) {
    const int d = idx / Ap, k = idx - d * Ap;
    sM[idx] = k < A ? e.M[static_cast<int64_t>(d) * A + k] : 0.0f;
  }
  __syncthreads();
  pdl::entry();  // M is constant: staged while the previous kernel drains
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int nch = (D + 31) >> 5;
  const bool id = nn.out ? (*nn.identity != 0) : true;
  const int n_tiles = (e.N + kEnvTile - 1) / kEnvTile;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int i0 = tile * kEnvTile;
    // ---- phase 1
    for (int j = w; j < kEnvTile && i0 + j < e.N; j += kEnvWarps) {
      const int i = i0 + j;
      const float* s = e.s + static_cast<int64_t>(i) * e.ld;
      float sd[kMaxDChunks];
#pragma unroll
      for (int c = 0; c < kMaxDChunks; ++c) {
        const int d = lane + 32 * c;
        sd[c] = (c < nch && d < D) ? s[d] : 0.0f;
      }
      const float* a_in = act + static_cast<int64_t>(i) * ld_act;
      float a[kMaxA];
      bool bad = false;
#pragma unroll
      for (int k = 0; k < kMaxA; ++k) {
        float u = 0.0f;
        if (k < A) {
          u = a_in[k];  // broadcast load
          if (!isfinite(u)) bad = true;
          u = u < e.low ? e.low : (u > e.high ? e.high : u);
        }
        a[k] = u;
      }
      if (bad && lane == 0) atomicOr(o.status, 8u);
      float acc[kMaxDChunks];
#pragma unroll
      for (int c = 0; c < kMaxDChunks; ++c) acc[c] = 0.0f;
#pragma unroll
      for (int k4 = 0; k4 < kMaxA / 4; ++k4) {
        if (4 * k4 < A) {
#pragma unroll
          for (int c = 0; c < kMaxDChunks; ++c) {
            const int d = lane + 32 * c;
            if (c < nch && d < D) {
              const float4 m4 = reinterpret_cast<const float4*>(sM + d * Ap)[k4];
              const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
              for (int u = 0; u < 4; ++u)
                if (4 * k4 + u < A) acc[c] = __fadd_rn(acc[c], __fmul_rn(mm[u], a[4 * k4 + u]));
            }
          }
        }
      }
#pragma unroll
      for (int c = 0; c < kMaxDChunks; ++c) {
        const int d = lane + 32 * c;
        if (c < nch && d < D) {
          float v = __fadd_rn(__fmul_rn(0.95f, sd[c]), __fmul_rn(0.05f, acc[c]));
          v = v < -10.0f ? -10.0f : (v > 10.0f ? 10.0f : v);
          sv[j * ldv + d] = v;
        }
      }
      if (lane == 0) {
        float aa = 0.0f;
#pragma unroll
        for (int k = 0; k < kMaxA; ++k)
          if (k < A) aa = __fadd_rn(aa, __fmul_rn(a[k], a[k]));
        saa[j] = aa;
      }
    }
    __syncthreads();
    // ---- phase 2
    if (w == 0) {
      const int i = i0 + lane;
      int done_i = 0;
      if (i < e.N) {
        const float* row = sv + lane * ldv;
        float ss = 0.0f;
        int d = 0;
        for (; d + 8 <= D; d += 8) {
          float q[8];
#pragma unroll
          for (int u = 0; u < 8; ++u) q[u] = row[d + u];
#pragma unroll
          for (int u = 0; u < 8; ++u) ss = __fadd_rn(ss, __fmul_rn(q[u], q[u]));
        }
        for (; d < D; ++d) ss = __fadd_rn(ss, __fmul_rn(row[d], row[d]));
        const float reward = -__fadd_rn(__fdiv_rn(ss, static_cast<float>(D)),
                                        __fmul_rn(0.01f, __fdiv_rn(saa[lane], static_cast<float>(A))));
        const bool terminal = fabsf(row[0]) > 9.0f;
        const int64_t ep = e.episode_step[i] + 1;
        const bool timeout = ep >= e.max_len;
        done_i = terminal || timeout;
        const int trunc_i = !terminal && timeout;
        e.episode_step[i] = done_i ? 0 : ep;
        o.rew[i] = reward;
        o.term[i] = static_cast<uint8_t>(done_i && !trunc_i);
        o.trunc[i] = static_cast<uint8_t>(trunc_i);
        if (o.done) o.done[i] = static_cast<uint8_t>(done_i);
      }
      sdone[lane] = done_i;
    }
    __syncthreads();
    // ---- phase 3
    for (int j = w; j < kEnvTile && i0 + j < e.N; j += kEnvWarps) {
      const int i = i0 + j;
      const int done_i = sdone[j];
      const uint64_t st0 = e.rng[i];
      float* s = e.s + static_cast<int64_t>(i) * e.ld;
      float* nxt = o.next_obs + static_cast<int64_t>(i) * o.ld_obs;
      float* bt = o.boot + static_cast<int64_t>(i) * o.ld_obs;
      float* xn = nn.out ? nn.out + static_cast<int64_t>(i) * nn.ld_out : nullptr;
      for (int d = lane; d < D; d += 32) {
        const float v = sv[j * ldv + d];
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
      if (done_i && lane == 0) e.rng[i] = st0 + static_cast<uint64_t>(D);
    }
    // the next tile's phase 1 writes only rows owned by the same warp; saa /
    // sdone are rewritten after the next barrier
  }
}

inline size_t env_step_smem(int D, int A) {
  const int Ap = (A + 3) & ~3;
  return (static_cast<size_t>(D) * Ap + static_cast<size_t>(kEnvTile) * (D | 1) + 2 * kEnvTile) *
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

struct NormState {
  int64_t* count;
  double* mean;
  double* m2;
  float* mean_f;
  float* inv_f;
  int* identity;
};

// RunningNormalizer::update (normalizer.hpp:33-50, :73-83) in one launch,
// parallel and deterministic.  Grid (ceil(D/32), kNormGroups): warp lanes own
// columns, warps stride the group's rows; sums are shifted by the batch's
// first row (no cancellation for offset data).  The last block to finish
// (atomic ticket) reduces the group partials per column in fixed order
// (lane-strided sums + xor butterfly), forms the batch (mean, M2), merges it
// into the running stats with Chan's formula and refreshes the fp32 apply
// constants (normalizer.hpp:62-66).
constexpr int kNormGroups = 64;
static __global__ void __launch_bounds__(256)
    norm_update_kernel(const float* __restrict__ x, int64_t ldx, int N, int D, double* partial,
                       unsigned int* ticket, NormState s) {
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int c = blockIdx.x * 32 + lane;
  const int g = blockIdx.y;
  const int per = (N + gridDim.y - 1) / gridDim.y;
  const int r0 = g * per, r1 = min(r0 + per, N);
  double s1 = 0.0, s2 = 0.0;
  if (c < D) {
    const double shift = x[c];
    int r = r0 + w;
    for (; r + 24 < r1; r += 32) {
      float v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) v[u] = x[static_cast<int64_t>(r + 8 * u) * ldx + c];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double t = static_cast<double>(v[u]) - shift;
        s1 += t;
        s2 += t * t;
      }
    }
    for (; r < r1; r += 8) {
      const double t = static_cast<double>(x[static_cast<int64_t>(r) * ldx + c]) - shift;
      s1 += t;
      s2 += t * t;
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
  __shared__ bool last;
  __threadfence();
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(ticket, 1u) == gridDim.x * gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  const int64_t n0i = *s.count;
  const int64_t cnt = n0i + N;
  const double nb = static_cast<double>(N);
  const double na = static_cast<double>(n0i);
  const double nab = na + nb;
  const int groups = gridDim.y;
  for (int d = w; d < D; d += blockDim.x / 32) {
    double s1 = 0.0, s2 = 0.0;
    for (int k = lane; k < groups; k += 32) {
      s1 += __ldcg(partial + (static_cast<int64_t>(k) * D + d) * 2);
      s2 += __ldcg(partial + (static_cast<int64_t>(k) * D + d) * 2 + 1);
    }
#pragma unroll
    for (int o = 16; o >= 1; o >>= 1) {
      s1 += __shfl_xor_sync(0xffffffffu, s1, o);
      s2 += __shfl_xor_sync(0xffffffffu, s2, o);
    }
    if (lane == 0) {
      const double bmean = static_cast<double>(x[d]) + s1 / nb;
      double bm2 = s2 - s1 * s1 / nb;
      if (bm2 < 0.0) bm2 = 0.0;
      const double delta = bmean - s.mean[d];
      const double mean = s.mean[d] + delta * (nb / nab);
      const double m2 = s.m2[d] + (bm2 + delta * delta * (na * nb / nab));
      s.mean[d] = mean;
      s.m2[d] = m2;
      s.mean_f[d] = static_cast<float>(mean);
      s.inv_f[d] = static_cast<float>(1.0 / sqrt(m2 / static_cast<double>(cnt) + 1e-8));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    *s.count = cnt;
    *s.identity = cnt <= 1 ? 1 : 0;
    *ticket = 0u;
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
