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
  float* s;                // [N x ld] state (= observation); null: the caller keeps the
  int64_t ld;              //   state in its obs buffers (s_in = this step's obs)
  const float* s_in;       // state read by the step (= s unless aliased)
  int64_t ld_in;
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

// kNch = number of 32-wide obs chunks per lane (ceil(D/32) rounded up to 1, 2, 4 or 8).
template <int kNch>
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
  float* sa_all = saa + 2 * kEnvTile;                    // [kEnvWarps x kPer x 32] clamped actions
  {
    // stage M (constant since env creation) before the PDL wait, under the
    // previous kernel's tail
    if ((A & 3) == 0) {  // rows are float4-aligned: straight vector copy
      const int total4 = D * A / 4;
      const float4* src = reinterpret_cast<const float4*>(e.M);
      for (int idx = threadIdx.x; idx < total4; idx += blockDim.x) sh4[idx] = src[idx];
    } else {
      const int total = D * Ap;
      for (int base = threadIdx.x; base < total; base += 8 * blockDim.x) {
        float v[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = base + q * blockDim.x;
          v[q] = 0.0f;
          if (idx < total) {
            const int d = idx / Ap, k = idx - d * Ap;
            if (k < A) v[q] = e.M[static_cast<int64_t>(d) * A + k];
          }
        }
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int idx = base + q * blockDim.x;
          if (idx < total) sM[idx] = v[q];
        }
      }
    }
  }
  __syncthreads();
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  constexpr int kPerW = kEnvTile / kEnvWarps;
  float* sa = sa_all + w * 32 * kPerW;
  const bool id = nn.out ? (*nn.identity != 0) : true;
  const int n_tiles = (e.N + kEnvTile - 1) / kEnvTile;
  const int A4 = (A + 3) >> 2;
  for (int tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    const int i0 = tile * kEnvTile;
    // ---- phase 1 (all of this warp's env rows are loaded before any math)
    constexpr int kPer = kEnvTile / kEnvWarps;
    float sdp[kPer][kNch], up[kPer];
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
      const int i = i0 + w + p * kEnvWarps;
      const bool ok = i < e.N;
      const float* s = e.s_in + static_cast<int64_t>(i) * e.ld_in;
#pragma unroll
      for (int c = 0; c < kNch; ++c) {
        const int d = lane + 32 * c;
        sdp[p][c] = (ok && d < D) ? s[d] : 0.0f;
      }
      up[p] = (ok && lane < A) ? act[static_cast<int64_t>(i) * ld_act + lane] : 0.0f;
    }
    // clamped actions of the warp's kPer envs -> smem (one row of 32 each)
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
      const int i = i0 + w + p * kEnvWarps;
      float u = 0.0f;
      bool bad = false;
      if (lane < A && i < e.N) {
        u = up[p];
        bad = !isfinite(u);
        u = u < e.low ? e.low : (u > e.high ? e.high : u);
      }
      sa[p * 32 + lane] = u;
      if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(o.status, 8u);
    }
    __syncwarp();
    // M a for all kPer envs at once: each M quad read from smem feeds kPer
    // independent k-ascending chains per d (mul then add, no FMA)
    float acc[kPer][kNch];
#pragma unroll
    for (int p = 0; p < kPer; ++p)
#pragma unroll
      for (int c = 0; c < kNch; ++c) acc[p][c] = 0.0f;
#pragma unroll 1
    for (int k4 = 0; k4 < A4; ++k4) {
      float av[kPer][4];
#pragma unroll
      for (int p = 0; p < kPer; ++p) {
        const float4 a4 = reinterpret_cast<const float4*>(sa + p * 32)[k4];
        av[p][0] = a4.x;
        av[p][1] = a4.y;
        av[p][2] = a4.z;
        av[p][3] = a4.w;
      }
      const int nu = A - 4 * k4;
      if (nu >= 4) {  // full quad (always when A % 4 == 0)
#pragma unroll
        for (int c = 0; c < kNch; ++c) {
          const int d = lane + 32 * c;
          if (c + 1 < kNch || d < D) {
            const float4 m4 = reinterpret_cast<const float4*>(sM + d * Ap)[k4];
#pragma unroll
            for (int p = 0; p < kPer; ++p) {
              acc[p][c] = __fadd_rn(acc[p][c], __fmul_rn(m4.x, av[p][0]));
              acc[p][c] = __fadd_rn(acc[p][c], __fmul_rn(m4.y, av[p][1]));
              acc[p][c] = __fadd_rn(acc[p][c], __fmul_rn(m4.z, av[p][2]));
              acc[p][c] = __fadd_rn(acc[p][c], __fmul_rn(m4.w, av[p][3]));
            }
          }
        }
      } else {
#pragma unroll
        for (int c = 0; c < kNch; ++c) {
          const int d = lane + 32 * c;
          if (d < D) {
            const float4 m4 = reinterpret_cast<const float4*>(sM + d * Ap)[k4];
            const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
            for (int p = 0; p < kPer; ++p)
#pragma unroll
              for (int q = 0; q < 4; ++q)
                if (q < nu) acc[p][c] = __fadd_rn(acc[p][c], __fmul_rn(mm[q], av[p][q]));
          }
        }
      }
    }
#pragma unroll
    for (int p = 0; p < kPer; ++p) {
      const int j = w + p * kEnvWarps;
      if (i0 + j >= e.N) break;
#pragma unroll
      for (int c = 0; c < kNch; ++c) {
        const int d = lane + 32 * c;
        if (d < D) {
          float v = __fadd_rn(__fmul_rn(0.95f, sdp[p][c]), __fmul_rn(0.05f, acc[p][c]));
          v = v < -10.0f ? -10.0f : (v > 10.0f ? 10.0f : v);
          sv[j * ldv + d] = v;
        }
      }
      if (lane == 0) {
        const float* ap = sa + p * 32;
        float aa = 0.0f;
        for (int k = 0; k < A; ++k) aa = __fadd_rn(aa, __fmul_rn(ap[k], ap[k]));
        saa[j] = aa;
      }
    }
    __syncwarp();
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
          for (int t = 0; t < 8; ++t) q[t] = row[d + t];
#pragma unroll
          for (int t = 0; t < 8; ++t) ss = __fadd_rn(ss, __fmul_rn(q[t], q[t]));
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
    float nm[kNch], ni[kNch];  // this lane's normalisation constants (d = lane + 32c)
#pragma unroll
    for (int c = 0; c < kNch; ++c) {
      const int d = lane + 32 * c;
      nm[c] = (nn.out && !id && d < D) ? nn.mean[d] : 0.0f;
      ni[c] = (nn.out && !id && d < D) ? nn.inv[d] : 1.0f;
    }
    for (int j = w; j < kEnvTile && i0 + j < e.N; j += kEnvWarps) {
      const int i = i0 + j;
      float* s = e.s ? e.s + static_cast<int64_t>(i) * e.ld : nullptr;
      float* nxt = o.next_obs + static_cast<int64_t>(i) * o.ld_obs;
      float* bt = o.boot + static_cast<int64_t>(i) * o.ld_obs;
      float* xn = nn.out ? nn.out + static_cast<int64_t>(i) * nn.ld_out : nullptr;
      auto emit = [&](int d, int c, float ns) {
        if (s) s[d] = ns;
        nxt[d] = ns;
        if (xn) {
          float z = ns;
          if (!id) {
            z = __fmul_rn(__fsub_rn(ns, nm[c]), ni[c]);
            if (z > 5.0f) z = 5.0f;
            if (z < -5.0f) z = -5.0f;
          }
          xn[d] = z;
        }
      };
      if (sdone[j]) {  // warp-uniform: terminal obs to boot, fresh reset draws
        const uint64_t st0 = e.rng[i];
#pragma unroll
        for (int c = 0; c < kNch; ++c) {
          const int d = lane + 32 * c;
          if (d < D) {
            bt[d] = sv[j * ldv + d];
            uint64_t st = st0 + static_cast<uint64_t>(d);  // draw d of the reset sequence
            emit(d, c, rng::env_uniform(st, -1.0f, 1.0f));
          }
        }
        if (lane == 0) e.rng[i] = st0 + static_cast<uint64_t>(D);
      } else {
#pragma unroll
        for (int c = 0; c < kNch; ++c) {
          const int d = lane + 32 * c;
          if (d < D) {
            const float v = sv[j * ldv + d];
            bt[d] = v;
            emit(d, c, v);
          }
        }
      }
    }
    // the next tile's phase 1 writes only rows owned by the same warp; saa /
    // sdone are rewritten after the next barrier
  }
}

inline size_t env_step_smem(int D, int A) {
  const int Ap = (A + 3) & ~3;
  return (static_cast<size_t>(D) * Ap + static_cast<size_t>(kEnvTile) * (D | 1) + 2 * kEnvTile +
          32 * kEnvTile) *
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
  // sharded actor: non-null -> the batch's (mean [D], M2 [D], n) are written
  // here instead of being merged (norm_merge_kernel merges every shard's)
  double* batch;
};

// Chan's parallel merge of (na, mean_a, m2_a) with a batch (nb, mean_b, m2_b)
// (normalizer.hpp:73-83), fp64, in the reference's operation order.
__device__ __forceinline__ void chan_merge(double na, double& mean, double& m2, double nb,
                                           double bmean, double bm2) {
  const double nab = na + nb;
  const double delta = bmean - mean;
  mean = mean + delta * (nb / nab);
  m2 = m2 + (bm2 + delta * delta * (na * nb / nab));
}

// RunningNormalizer::update (normalizer.hpp:33-50, :73-83) in one launch,
// parallel and deterministic.  Grid (ceil(D/32) column strips, kNormGroups
// row groups), 8 warps: lanes own columns, warp w sums rows r0 + w + 8t of
// its group with all loads in flight; sums are shifted by the batch's first
// row (no cancellation for offset data).  The last block of each column strip
// (atomic ticket) reduces that strip's group partials in fixed order (8
// threads per column, then the 8 parts in order), forms the batch (mean, M2),
// merges it into the running stats with Chan's formula and refreshes the
// fp32 apply constants (normalizer.hpp:62-66); the last strip to finish
// advances the count.
constexpr int kNormGroups = 128;  // upper bound (partials buffer)
// row groups so the (strips x groups) grid is one wave at 4 blocks per SM
inline int norm_groups(int D) {
  const int strips = (D + 31) / 32;
  int g = 4 * 148 / strips;
  if (g > kNormGroups) g = kNormGroups;
  if (g < 1) g = 1;
  return g;
}
constexpr int kNormRowsPerWarp = 16;  // rows per warp per group (N <= 8*16*kNormGroups in one pass)
static __global__ void __launch_bounds__(256, 4)
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
    for (int rb = r0 + w; rb < r1; rb += 8 * kNormRowsPerWarp) {
      float v[kNormRowsPerWarp];
#pragma unroll
      for (int u = 0; u < kNormRowsPerWarp; ++u) {
        const int r = rb + 8 * u;
        v[u] = r < r1 ? x[static_cast<int64_t>(r) * ldx + c] : 0.0f;
      }
#pragma unroll
      for (int u = 0; u < kNormRowsPerWarp; ++u) {
        if (rb + 8 * u < r1) {
          const double t = static_cast<double>(v[u]) - shift;
          s1 += t;
          s2 += t * t;
        }
      }
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
  if (w == 0) __threadfence();  // only warp 0 wrote partials
  __syncthreads();
  if (threadIdx.x == 0) last = atomicAdd(&ticket[1 + blockIdx.x], 1u) == gridDim.y - 1;
  __syncthreads();
  if (!last) return;
  __threadfence();
  // strip finish: thread (column lane, part w) sums groups w, w+8, ... in order
  const int groups = gridDim.y;
  {
    double a1 = 0.0, a2 = 0.0;
    if (c < D) {
      constexpr int kIn = 4;
      for (int k0 = w; k0 < groups; k0 += 8 * kIn) {
        double v1[kIn], v2[kIn];
#pragma unroll
        for (int q = 0; q < kIn; ++q) {
          const int k = k0 + 8 * q;
          const double* src = partial + (static_cast<int64_t>(k) * D + c) * 2;
          v1[q] = k < groups ? __ldcg(src) : 0.0;
          v2[q] = k < groups ? __ldcg(src + 1) : 0.0;
        }
#pragma unroll
        for (int q = 0; q < kIn; ++q) {
          a1 += v1[q];
          a2 += v2[q];
        }
      }
    }
    __syncthreads();  // red reuse
    red[w][lane][0] = a1;
    red[w][lane][1] = a2;
  }
  __syncthreads();
  const int64_t n0i = s.batch ? 0 : *s.count;
  if (w == 0 && c < D) {
    const double nb = static_cast<double>(N);
    const double na = static_cast<double>(n0i);
    const int64_t cnt = n0i + N;
    double t1 = 0.0, t2 = 0.0;
    for (int k = 0; k < 8; ++k) {
      t1 += red[k][lane][0];
      t2 += red[k][lane][1];
    }
    const double bmean = static_cast<double>(x[c]) + t1 / nb;
    double bm2 = t2 - t1 * t1 / nb;
    if (bm2 < 0.0) bm2 = 0.0;
    if (s.batch) {
      s.batch[c] = bmean;
      s.batch[D + c] = bm2;
    } else {
      double mean = s.mean[c], m2 = s.m2[c];
      chan_merge(na, mean, m2, nb, bmean, bm2);
      s.mean[c] = mean;
      s.m2[c] = m2;
      s.mean_f[c] = static_cast<float>(mean);
      s.inv_f[c] = static_cast<float>(1.0 / sqrt(m2 / static_cast<double>(cnt) + 1e-8));
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    ticket[1 + blockIdx.x] = 0u;
    __threadfence();
    // every strip read the old count before its ticket: the last one advances it
    if (atomicAdd(&ticket[0], 1u) == gridDim.x - 1) {
      if (s.batch) {
        s.batch[2 * D] = static_cast<double>(N);
      } else {
        *s.count = n0i + N;
        *s.identity = n0i + N <= 1 ? 1 : 0;
      }
      ticket[0] = 0u;
    }
  }
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

inline int norm_tickets(int D) { return 1 + (D + 31) / 32; }

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
