// GEMM epilogues of the MLP layers.  Each thread of the 4 epilogue warps owns
// one output row (TMEM lane) and receives 32 consecutive accumulator columns
// per call, so row-wise heads (DDPG value dot, policy squash + exploration
// noise, C51 logits) fuse without a cross-thread reduction.
//
// Reference arithmetic they replace:
//   affine_forward bias add + relu          scalar.hpp:12-25, :57-60
//   DeterministicPolicy::act squash         policy.hpp:33-38
//   apply_noise (mixed exploration)         noise.hpp:56-72
//   relu_backward mask on the dgrad output  scalar.hpp:62-67, mlp.hpp:171-172
//   bias gradient column sums               scalar.hpp:48 (db[o] += g[b,o])
#pragma once

#include <cstdint>

#include "rng.cuh"

namespace pqlg::epi {

// relu(acc + b), stored; optional head dot  sum_n relu(.)*w_head[n]  per
// n-tile, written to partial[(group*n_tiles + n_tile)*ld_part + m].
struct Hidden {
  const float* bias[2];
  float* out[2];
  int64_t ld_out;
  const float* w_head[2];  // null: no head dot
  float* partial;
  int64_t ld_part;
  int n_tiles;
  int M, N;
  int store;  // 0: skip storing the activation (target critics)
  struct Row {
    float dot;
  };
  __device__ void begin(Row& r, int, int, int, int) const { r.dot = 0.0f; }
  __device__ void chunk(Row& r, int group, int, int m, int n0, const float (&v)[32]) const {
    if (m >= M) return;
    const float* b = bias[group];
    float* o = out[group] + static_cast<int64_t>(m) * ld_out;
    const float* wh = w_head[group];
    if (n0 + 32 <= N) {
      float x[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const float y = __fadd_rn(v[t], b[n0 + t]);
        x[t] = y > 0.0f ? y : 0.0f;
      }
      if (store) {
#pragma unroll
        for (int t = 0; t < 32; t += 4)
          *reinterpret_cast<float4*>(o + n0 + t) = make_float4(x[t], x[t + 1], x[t + 2], x[t + 3]);
      }
      if (wh) {
#pragma unroll
        for (int t = 0; t < 32; ++t) r.dot = __fadd_rn(r.dot, __fmul_rn(x[t], wh[n0 + t]));
      }
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int n = n0 + t;
        if (n < N) {
          const float y = __fadd_rn(v[t], b[n]);
          const float x = y > 0.0f ? y : 0.0f;
          if (store) o[n] = x;
          if (wh) r.dot = __fadd_rn(r.dot, __fmul_rn(x, wh[n]));
        }
      }
    }
  }
  __device__ void end(Row& r, int group, int, int m, int n_tile) const {
    if (m < M && w_head[group])
      partial[(static_cast<int64_t>(group) * n_tiles + n_tile) * ld_part + m] = r.dot;
  }
};

// Deterministic policy head (policy.hpp:33-38): y = acc + b (identity layer),
// a = mid + half*tanh(y) written to act[m*ld_act + n]; optionally the tanh
// values (for the backward, policy.hpp:41-51) and, for the actor, mixed
// exploration noise + clamp (noise.hpp:56-72) from the per-env SplitMix
// stream.  Noise draws consume columns in order n = 0..A-1, so the row state
// (stream position, cached polar value) persists across 32-column chunks.
struct PolicyHead {
  const float* bias;
  float* act;
  int64_t ld_act;
  float* tanh_out;  // nullable [M x A]
  int64_t ld_tanh;
  int M, A;
  float mid, half;
  // exploration (actor only)
  uint64_t* noise_state;  // nullable: per-env SplitMix state
  const float* sigma;     // per-env sigma_i
  float low, high;
  struct Row {
    uint64_t st;
    float saved;
    int has_saved;
    float sig;
  };
  __device__ void begin(Row& r, int, int, int m, int) const {
    r.has_saved = 0;
    r.saved = 0.0f;
    if (noise_state && m < M) {
      r.st = noise_state[m];
      r.sig = sigma[m];
    } else {
      r.st = 0;
      r.sig = 0.0f;
    }
  }
  __device__ void chunk(Row& r, int, int, int m, int n0, const float (&v)[32]) const {
    if (m >= M) return;
#pragma unroll 1
    for (int t = 0; t < 32; ++t) {
      const int n = n0 + t;
      if (n >= A) break;
      const float y = __fadd_rn(v[t], bias[n]);
      const float th = tanhf(y);
      float a = __fadd_rn(mid, __fmul_rn(half, th));
      if (tanh_out) tanh_out[static_cast<int64_t>(m) * ld_tanh + n] = th;
      if (noise_state) {
        if (r.sig > 0.0f) {
          float z;
          if (r.has_saved) {
            r.has_saved = 0;
            z = r.saved;
          } else {
            z = rng::polar_pair(r.st, r.saved);
            r.has_saved = 1;
          }
          a = __fadd_rn(a, __fadd_rn(__fmul_rn(z, r.sig), 0.0f));
        }
        if (a < low) a = low;
        if (a > high) a = high;
      }
      act[static_cast<int64_t>(m) * ld_act + n] = a;
    }
  }
  __device__ void end(Row& r, int, int, int m, int) const {
    if (noise_state && m < M) noise_state[m] = r.st;
  }
};

// dgrad output with the ReLU mask of the layer below (pre > 0 <=> post > 0),
// plus per-CTA column sums of the masked gradient (the bias gradient of that
// layer) written to colsum[(group*m_tiles + m_tile)*ld_cs + n].
struct DgradMask {
  const float* post[2];  // activation whose ReLU mask applies (nullable: no mask)
  int64_t ld_post;
  float* out[2];
  int64_t ld_out;
  float* colsum;  // nullable
  int64_t ld_cs;
  int m_tiles;
  int M, N;
  struct Row {};
  __device__ void begin(Row&, int, int, int, int) const {}
  __device__ void end(Row&, int, int, int, int) const {}
  __device__ void chunk(Row&, int group, int, int m, int n0, const float (&v)[32]) const {
    float g[32];
    const bool row_ok = m < M;
    if (row_ok) {
      const float* pp = post[group] ? post[group] + static_cast<int64_t>(m) * ld_post : nullptr;
      float* o = out[group] + static_cast<int64_t>(m) * ld_out;
#pragma unroll
      for (int t = 0; t < 32; ++t) {
        const int n = n0 + t;
        float x = v[t];
        if (n >= N) x = 0.0f;
        else if (pp && !(pp[n] > 0.0f)) x = 0.0f;
        g[t] = x;
      }
      if (n0 + 32 <= N) {
#pragma unroll
        for (int t = 0; t < 32; t += 4)
          *reinterpret_cast<float4*>(o + n0 + t) = make_float4(g[t], g[t + 1], g[t + 2], g[t + 3]);
      } else {
#pragma unroll
        for (int t = 0; t < 32; ++t)
          if (n0 + t < N) o[n0 + t] = g[t];
      }
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) g[t] = 0.0f;
    }
    if (!colsum) return;
    // Column sums over the 32 rows of this warp: recursive halving leaves
    // lane l with the sum of one column (fixed order -> deterministic).
    const int lane = threadIdx.x & 31;
#pragma unroll
    for (int w = 16; w >= 1; w >>= 1) {
      const bool upper = (lane & w) != 0;
#pragma unroll
      for (int t = 0; t < w; ++t) {
        const float send = upper ? g[t] : g[t + w];
        const float keep = upper ? g[t + w] : g[t];
        const float recv = __shfl_xor_sync(0xffffffffu, send, w);
        g[t] = __fadd_rn(keep, recv);
      }
    }
    // lane l now holds column c(l) where c is the bit-reversal-free mapping:
    // at each level the upper half of lanes kept the upper half of columns.
    const int col = n0 + lane;
    const int q = (threadIdx.x >> 5) & 3;  // TMEM lane quadrant of this warp
    // Cross-warp combine through shared memory in quadrant order.
    __shared__ float cs[4][32];
    cs[q][lane] = g[0];
    asm volatile("bar.sync 1, 128;" ::: "memory");
    if (q == 0 && col < N) {
      const float s = __fadd_rn(__fadd_rn(cs[0][lane], cs[1][lane]),
                                __fadd_rn(cs[2][lane], cs[3][lane]));
      const int m_tile = (m - lane) / 128;  // all rows of this CTA share the tile
      colsum[(static_cast<int64_t>(group) * m_tiles + m_tile) * ld_cs + col] = s;
    }
    asm volatile("bar.sync 1, 128;" ::: "memory");
  }
};

// Split-K partial tiles: W[((group*splits + split)*M + m)*N + n].
struct Partial {
  float* W;
  int splits;
  int M, N;
  struct Row {};
  __device__ void begin(Row&, int, int, int, int) const {}
  __device__ void end(Row&, int, int, int, int) const {}
  __device__ void chunk(Row&, int group, int split, int m, int n0, const float (&v)[32]) const {
    if (m >= M) return;
    float* d = W + ((static_cast<int64_t>(group) * splits + split) * M + m) * N;
    if (n0 + 32 <= N && (N & 3) == 0) {
#pragma unroll
      for (int t = 0; t < 32; t += 4)
        *reinterpret_cast<float4*>(d + n0 + t) = make_float4(v[t], v[t + 1], v[t + 2], v[t + 3]);
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t)
        if (n0 + t < N) d[n0 + t] = v[t];
    }
  }
};

// Raw store of the accumulator (identity layer without bias): din columns.
struct Store {
  float* out[2];
  int64_t ld_out;
  int M, N;
  struct Row {};
  __device__ void begin(Row&, int, int, int, int) const {}
  __device__ void end(Row&, int, int, int, int) const {}
  __device__ void chunk(Row&, int group, int, int m, int n0, const float (&v)[32]) const {
    if (m >= M) return;
    float* o = out[group] + static_cast<int64_t>(m) * ld_out;
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if (n0 + t < N) o[n0 + t] = v[t];
  }
};

}  // namespace pqlg::epi
