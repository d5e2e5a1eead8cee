// GEMM epilogues of the MLP layers.  Each thread of the 4 epilogue warps owns
// one output row (TMEM lane) and receives 32 consecutive accumulator columns
// per call, so row-wise heads (DDPG value dot, policy squash + exploration
// noise) fuse without a cross-thread reduction.  Per-tile constants (bias,
// head weights, ReLU masks) are preloaded in prepare() while the mainloop
// runs; results leave through 128B-swizzled smem + TMA stores
// (kStoreRank > 0) or direct stores for narrow heads.
//
// Reference arithmetic they replace:
//   affine_forward bias add + relu          scalar.hpp:12-25, :57-60
//   DeterministicPolicy::act squash         policy.hpp:33-38
//   apply_noise (mixed exploration)         noise.hpp:56-72
//   relu_backward mask on the dgrad output  scalar.hpp:62-67, mlp.hpp:171-172
//   bias gradient column sums               scalar.hpp:48 (db[o] += g[b,o])
#pragma once

#include <cstdint>

#include "ptx.cuh"
#include "rng.cuh"

namespace pqlg::epi {

// Where an epilogue thread is: its tile, its row, and how the tile's columns
// are shared between the epilogue warps (halves == 2: two warps per row,
// warp `half` takes columns [half*BN/2, (half+1)*BN/2)).
struct Ctx {
  int group, split, m_tile, n_tile;
  int m;     // this thread's row
  int row0;  // first row of the warp's 32-row slab
  int et;    // epilogue thread index in [0, ne)
  int ne;    // epilogue threads
  int half, halves;
};

// relu(acc + b) -> TMA store (store = 1) and/or a ReLU bitmask (bit t of
// word n/32 = post[m, n] > 0) used by the backward, stored word-major
// (mask[(n/32) * ld_mask + m]: a warp's 32 rows write one coalesced 128 B
// line per word); optional head dot sum_n relu(.)*w_head[n] per 64-column
// block (min(64, bn) columns; independent of how the epilogue warps split
// the tile) -> partial[group][(n / unit) * ld_part + m].
struct Hidden {
  static constexpr int kStoreRank = 2;
  static constexpr bool kSplitCols = true;
  const float* bias[4];
  const float* w_head[4];  // null: no head dot
  uint32_t* mask[4];       // null: no bitmask
  int ld_mask;             // word-major: stride between words (>= M rows)
  float* partial[4];       // per group [slot][ld_part], slot = n / min(64, bn)
  int64_t ld_part;
  int n_slots;             // ceil(N / min(64, bn)) (mlp::hidden_slots)
  int bn;
  int M, N;
  int store;  // bit g: store group g's activation (0 for the target critics' last layer)
  struct Row {
    float dot;
  };
  __device__ void prepare(Row& r, const Ctx& c, float* scratch) const {
    r.dot = 0.0f;
    const float* b = bias[c.group];
    const float* wh = w_head[c.group];
    for (int i = c.et; i < bn; i += c.ne) {
      const int n = c.n_tile * bn + i;
      scratch[i] = n < N ? b[n] : 0.0f;
      if (wh) scratch[bn + i] = n < N ? wh[n] : 0.0f;
    }
  }
  __device__ bool chunk(Row& r, const Ctx& c, int n0, float (&v)[32], float* scratch) const {
    const int c0 = n0 % bn;
    uint32_t bits = 0;
#pragma unroll
    for (int t = 0; t < 32; t += 4) {
      const float4 b4 = *reinterpret_cast<const float4*>(scratch + c0 + t);
      const float bb[4] = {b4.x, b4.y, b4.z, b4.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float y = __fadd_rn(v[t + u], bb[u]);
        const float x = y > 0.0f ? y : 0.0f;
        v[t + u] = x;
        bits |= (x > 0.0f ? 1u : 0u) << (t + u);
      }
    }
    if (w_head[c.group]) {
#pragma unroll
      for (int t = 0; t < 32; ++t) r.dot = __fadd_rn(r.dot, __fmul_rn(v[t], scratch[bn + c0 + t]));
      // a 64-column block (or the tile / matrix edge) is complete: one slot
      const int unit = bn < 64 ? bn : 64;
      if ((c0 + 32) % unit == 0 || n0 + 32 >= N) {
        if (c.m < M) partial[c.group][static_cast<int64_t>(n0 / unit) * ld_part + c.m] = r.dot;
        r.dot = 0.0f;
      }
    }
    if (mask[c.group] && c.m < M)
      mask[c.group][static_cast<int64_t>(n0 >> 5) * ld_mask + c.m] = bits;
    return ((store >> c.group) & 1) != 0;
  }
  __device__ void end(Row&, const Ctx&) const {}
};

// Deterministic policy head (policy.hpp:33-38): y = acc + b (identity layer),
// a = mid + half*tanh(y) written to act[m*ld_act + n]; optionally the tanh
// values (for the backward, policy.hpp:41-51) and, for the actor, mixed
// exploration noise + clamp (noise.hpp:56-72) from the per-env SplitMix
// stream.  Noise draws consume columns in order n = 0..A-1, so the row state
// (stream position, cached polar value) persists across 32-column chunks.
struct PolicyHead {
  static constexpr int kStoreRank = 0;
  static constexpr bool kSplitCols = false;
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
  // The normal draws depend only on the env's stream (not on the action
  // values), so prepare() generates all A of them while the mainloop runs
  // (A <= 32, one 32-column chunk); chunk() only squashes, adds and clamps.
  struct Row {
    float z[32];
    float sig;
  };
  __device__ void prepare(Row& r, const Ctx& c, float* scratch) const {
    const int m = c.m;
    for (int i = c.et; i < A; i += c.ne) scratch[i] = bias[i];
    r.sig = 0.0f;
    if (noise_state && m < M) {
      r.sig = sigma[m];
      if (r.sig > 0.0f) {
        uint64_t st = noise_state[m];
        float saved = 0.0f;
#pragma unroll
        for (int d = 0; d < 32; d += 2) {
          if (d < A) {
            r.z[d] = rng::polar_pair(st, saved);  // y*mult first, x*mult cached
            r.z[d + 1] = saved;
          }
        }
        noise_state[m] = st;
      }
    }
  }
  __device__ bool chunk(Row& r, const Ctx& c, int n0, float (&v)[32], float* scratch) const {
    const int m = c.m;
    if (m >= M) return false;
    float* out = act + static_cast<int64_t>(m) * ld_act;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      const int n = n0 + t;
      if (n < A) {
        const float y = __fadd_rn(v[t], scratch[n]);
        const float th = tanhf(y);
        float a = __fadd_rn(mid, __fmul_rn(half, th));
        if (tanh_out) tanh_out[static_cast<int64_t>(m) * ld_tanh + n] = th;
        if (noise_state) {
          if (r.sig > 0.0f) a = __fadd_rn(a, __fadd_rn(__fmul_rn(r.z[t], r.sig), 0.0f));
          if (a < low) a = low;
          if (a > high) a = high;
        }
        out[n] = a;
      }
    }
    return false;
  }
  __device__ void end(Row&, const Ctx&) const {}
};

// dgrad output with the ReLU mask of the layer below (from its bitmask),
// TMA-stored, plus per-CTA column sums of the masked gradient (the bias
// gradient of that layer) written to colsum[(group*m_tiles + m_tile)*ld_cs + n].
struct DgradMask {
  static constexpr int kStoreRank = 2;
  static constexpr bool kSplitCols = true;
  const uint32_t* mask[2];  // nullable: no mask (word-major, as Hidden writes it)
  int ld_mask;
  float* colsum;  // nullable
  int64_t ld_cs;
  int m_tiles;
  int bn;
  int M, N;
  struct Row {
    uint32_t bits[8];  // mask words of this row for the n-tile (bn <= 256)
  };
  __device__ void prepare(Row& r, const Ctx& c, float*) const {
#pragma unroll
    for (int i = 0; i < 8; ++i) r.bits[i] = 0xffffffffu;
    if (mask[c.group] && c.m < M) {
      const uint32_t* p = mask[c.group] + static_cast<int64_t>(c.n_tile * (bn >> 5)) * ld_mask + c.m;
#pragma unroll
      for (int i = 0; i < 8; ++i)
        if (i < (bn >> 5)) r.bits[i] = p[static_cast<int64_t>(i) * ld_mask];
    }
  }
  __device__ bool chunk(Row& r, const Ctx& c, int n0, float (&v)[32], float* scratch) const {
    const int ci = (n0 % bn) >> 5;
    uint32_t bits = 0;
#pragma unroll
    for (int i = 0; i < 8; ++i)
      if (i == ci) bits = r.bits[i];
    const bool row_ok = c.m < M;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      const bool keep = row_ok && (n0 + t < N) && ((bits >> t) & 1u);
      v[t] = keep ? v[t] : 0.0f;
    }
    if (colsum) {
      // Column sums over the 32 rows of this warp: recursive halving leaves
      // lane l with the sum of column l (fixed order -> deterministic); then
      // the 4 warps of this column half add their slabs in quadrant order.
      float g[32];
#pragma unroll
      for (int t = 0; t < 32; ++t) g[t] = v[t];
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
      const int q = (threadIdx.x >> 5) & 3;
      float* sc = scratch + c.half * 128;  // (DgradMask keeps no constants in scratch)
      sc[q * 32 + lane] = g[0];
      ptx::named_bar_sync(2 + c.half, 128);
      if (q == 0 && n0 + lane < N) {
        const float s = __fadd_rn(__fadd_rn(sc[lane], sc[32 + lane]),
                                  __fadd_rn(sc[64 + lane], sc[96 + lane]));
        colsum[(static_cast<int64_t>(c.group) * m_tiles + c.m_tile) * ld_cs + n0 + lane] = s;
      }
      ptx::named_bar_sync(2 + c.half, 128);
    }
    return true;
  }
  __device__ void end(Row&, const Ctx&) const {}
};

// Split-K partial tiles, TMA-stored through a 3-D map
// {N, M, groups*splits}: W[((group*splits + split)*M + m)*N + n].
struct Partial {
  static constexpr int kStoreRank = 3;
  static constexpr bool kSplitCols = true;
  struct Row {};
  __device__ void prepare(Row&, const Ctx&, float*) const {}
  __device__ bool chunk(Row&, const Ctx&, int, float (&)[32], float*) const { return true; }
  __device__ void end(Row&, const Ctx&) const {}
};

// out = acc (+ bias) (ReLU optional), TMA-stored: the plain affine layer.
struct Linear {
  static constexpr int kStoreRank = 2;
  static constexpr bool kSplitCols = true;
  const float* bias;  // nullable
  int relu;
  int bn;
  int N;
  struct Row {};
  __device__ void prepare(Row&, const Ctx& c, float* scratch) const {
    for (int i = c.et; i < bn; i += c.ne) {
      const int n = c.n_tile * bn + i;
      scratch[i] = (bias && n < N) ? bias[n] : 0.0f;
    }
  }
  __device__ bool chunk(Row&, const Ctx&, int n0, float (&v)[32], float* scratch) const {
    const int c0 = n0 % bn;
#pragma unroll
    for (int t = 0; t < 32; ++t) {
      float x = bias ? __fadd_rn(v[t], scratch[c0 + t]) : v[t];
      if (relu) x = x > 0.0f ? x : 0.0f;
      v[t] = x;
    }
    return true;
  }
  __device__ void end(Row&, const Ctx&) const {}
};

// Raw store of the accumulator (narrow outputs, e.g. the action columns of
// the critic input gradient).
struct Store {
  static constexpr int kStoreRank = 0;
  static constexpr bool kSplitCols = false;
  float* out[2];
  int64_t ld_out;
  int M, N;
  struct Row {};
  __device__ void prepare(Row&, const Ctx&, float*) const {}
  __device__ bool chunk(Row&, const Ctx& c, int n0, float (&v)[32], float*) const {
    if (c.m >= M) return false;
    float* o = out[c.group] + static_cast<int64_t>(c.m) * ld_out;
#pragma unroll
    for (int t = 0; t < 32; ++t)
      if (n0 + t < N) o[n0 + t] = v[t];
    return false;
  }
  __device__ void end(Row&, const Ctx&) const {}
};

}  // namespace pqlg::epi

namespace pqlg::epi {

// Categorical (C51) critic head, c51.hpp:43-53 and :117-126: logits = acc +
// b over the L <= 64 atoms of a row (one 64-column tile, so each epilogue
// thread owns a whole row), then softmax_row (max, exp, running sum, divide)
// and the expected value E = sum_j p_j z_j (float, j ascending, no FMA).
// Writes probs[m*ld + j] and, if ev is set, ev[m].
struct C51Head {
  static constexpr int kStoreRank = 0;
  static constexpr bool kSplitCols = false;
  static constexpr int kMaxAtoms = 64;
  const float* bias[4];
  float* probs[4];
  int64_t ld;
  float* ev[4];  // nullable
  const float* atoms;
  int M, L;
  struct Row {
    float x[kMaxAtoms];
  };
  __device__ void prepare(Row&, const Ctx& c, float* scratch) const {
    for (int i = c.et; i < kMaxAtoms; i += c.ne) {
      scratch[i] = i < L ? bias[c.group][i] : 0.0f;
      scratch[kMaxAtoms + i] = i < L ? atoms[i] : 0.0f;
    }
  }
  __device__ bool chunk(Row& r, const Ctx& c, int n0, float (&v)[32], float* scratch) const {
    if (n0 == 0) {
#pragma unroll
      for (int t = 0; t < 32; ++t) r.x[t] = __fadd_rn(v[t], scratch[t]);
      if (L > 32) return false;
    } else {
#pragma unroll
      for (int t = 0; t < 32; ++t) r.x[32 + t] = __fadd_rn(v[t], scratch[32 + t]);
    }
    // last chunk of the row (BN = 64 covers L <= 64): softmax_row + E with
    // the atoms from shared memory (c51.hpp:44-53, :135-138)
    finish(r, c, scratch + kMaxAtoms);
    return false;
  }
  __device__ void finish(Row& r, const Ctx& c, const float* z) const {
    const int m = c.m, group = c.group;
    if (m >= M) return;
    float mx = r.x[0];
#pragma unroll
    for (int j = 1; j < kMaxAtoms; ++j)
      if (j < L) mx = mx < r.x[j] ? r.x[j] : mx;  // std::max(mx, l)
    float sum = 0.0f;
#pragma unroll
    for (int j = 0; j < kMaxAtoms; ++j)
      if (j < L) {
        r.x[j] = expf(__fsub_rn(r.x[j], mx));
        sum = __fadd_rn(sum, r.x[j]);
      }
    float e = 0.0f;
    float* out = probs[group] + static_cast<int64_t>(m) * ld;
#pragma unroll
    for (int j = 0; j < kMaxAtoms; ++j)
      if (j < L) {
        const float p = __fdiv_rn(r.x[j], sum);
        out[j] = p;
        e = __fadd_rn(e, __fmul_rn(p, z[j]));
      }
    if (ev[group]) ev[group][m] = e;
  }
  __device__ void end(Row&, const Ctx&) const {}
};

}  // namespace pqlg::epi
