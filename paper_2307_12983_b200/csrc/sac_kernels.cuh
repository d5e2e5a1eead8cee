// pql_sac on the device (proj/include/pql/agents/sac.hpp, policy.hpp:54-153,
// learners.cpp:87-94, :168-176, :246-258):
//
//   eps_count_kernel / eps_emit_kernel  the learners' eps draws: one
//        normal_distribution<float> per update over the Philox counter URBG
//        (polar method, libstdc++ random.tcc:1811-1844), generated in
//        parallel: candidate pair j uses draws 2j, 2j+1; a scan over the
//        accepted candidates gives every normal its place, so the values
//        equal the sequential loop's (orc_normals, kind 1) bit for bit.
//   gauss_finish_kernel  GaussianPolicy::sample from the split-K head
//        partials: [mean | log_std] + bias, clamp, reparameterised sample,
//        squash, log-prob; eps from the learners' stream or (actor) a fresh
//        normal_distribution per env over its SplitMix state, drawn
//        warp-parallel.
//   sac_pick_kernel      sac_actor_loss's row loop (sac.hpp:86-96): loss,
//        mean log-prob (for the alpha update) and the picked critic's upstream.
//   sac_head_backward_kernel  GaussianPolicy::backward's dy (policy.hpp:127-150)
//        + bias-gradient partials of the head.
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "rng.cuh"

namespace pqlg::sac {

constexpr float kLogStdMin = -5.0f;                                      // policy.hpp:61
constexpr float kLogStdMax = 2.0f;                                       // policy.hpp:62
constexpr float kSquashFloor = static_cast<float>(1e-6);                 // policy.hpp:63
constexpr float kHalfLog2Pi = static_cast<float>(0.5 * 1.8378770664093453);  // policy.hpp:87

// ------------------------------------------------------------ eps stream
struct EpsState {
  uint64_t key;
  uint64_t ctr;  // next Philox draw
};

constexpr int kEpsThreads = 256;
constexpr int kEpsPer = 1;  // candidates per thread (many blocks: the draws are latency-bound)
constexpr int kEpsChunk = kEpsThreads * kEpsPer;

struct EpsArgs {
  EpsState* st;
  float* out;            // [n]
  int64_t n;             // normals to draw
  int64_t need;          // accepted pairs needed = ceil(n / 2)
  unsigned int* counts;  // [gridDim.x] accepted candidates per block
  unsigned int* ticket;
  int64_t* last_j;       // candidate index of pair need-1 (written by its block; -1 between calls)
};

// Candidate pair j of the stream at counter c: (x, y, r2) from draws c+2j, c+2j+1.
__device__ __forceinline__ bool eps_candidate(uint64_t key, uint64_t c, int64_t j, float& x,
                                              float& y, float& r2) {
  auto canon = [](uint64_t v) {
    float u = __fmul_rn(__ull2float_rn(v), 0x1p-64f);
    if (u >= 1.0f) u = __uint_as_float(0x3f7fffffu);
    return u;
  };
  const uint64_t d0 = rng::philox_draw(key, c + 2 * static_cast<uint64_t>(j));
  const uint64_t d1 = rng::philox_draw(key, c + 2 * static_cast<uint64_t>(j) + 1);
  x = __double2float_rn(static_cast<double>(__fmul_rn(2.0f, canon(d0))) - 1.0);
  y = __double2float_rn(static_cast<double>(__fmul_rn(2.0f, canon(d1))) - 1.0);
  r2 = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
  return !(r2 > 1.0f || r2 == 0.0f);
}

__device__ __forceinline__ void eps_write(const EpsArgs& a, int64_t p, float x, float y,
                                          float r2) {
  const float mult = __fsqrt_rn(__fdiv_rn(__fmul_rn(-2.0f, rng::glibc_logf(r2)), r2));
  if (2 * p < a.n) a.out[2 * p] = __fmul_rn(y, mult);          // returned first
  if (2 * p + 1 < a.n) a.out[2 * p + 1] = __fmul_rn(x, mult);  // the cached value
}

static __global__ void __launch_bounds__(kEpsThreads) eps_count_kernel(EpsArgs a) {
  pdl::entry();
  const uint64_t key = a.st->key, c = a.st->ctr;
  unsigned int n = 0;
#pragma unroll
  for (int u = 0; u < kEpsPer; ++u) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * kEpsChunk + threadIdx.x * kEpsPer + u;
    float x, y, r2;
    n += eps_candidate(key, c, j, x, y, r2) ? 1u : 0u;
  }
  n = __reduce_add_sync(0xffffffffu, n);
  __shared__ unsigned int wsum[kEpsThreads / 32];
  if ((threadIdx.x & 31) == 0) wsum[threadIdx.x >> 5] = n;
  __syncthreads();
  if (threadIdx.x == 0) {
    unsigned int s = 0;
    for (int w = 0; w < kEpsThreads / 32; ++w) s += wsum[w];
    a.counts[blockIdx.x] = s;
  }
}

static __global__ void __launch_bounds__(kEpsThreads) eps_emit_kernel(EpsArgs a) {
  pdl::entry();
  const uint64_t key = a.st->key, c = a.st->ctr;
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  __shared__ unsigned int wsum[kEpsThreads / 32];
  __shared__ int64_t prefix_s;
  __shared__ bool last;
  // accepted pairs of the blocks before this one
  unsigned long long pre = 0;
  for (unsigned i = threadIdx.x; i < blockIdx.x; i += kEpsThreads) pre += a.counts[i];
  pre = __reduce_add_sync(0xffffffffu, static_cast<unsigned>(pre));  // < 2^32 candidates
  if (lane == 0) wsum[w] = static_cast<unsigned>(pre);
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t s = 0;
    for (int k = 0; k < kEpsThreads / 32; ++k) s += wsum[k];
    prefix_s = s;
  }
  __syncthreads();
  const int64_t base = prefix_s;
  float x[kEpsPer], y[kEpsPer], r2[kEpsPer];
  bool ok[kEpsPer];
  unsigned int mine = 0;
#pragma unroll
  for (int u = 0; u < kEpsPer; ++u) {
    const int64_t j = static_cast<int64_t>(blockIdx.x) * kEpsChunk + threadIdx.x * kEpsPer + u;
    ok[u] = eps_candidate(key, c, j, x[u], y[u], r2[u]);
    mine += ok[u] ? 1u : 0u;
  }
  // exclusive scan of `mine` over the block (thread order = candidate order)
  unsigned int incl = mine;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const unsigned int v = __shfl_up_sync(0xffffffffu, incl, d);
    if (lane >= d) incl += v;
  }
  __syncthreads();
  if (lane == 31) wsum[w] = incl;
  __syncthreads();
  unsigned int woff = 0;
  for (int k = 0; k < w; ++k) woff += wsum[k];
  int64_t p = base + woff + incl - mine;
#pragma unroll
  for (int u = 0; u < kEpsPer; ++u) {
    if (!ok[u]) continue;
    if (p < a.need) {
      eps_write(a, p, x[u], y[u], r2[u]);
      if (p == a.need - 1) {
        *a.last_j = static_cast<int64_t>(blockIdx.x) * kEpsChunk + threadIdx.x * kEpsPer + u;
        __threadfence();  // visible to the last block (ticket below)
      }
    }
    ++p;
  }
  // the last block to finish advances the counter (and, if the candidates
  // ran out -- probability ~1e-12 -- continues the stream sequentially)
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(a.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x != 0) return;
  __threadfence();
  *a.ticket = 0;
  int64_t lj = __ldcg(a.last_j);
  if (lj < 0) {  // shortfall: every candidate was taken; continue sequentially
    int64_t q = 0;
    for (unsigned i = 0; i < gridDim.x; ++i) q += __ldcg(a.counts + i);
    int64_t j = static_cast<int64_t>(gridDim.x) * kEpsChunk;
    for (;; ++j) {
      float xx, yy, rr;
      if (!eps_candidate(key, c, j, xx, yy, rr)) continue;
      eps_write(a, q, xx, yy, rr);
      if (++q == a.need) break;
    }
    lj = j;
  }
  *a.last_j = -1;
  a.st->ctr = c + 2 * static_cast<uint64_t>(lj + 1);
}

// ------------------------------------------------------ Gaussian head
constexpr int kFinishWarps = 8;

struct GaussArgs {
  const float* part;  // [S][M][ld_part] split-K partial sums of the 2A head columns
  int S;
  int64_t ld_part;
  const float* bias;  // [2A]
  const float* eps;   // [M x A] (learners), or null: per-row draws from rng
  uint64_t* rng;      // [M] SplitMix states (actor), advanced by the draws
  float* act;         // [M x ld_act]
  int64_t ld_act;
  float* logp;        // nullable [M]
  float* tanh_out;    // nullable [M x ld_aux]  tanh(pre)
  float* sd_out;      // nullable [M x ld_aux]  std, negated where log_std was clamped
  int64_t ld_aux;
  int M, A;
  float mid, half;
};

// Warp per row (grid-stride), lane d < A handles mean column d and log_std
// column A + d; the log-prob sum runs over d ascending as the reference's.
static __global__ void __launch_bounds__(32 * kFinishWarps)
    gauss_finish_kernel(const __grid_constant__ GaussArgs a) {
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warps = gridDim.x * kFinishWarps;
  const int64_t ss = static_cast<int64_t>(a.M) * a.ld_part;
  const bool on = lane < a.A;
  const float bm = on ? a.bias[lane] : 0.0f;
  const float bl = on ? a.bias[a.A + lane] : 0.0f;
  for (int m = blockIdx.x * kFinishWarps + w; m < a.M; m += warps) {
    float e = 0.0f;
    if (a.eps) {
      if (on) e = a.eps[static_cast<int64_t>(m) * a.A + lane];
    } else {
      e = rng::warp_row_normals(a.rng + m, a.A, lane);
    }
    float term = 0.0f;
    if (on) {
      const float* p = a.part + static_cast<int64_t>(m) * a.ld_part;
      float ym = p[lane], yl = p[a.A + lane];
      for (int s = 1; s < a.S; ++s) {
        ym = __fadd_rn(ym, p[s * ss + lane]);
        yl = __fadd_rn(yl, p[s * ss + a.A + lane]);
      }
      ym = __fadd_rn(ym, bm);
      float ls = __fadd_rn(yl, bl);
      const bool clamped = ls < kLogStdMin || ls > kLogStdMax;
      if (ls < kLogStdMin) ls = kLogStdMin;
      if (ls > kLogStdMax) ls = kLogStdMax;
      const float sd = expf(ls);
      const float pre = __fadd_rn(ym, __fmul_rn(sd, e));
      const float t = tanhf(pre);
      const int64_t r = static_cast<int64_t>(m);
      a.act[r * a.ld_act + lane] = __fadd_rn(a.mid, __fmul_rn(a.half, t));
      if (a.tanh_out) a.tanh_out[r * a.ld_aux + lane] = t;
      if (a.sd_out) a.sd_out[r * a.ld_aux + lane] = clamped ? -sd : sd;
      const float jac =
          __fadd_rn(__fmul_rn(a.half, __fsub_rn(1.0f, __fmul_rn(t, t))), kSquashFloor);
      term = __fsub_rn(__fsub_rn(__fsub_rn(__fmul_rn(__fmul_rn(-0.5f, e), e), ls), kHalfLog2Pi),
                       rng::glibc_logf(jac));
    }
    if (a.logp) {
      float lp = 0.0f;
      for (int d = 0; d < a.A; ++d) lp = __fadd_rn(lp, __shfl_sync(0xffffffffu, term, d));
      if (lane == 0) a.logp[m] = lp;
    }
  }
}

// ------------------------------------------------- actor objective rows
constexpr int kRowThreads = 256;

struct PickArgs {
  const float* partial;  // online head partials [2][n_tiles][ld]
  int64_t ld;
  int n_tiles;
  const float* q1;
  const float* q2;
  int64_t head_b_off;
  const float* logp;       // [B]
  const float* log_alpha;  // device scalar (the policy's, before this update's step)
  float* up;               // [2][B]
  int64_t* step;
  double* block_part;      // [2][gridDim.x]
  unsigned int* counter;
  float* out;              // [0] loss, [1] mean log-prob (both / Bg)
  uint32_t* status;
  int B, Bg;
};

__device__ __forceinline__ float head_q(const float* partial, int64_t ld, int n_tiles, int group,
                                        float bias, int64_t b) {
  float q = bias;
  for (int t = 0; t < n_tiles; ++t)
    q = __fadd_rn(q, partial[(static_cast<int64_t>(group) * n_tiles + t) * ld + b]);
  return q;
}

static __global__ void __launch_bounds__(kRowThreads) sac_pick_kernel(PickArgs a) {
  pdl::entry();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) *a.step += 1;
  const float alpha = expf(*a.log_alpha);
  double l = 0.0, lp = 0.0;
  if (b < a.B) {
    const float q1 = head_q(a.partial, a.ld, a.n_tiles, 0, a.q1[a.head_b_off], b);
    const float q2 = head_q(a.partial, a.ld, a.n_tiles, 1, a.q2[a.head_b_off], b);
    const bool pick1 = q1 <= q2;
    const float logp = a.logp[b];
    l = static_cast<double>(__fsub_rn(__fmul_rn(alpha, logp), pick1 ? q1 : q2));
    lp = static_cast<double>(logp);
    const float up = __fdiv_rn(-1.0f, static_cast<float>(a.Bg));
    a.up[b] = pick1 ? up : 0.0f;
    a.up[a.B + b] = pick1 ? 0.0f : up;
  }
  __shared__ double red[2][kRowThreads / 32];
  __shared__ bool last;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    l += __shfl_down_sync(0xffffffffu, l, d);
    lp += __shfl_down_sync(0xffffffffu, lp, d);
  }
  if ((threadIdx.x & 31) == 0) {
    red[0][threadIdx.x >> 5] = l;
    red[1][threadIdx.x >> 5] = lp;
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    double s0 = 0.0, s1 = 0.0;
    for (int k = 0; k < kRowThreads / 32; ++k) {
      s0 += red[0][k];
      s1 += red[1][k];
    }
    a.block_part[blockIdx.x] = s0;
    a.block_part[gridDim.x + blockIdx.x] = s1;
    __threadfence();
    last = atomicAdd(a.counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  double t0 = 0.0, t1 = 0.0;
  for (unsigned i = lane; i < gridDim.x; i += 32) {
    t0 += __ldcg(a.block_part + i);
    t1 += __ldcg(a.block_part + gridDim.x + i);
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    t0 += __shfl_xor_sync(0xffffffffu, t0, d);
    t1 += __shfl_xor_sync(0xffffffffu, t1, d);
  }
  if (lane == 0) {
    *a.counter = 0;
    const float loss = static_cast<float>(t0 / static_cast<double>(a.Bg));
    a.out[0] = loss;
    a.out[1] = static_cast<float>(t1 / static_cast<double>(a.Bg));
    if (!isfinite(loss)) atomicOr(a.status, 4u);
  }
}

// GaussianPolicy::backward's dy for upstream dact = din1 + din2 (action
// columns) and dlogp = alpha / B; warp per 8-row tile, lane = action dim.
struct HeadBwdArgs {
  const float* dact1;
  const float* dact2;
  int64_t ld_dact;
  const float* tanh_in;  // [B x ld_aux] tanh(pre)
  const float* sd_in;    // [B x ld_aux] +-std (negative: log_std clamped)
  int64_t ld_aux;
  const float* eps;      // [B x A]
  const float* log_alpha;
  float* dy;             // [B x ld_dy], columns [mean | log_std]
  int64_t ld_dy;
  float* db_part;        // [tiles][2A]
  float half;
  int B, A, Bg, rows_per_tile;
};

static __global__ void __launch_bounds__(32)
    sac_head_backward_kernel(const __grid_constant__ HeadBwdArgs a) {
  pdl::entry();
  const int tile = blockIdx.x;
  const int b0 = tile * a.rows_per_tile;
  const int c = threadIdx.x;
  if (c >= a.A) return;
  const float alpha = expf(*a.log_alpha);
  const float dlp = __fdiv_rn(alpha, static_cast<float>(a.Bg));
  const float h = a.half;
  float dbm = 0.0f, dbl = 0.0f;
  for (int u = 0; u < a.rows_per_tile; ++u) {
    const int b = b0 + u;
    if (b >= a.B) break;
    const int64_t r = static_cast<int64_t>(b);
    const float da = __fadd_rn(a.dact1[r * a.ld_dact + c], a.dact2[r * a.ld_dact + c]);
    const float t = a.tanh_in[r * a.ld_aux + c];
    const float sds = a.sd_in[r * a.ld_aux + c];
    const float sd = fabsf(sds);
    const float e = a.eps[r * a.A + c];
    const float sech2 = __fsub_rn(1.0f, __fmul_rn(t, t));
    const float jac = __fadd_rn(__fmul_rn(h, sech2), kSquashFloor);
    const float da_dpre = __fmul_rn(h, sech2);
    const float dlp_dpre = __fdiv_rn(__fmul_rn(__fmul_rn(__fmul_rn(2.0f, t), h), sech2), jac);
    const float gm = __fadd_rn(__fmul_rn(da, da_dpre), __fmul_rn(dlp, dlp_dpre));
    float gl = __fadd_rn(__fmul_rn(__fmul_rn(__fmul_rn(da, da_dpre), sd), e),
                         __fmul_rn(dlp, __fsub_rn(__fmul_rn(__fmul_rn(dlp_dpre, sd), e), 1.0f)));
    if (sds < 0.0f) gl = 0.0f;
    a.dy[r * a.ld_dy + c] = gm;
    a.dy[r * a.ld_dy + a.A + c] = gl;
    dbm = __fadd_rn(dbm, gm);
    dbl = __fadd_rn(dbl, gl);
  }
  a.db_part[static_cast<int64_t>(tile) * 2 * a.A + c] = dbm;
  a.db_part[static_cast<int64_t>(tile) * 2 * a.A + a.A + c] = dbl;
}

// sac_alpha_loss + adam_step on log alpha (sac.hpp:117-125,
// learners.cpp:254-256), run by one thread of the policy's Adam launch.
struct AlphaArgs {
  float* log_alpha;        // null: not SAC
  float* m;
  float* v;
  const float* mean_logp;  // mean log-prob of this update (all ranks)
  float target_entropy;    // -act_dim
  float lr;
};

}  // namespace pqlg::sac
