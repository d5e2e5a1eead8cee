// Row-wise heads of the DDPG critic losses (ddpg.hpp) that sit between the
// tensor-core GEMMs: the value head 512->1 is folded into the last hidden
// layer's epilogue as per-n-tile partial dots; these kernels finish it.
//
//   critic_loss_kernel   ddpg_critic_target  y = G + eff * min(Q1', Q2')      ddpg.hpp:24-40
//                        + ddpg_critic_loss  e = Q - y, up = 2e/B, loss       ddpg.hpp:50-76
//   actor_pick_kernel    ddpg_actor_loss     pick1 = Q1 <= Q2, up = -1/B      ddpg.hpp:86-118
//   head_backward_kernel fa::backward of the 512->1 layer + ReLU mask of the
//                        layer below (mlp.hpp:161-184) and its bias/weight
//                        gradient partials (scalar.hpp:42-55)
#pragma once

#include "pdl.cuh"
#include <cstdint>

namespace pqlg::critic {

constexpr int kRowThreads = 256;

// q_k[b] = b_head_k + sum_t partial[k][t][b]   (t ascending)
__device__ __forceinline__ float head_value(const float* partial, int64_t ld, int n_tiles,
                                            int group, float bias, int64_t b) {
  float q = bias;
  for (int t = 0; t < n_tiles; ++t)
    q = __fadd_rn(q, partial[(static_cast<int64_t>(group) * n_tiles + t) * ld + b]);
  return q;
}

// Block sums of l -> block_loss[blockIdx.x]; the last block (ticket) adds the
// block sums in fixed order (lane-strided, then an xor tree) and writes
// out = sum / B, flagging a non-finite result in status.
template <int kThreads = kRowThreads>
__device__ __forceinline__ void block_mean_finish(double l, double* block_loss,
                                                  unsigned int* counter, int B, float* out,
                                                  uint32_t* status, uint32_t bit) {
  __shared__ double red[kThreads / 32];
  __shared__ bool last;
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) l += __shfl_down_sync(0xffffffffu, l, d);
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = l;
  __syncthreads();
  if (threadIdx.x == 0) {
    double s = 0.0;
    for (int w = 0; w < kThreads / 32; ++w) s += red[w];
    block_loss[blockIdx.x] = s;
    __threadfence();
    last = atomicAdd(counter, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  double tot = 0.0;
  for (unsigned i = lane; i < gridDim.x; i += 32) tot += __ldcg(block_loss + i);
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) tot += __shfl_xor_sync(0xffffffffu, tot, d);
  if (lane == 0) {
    *counter = 0;
    const float v = static_cast<float>(tot / static_cast<double>(B));
    *out = v;
    if (!isfinite(v)) atomicOr(status, bit);
  }
}

// ddpg_critic_target + ddpg_critic_loss in one launch (ddpg.hpp:24-40,
// :50-76): y = G + eff * min(Q1', Q2') from the target critics' head
// partials, e_k = Q_k - y from the online ones, up_k = 2 e_k / B, loss =
// mean(e1^2 + e2^2).  Also advances the device Adam step (once per update).
struct LossArgs {
  const float* partial;  // online [2][n_tiles][ld]
  int64_t ld;
  int n_tiles;
  const float* q1;
  const float* q2;
  int64_t head_b_off;
  // target side (critic loss only)
  const float* partial_t;  // target [2][n_tiles][ld]
  const float* q1t;
  const float* q2t;
  const float* ret;
  const float* eff;
  float* y;                // [B] TD targets (kept for inspection)
  const float* logp;       // pql_sac: log pi(a'|s+) [B] (null: DDPG target)
  const float* log_alpha;  // pql_sac: the lagged policy's log alpha
  int64_t* step;           // Adam step
  float* up;          // [2][B]  dLoss/dQ_k
  double* block_loss; // [gridDim.x]
  unsigned int* counter;
  float* loss_out;
  uint32_t* status;   // bit1: non-finite target, bit2: non-finite loss
  int B;
  int Bg;             // mean divisor: B, or the global batch of a data-parallel update
};

static __global__ void __launch_bounds__(kRowThreads) critic_loss_kernel(LossArgs a) {
  pdl::entry();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0) *a.step += 1;
  double l = 0.0;
  if (b < a.B) {
    const float t1 = head_value(a.partial_t, a.ld, a.n_tiles, 0, a.q1t[a.head_b_off], b);
    const float t2 = head_value(a.partial_t, a.ld, a.n_tiles, 1, a.q2t[a.head_b_off], b);
    float qmin = t2 < t1 ? t2 : t1;  // std::min(q1, q2)
    if (a.logp)  // sac_critic_loss: qmin - alpha * log pi (sac.hpp:38-39)
      qmin = __fsub_rn(qmin, __fmul_rn(expf(*a.log_alpha), a.logp[b]));
    const float y = __fadd_rn(a.ret[b], __fmul_rn(a.eff[b], qmin));
    a.y[b] = y;
    if (!isfinite(y)) atomicOr(a.status, 2u);
    const float q1 = head_value(a.partial, a.ld, a.n_tiles, 0, a.q1[a.head_b_off], b);
    const float q2 = head_value(a.partial, a.ld, a.n_tiles, 1, a.q2[a.head_b_off], b);
    const float e1 = __fsub_rn(q1, y);
    const float e2 = __fsub_rn(q2, y);
    l = static_cast<double>(__fadd_rn(__fmul_rn(e1, e1), __fmul_rn(e2, e2)));
    const float Bf = static_cast<float>(a.Bg);
    a.up[b] = __fdiv_rn(__fmul_rn(2.0f, e1), Bf);
    a.up[a.B + b] = __fdiv_rn(__fmul_rn(2.0f, e2), Bf);
  }
  block_mean_finish(l, a.block_loss, a.counter, a.Bg, a.loss_out, a.status, 4u);
}

// ddpg_actor_loss row head: pick1 = q1 <= q2; loss -= min; upstream of the
// picked critic -1/B (ddpg.hpp:100-105).
static __global__ void __launch_bounds__(kRowThreads) actor_pick_kernel(LossArgs a) {
  pdl::entry();
  const int b = blockIdx.x * blockDim.x + threadIdx.x;
  if (b == 0 && a.step) *a.step += 1;
  double l = 0.0;
  if (b < a.B) {
    const float q1 = head_value(a.partial, a.ld, a.n_tiles, 0, a.q1[a.head_b_off], b);
    const float q2 = head_value(a.partial, a.ld, a.n_tiles, 1, a.q2[a.head_b_off], b);
    const bool pick1 = q1 <= q2;
    l = -static_cast<double>(pick1 ? q1 : q2);
    const float up = __fdiv_rn(-1.0f, static_cast<float>(a.Bg));
    a.up[b] = pick1 ? up : 0.0f;
    a.up[a.B + b] = pick1 ? 0.0f : up;
  }
  block_mean_finish(l, a.block_loss, a.counter, a.Bg, a.loss_out, a.status, 4u);
}

// Backward through the 512->1 value head for both critics.
//   G[b,i]   = up[b] * w[i] * [h[b,i] > 0]            (dgrad + ReLU mask)
//   dW[i]   += h[b,i] * up[b]     db_head += up[b]    (wgrad of the head)
//   db[i]   += G[b,i]                                 (bias grad of layer below)
// grid = (row tiles of kHeadRows, groups), one thread per column: loads and
// stores are coalesced across the block; partials per row tile are summed
// later in tile order.  with_params = 0 for the actor gradient.
constexpr int kHeadRows = 64;
constexpr int kHeadThreads = 512;

struct HeadBwdArgs {
  const float* up;     // [2][B]
  const float* h[2];   // post-activations of the last hidden layer [B x H]
  int64_t ld_h;
  const float* w[2];   // head weights [H] (W_head is [H x 1])
  float* G[2];         // out [B x H]
  int64_t ld_g;
  float* dw_part;      // [2][tiles][H]
  float* db_head_part; // [2][tiles]
  float* db_part;      // [2][tiles][H]
  int B, H, tiles;
  int with_params;
};

static __global__ void __launch_bounds__(kHeadThreads)
    head_backward_kernel(const __grid_constant__ HeadBwdArgs a) {
  pdl::entry();
  const int tile = blockIdx.x, k = blockIdx.y;
  const int b0 = tile * kHeadRows;
  const int b1 = min(b0 + kHeadRows, a.B);
  const float* up = a.up + static_cast<int64_t>(k) * a.B;
  __shared__ float sup[kHeadRows];
  for (int b = threadIdx.x; b < b1 - b0; b += blockDim.x) sup[b] = up[b0 + b];
  __syncthreads();
  const float* __restrict__ h = a.h[k];
  const float* __restrict__ w = a.w[k];
  float* __restrict__ G = a.G[k];
  for (int i = threadIdx.x; i < a.H; i += blockDim.x) {
    const float wi = w[i];
    float dw = 0.0f, db = 0.0f;
    for (int bb = b0; bb < b1; bb += 8) {
      float hv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        hv[u] = bb + u < b1 ? __ldg(h + static_cast<int64_t>(bb + u) * a.ld_h + i) : 0.0f;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (bb + u >= b1) break;
        const float uu = sup[bb + u - b0];
        const float g = hv[u] > 0.0f ? __fmul_rn(uu, wi) : 0.0f;
        G[static_cast<int64_t>(bb + u) * a.ld_g + i] = g;
        dw = __fadd_rn(dw, __fmul_rn(hv[u], uu));
        db = __fadd_rn(db, g);
      }
    }
    if (a.with_params) {
      a.dw_part[(static_cast<int64_t>(k) * a.tiles + tile) * a.H + i] = dw;
      a.db_part[(static_cast<int64_t>(k) * a.tiles + tile) * a.H + i] = db;
    }
  }
  if (a.with_params && threadIdx.x == 0) {
    float s = 0.0f;
    for (int b = 0; b < b1 - b0; ++b) s = __fadd_rn(s, sup[b]);
    a.db_head_part[static_cast<int64_t>(k) * a.tiles + tile] = s;
  }
}

// Input gradient through the value head only (ddpg_actor_loss, critics
// frozen: mlp.hpp:187-201): G[b,i] = up[b] * w[i] * [post[b,i] > 0] with the
// ReLU mask taken from the forward pass's bitmask.  One thread per element.
struct HeadInputGradArgs {
  const float* up;         // [2][B]
  const uint32_t* mask[2]; // [B x H/32]
  const float* w[2];       // [H]
  float* G[2];             // [B x H]
  int B, H;
};

// Row-blocked: each warp takes whole rows, lane l covering columns
// [4l, 4l+4) + 128j -- one mask word per 8 lanes, float4 stores.
static __global__ void __launch_bounds__(256)
    head_input_grad_kernel(const __grid_constant__ HeadInputGradArgs a) {
  pdl::entry();
  const int k = blockIdx.y;
  const int lane = threadIdx.x & 31;
  const int warps = gridDim.x * (blockDim.x >> 5);
  const float* __restrict__ w = a.w[k];
  const float* __restrict__ up = a.up + static_cast<int64_t>(k) * a.B;
  for (int b = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5); b < a.B; b += warps) {
    const float u = up[b];
    // word-major masks (epi::Hidden): word j of row b at mask[j * B + b]
    const uint32_t* mrow = a.mask[k] + b;
    float* g = a.G[k] + static_cast<int64_t>(b) * a.H;
    for (int c = 4 * lane; c < a.H; c += 128) {
      const uint32_t bits = mrow[static_cast<int64_t>(c >> 5) * a.B] >> (c & 31);
      const float4 w4 = *reinterpret_cast<const float4*>(w + c);
      float4 o;
      o.x = (bits & 1u) ? __fmul_rn(u, w4.x) : 0.0f;
      o.y = (bits & 2u) ? __fmul_rn(u, w4.y) : 0.0f;
      o.z = (bits & 4u) ? __fmul_rn(u, w4.z) : 0.0f;
      o.w = (bits & 8u) ? __fmul_rn(u, w4.w) : 0.0f;
      *reinterpret_cast<float4*>(g + c) = o;
    }
  }
}

// DeterministicPolicy::backward head (policy.hpp:41-51) fed by the actor
// gradient: dact = din1[:, obs:] + din2[:, obs:] (ddpg.hpp:112-115), then
// dy = dact * half * (1 - t^2) with t = tanh(y) from the forward; plus the
// head-bias gradient partials db[tile][a] = sum over the tile's rows of dy.
struct PolicyHeadBwdArgs {
  const float* dact1;  // [B x lda]
  const float* dact2;
  int64_t ld_dact;
  const float* t;      // tanh(y) [B x ld_t]
  int64_t ld_t;
  float* dy;           // [B x ld_dy]
  int64_t ld_dy;
  float* db_part;      // [tiles][A]
  float half;
  int B, A, rows_per_tile;
};

// One warp per tile of rows_per_tile (<= 8) rows, lane = action column:
// every load of the tile is in flight before the math.
static __global__ void __launch_bounds__(32)
    policy_head_backward_kernel(const __grid_constant__ PolicyHeadBwdArgs a) {
  pdl::entry();
  const int tile = blockIdx.x;
  const int b0 = tile * a.rows_per_tile;
  const int c = threadIdx.x;
  if (c >= a.A) return;
  float d1[8], d2[8], tv[8];
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int b = b0 + u;
    const bool ok = u < a.rows_per_tile && b < a.B;
    d1[u] = ok ? a.dact1[static_cast<int64_t>(b) * a.ld_dact + c] : 0.0f;
    d2[u] = ok ? a.dact2[static_cast<int64_t>(b) * a.ld_dact + c] : 0.0f;
    tv[u] = ok ? a.t[static_cast<int64_t>(b) * a.ld_t + c] : 0.0f;
  }
  float db = 0.0f;
#pragma unroll
  for (int u = 0; u < 8; ++u) {
    const int b = b0 + u;
    if (u >= a.rows_per_tile || b >= a.B) break;
    const float da = __fadd_rn(d1[u], d2[u]);
    const float g = __fmul_rn(__fmul_rn(da, a.half), __fsub_rn(1.0f, __fmul_rn(tv[u], tv[u])));
    a.dy[static_cast<int64_t>(b) * a.ld_dy + c] = g;
    db = __fadd_rn(db, g);
  }
  a.db_part[static_cast<int64_t>(tile) * a.A + c] = db;
}

}  // namespace pqlg::critic
