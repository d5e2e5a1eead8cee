// The learners' narrow policy head (H -> act_dim, DeterministicPolicy::act,
// policy.hpp:33-38) as split-K GEMM partials + one finishing kernel.  With
// only M/128 row tiles of 32 columns the head GEMM alone would stream its
// [M x H] input through a fraction of the SMs; split over K it uses all of
// them, and the finish sums the splits in fixed order, adds the bias and
// squashes.
#pragma once

#include <cstdint>

#include "pdl.cuh"
#include "ptx.cuh"

namespace pqlg::head {

constexpr int kFinishWarps = 8;

struct FinishArgs {
  const float* part;     // [S][M][ld_part] head-GEMM partial sums
  int S;
  int64_t ld_part;
  const float* bias;     // [A]
  float* act;            // [M x ld_act]
  int64_t ld_act;
  float* tanh_out;       // nullable [M x ld_tanh] (policy backward)
  int64_t ld_tanh;
  int M, A;
  float mid, half;
};

// Warp per row (grid-stride), lane = action column: y = sum_s part[s]
// (s ascending) + b, a = mid + half*tanh(y); coalesced loads and stores.
// (The actor's head, which also draws exploration noise, keeps the fused
// GEMM epilogue: its per-row draws overlap the mainloop there.)
static __global__ void __launch_bounds__(32 * kFinishWarps)
    policy_head_finish_kernel(const __grid_constant__ FinishArgs a) {
  pdl::entry();
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int warps = gridDim.x * kFinishWarps;
  const int64_t split_stride = static_cast<int64_t>(a.M) * a.ld_part;
  if (lane >= a.A) return;
  const float bc = a.bias[lane];
  for (int m = blockIdx.x * kFinishWarps + w; m < a.M; m += warps) {
    const float* p = a.part + static_cast<int64_t>(m) * a.ld_part + lane;
    float acc = p[0];
    for (int s = 1; s < a.S; ++s) acc = __fadd_rn(acc, p[s * split_stride]);
    const float y = __fadd_rn(acc, bc);
    const float th = tanhf(y);
    if (a.tanh_out) a.tanh_out[static_cast<int64_t>(m) * a.ld_tanh + lane] = th;
    a.act[static_cast<int64_t>(m) * a.ld_act + lane] = __fadd_rn(a.mid, __fmul_rn(a.half, th));
  }
}

}  // namespace pqlg::head

#include "norm_finish.cuh"
#include "rng.cuh"

namespace pqlg::head {

// ---------------------------------------------------------------------------
// The narrow policy head H -> N (N <= 72) with its finish fused
// (DeterministicPolicy::act, policy.hpp:33-38; for the actor also
// apply_noise, noise.hpp:56-72), one launch:
//
// A 512 -> 20 layer is 0.17 GFLOP against a 16.8 MB (B = 8192) or 33.5 MB
// (16384 envs) activation read: it is bound by streaming its input.  As a
// tcgen05 tile (32 useful columns, one 128-row tile per SM) it left the SMs
// latency bound; on the CUDA cores the W operand reads from shared memory
// bound it.  Here each warp owns 16 rows (one m16 tile) and half of K, and
// runs warp-level tensor-core MMAs (mma.sync m16n8k8 tf32, like the rest of
// the MLP: tf32 products, fp32 accumulation):
//   - A fragments come straight from global memory as float4 per lane:
//     lane (g, t) loads x[g][16b + 4t .. +3] and x[g + 8][...], i.e. k is
//     permuted inside each 16-block (logical (t, t+4) of the first k8 MMA
//     -> physical 4t, 4t+1, of the second -> 4t+2, 4t+3); every row is read
//     as whole 64-byte segments, 8 k16 blocks in flight per lane
//   - B fragments are staged once per block in that same order
//     ([k16 block][n8 tile][lane] float4: one conflict-free LDS.128 per
//     n-tile per k16 block), rounded to tf32 (3xTF32: raw, split hi / lo
//     where used, with the A hi / lo split: lo*hi + hi*lo + hi*hi)
//   - the two K halves are added in fixed order through shared memory
// Rows of the actor additionally draw their exploration normals (8 lanes
// per row, group_row_normals) while the loads are in flight.
// ---------------------------------------------------------------------------
constexpr int kHeadWarps = 8;          // kMT m16 tiles x (8 / kMT) K parts
// Rows per block: 16 kMT.  kMT = 4 (64 rows, K halves) for the actor's
// 16384 rows; kMT = 2 (32 rows, K quarters: one load round per warp, twice
// the blocks) for the learners' 8192 (head_mt()).
template <int kMT>
constexpr int head_rows() { return 16 * kMT; }
inline int head_mt(int M) { return M > 8192 ? 4 : 2; }
constexpr int kHeadMaxNT = 9;          // n8 tiles (N <= 72)

struct RowsArgs {
  const float* x;  // [M x K] (ldx % 4 == 0, 16-byte aligned rows), K % 4 == 0
  int64_t ldx;
  const float* w;  // [K x ldw] row-major (fa::Mlp layout); columns [0, N) are used
  int64_t ldw;
  const float* bias;  // [N] (squash mode)
  int M, K, N;
  int mode;  // 0 raw (out = x W), 1 squash
  float* out;  // raw: [M x ld_out]; squash: actions
  int64_t ld_out;
  float* tanh_out;  // nullable [M x ld_tanh]
  int64_t ld_tanh;
  float mid, half;
  uint64_t* noise_state;  // nullable: per-row SplitMix state (actor exploration)
  const float* sigma;     // [M]
  float low, high;
  // nullable: W already in the kernel's fragment order ([KB][kNT][32] float4,
  // head_pack_kernel), copied into shared memory with cp.async instead of
  // being gathered from W (the actor packs it whenever its policy changes)
  const float4* wpack;
  // optional: the actor's running-normalizer finish rides along as
  // fin.nblk extra blocks after the head's (independent work, one launch)
  actor::NormFinishArgs fin;
};

// W -> the head kernel's B-fragment order (tf32-rounded; raw for 3xTF32):
// element e = (kb * kNT + nt) * 32 + lane (g, t) holds W[16 kb + 4 t + q][8 nt + g], q = 0..3.
template <int kNT, bool k3x>
static __global__ void head_pack_kernel(const float* __restrict__ w, int64_t ldw, int K, int N,
                                        float4* __restrict__ out) {
  pdl::entry();
  const int KB = (K + 15) >> 4;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= KB * kNT * 32) return;
  const int ln = e & 31, nt = (e >> 5) % kNT, kb = (e >> 5) / kNT;
  const int g = ln >> 2, t = ln & 3;
  const int n = 8 * nt + g;
  float v[4];
#pragma unroll
  for (int q = 0; q < 4; ++q) {
    const int k = 16 * kb + 4 * t + q;
    v[q] = (k < K && n < N) ? w[static_cast<int64_t>(k) * ldw + n] : 0.0f;
    if constexpr (!k3x) {
      uint32_t r;
      asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(v[q]));
      v[q] = __uint_as_float(r);
    }
  }
  out[e] = make_float4(v[0], v[1], v[2], v[3]);
}

// The row's A normals (normal_distribution<float> polar pairs over its
// stream) drawn by the G lanes of its group: candidate pair c of the row uses
// stream states s0 + 2c, s0 + 2c + 1; accepted candidates are consumed in
// order.  Lanes of finished groups idle until the warp is done.
template <int G>
__device__ __forceinline__ void group_row_normals(uint64_t* state, uint64_t s0, bool active, int A,
                                                  int j, float* z) {
  const int lane = threadIdx.x & 31;
  const int base = lane & ~(G - 1);
  const unsigned gm = (G == 32) ? 0xffffffffu : ((1u << G) - 1u);
  if (!active) s0 = 0ull;
  const int need = (A + 1) / 2;
  int got = 0;
  bool done = !active;
  for (int round = 0; __any_sync(0xffffffffu, !done); ++round) {
    bool ok = false;
    float x = 0.0f, y = 0.0f, r2 = 0.0f;
    if (!done) {
      uint64_t s = s0 + 2 * (static_cast<uint64_t>(round) * G + j);
      x = __double2float_rn(static_cast<double>(__fmul_rn(2.0f, rng::canonical_f32(s))) - 1.0);
      y = __double2float_rn(static_cast<double>(__fmul_rn(2.0f, rng::canonical_f32(s))) - 1.0);
      r2 = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
      ok = !(r2 > 1.0f || r2 == 0.0f);
    }
    const unsigned bits = (__ballot_sync(0xffffffffu, ok) >> base) & gm;
    if (!done) {
      const int p = got + __popc(bits & ((1u << j) - 1u));
      if (ok && p < need) {
        const float mult = __fsqrt_rn(__fdiv_rn(__fmul_rn(-2.0f, rng::glibc_logf(r2)), r2));
        z[2 * p] = __fmul_rn(y, mult);  // y*mult first, x*mult cached (random.tcc:1838-1843)
        if (2 * p + 1 < A) z[2 * p + 1] = __fmul_rn(x, mult);
      }
      const int n = __popc(bits);
      if (got + n >= need) {
        const uint64_t consumed =
            static_cast<uint64_t>(round) * G + rng::nth_set_bit(bits, need - got - 1) + 1;
        if (j == 0) *state = s0 + 2 * consumed;
        done = true;
      } else {
        got += n;
      }
    }
  }
}

__device__ __forceinline__ void mma_tf32(float (&c)[4], uint32_t a0, uint32_t a1, uint32_t a2,
                                         uint32_t a3, uint32_t b0, uint32_t b1) {
  asm volatile(
      "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0, %1, %2, %3}, {%4, %5, %6, %7}, "
      "{%8, %9}, {%0, %1, %2, %3};"
      : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
      : "r"(a0), "r"(a1), "r"(a2), "r"(a3), "r"(b0), "r"(b1));
}

__device__ __forceinline__ uint32_t tf32_bits(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return r;
}

// Shared memory: W fragments [KB][kNT][32] float4, the K-part exchange
// [K parts - 1][kMT m-tiles][32 lanes][kNT * 4] floats, and the rows'
// exploration normals [rows][kNT * 8].
template <int kNT, bool k3x, int kMT>
inline size_t head_smem(int K) {
  const size_t kb = (static_cast<size_t>(K) + 15) / 16;
  constexpr int kKP = kHeadWarps / kMT;
  return kb * kNT * 32 * 16 + (kKP - 1) * kMT * 32 * kNT * 4 * 4 + head_rows<kMT>() * kNT * 8 * 4;
}

template <int kNT, bool k3x, int kMT>
static __global__ void __launch_bounds__(32 * kHeadWarps)
    head_mma_kernel(const __grid_constant__ RowsArgs a) {
  extern __shared__ float4 smem4[];
  constexpr int kHeadRows = head_rows<kMT>();
  constexpr int kKP = kHeadWarps / kMT;      // K parts
  constexpr int kDrawCalls = kHeadRows / 32;  // 4 rows per warp per draw call
  const int head_blocks = (a.M + kHeadRows - 1) / kHeadRows;
  if (static_cast<int>(blockIdx.x) >= head_blocks) {  // normalizer finish blocks
    pdl::entry();
    actor::norm_finish_block(a.fin, blockIdx.x - head_blocks, reinterpret_cast<double2*>(smem4));
    return;
  }
  const int K = a.K, N = a.N;
  const int KB = (K + 15) >> 4;
  float4* wf = smem4;  // [KB][kNT][32]: tf32-rounded, or raw fp32 for 3xTF32
  float* xch = reinterpret_cast<float*>(wf + static_cast<int64_t>(KB) * kNT * 32);
  float* sz = xch + (kKP - 1) * kMT * 32 * kNT * 4;  // [rows][kNT * 8]
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  // A loads first (the previous kernel's output), then -- while they are in
  // flight -- the exploration inputs, the W fragments and the noise draws.
  // (The previous grid holds every SM until it drains, so staging W before
  // the PDL wait would not overlap anything.)
  pdl::entry();
  const int mt = warp % kMT, kh = warp / kMT;  // m16 tile, K part
  const int g = lane >> 2, t = lane & 3;
  const int row0 = blockIdx.x * kHeadRows + 16 * mt;
  const int ra = row0 + g < a.M ? row0 + g : a.M - 1;   // clamped rows: results discarded
  const int rb = row0 + g + 8 < a.M ? row0 + g + 8 : a.M - 1;
  const float* xa = a.x + static_cast<int64_t>(ra) * a.ldx + 4 * t;
  const float* xb = a.x + static_cast<int64_t>(rb) * a.ldx + 4 * t;
  const int kp_len = (KB + kKP - 1) / kKP;
  const int kb0 = kh * kp_len < KB ? kh * kp_len : KB;
  const int kb1 = kb0 + kp_len < KB ? kb0 + kp_len : KB;
  constexpr int kU = 8;  // k16 blocks with loads in flight
  float4 va[kU], vb[kU];
  auto load = [&](int kb) {
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      const int k = 16 * (kb + u) + 4 * t;
      const bool ok = kb + u < kb1 && k < K;
      va[u] = ok ? __ldg(reinterpret_cast<const float4*>(xa + 16 * (kb + u))) : make_float4(0.f, 0.f, 0.f, 0.f);
      vb[u] = ok ? __ldg(reinterpret_cast<const float4*>(xb + 16 * (kb + u))) : make_float4(0.f, 0.f, 0.f, 0.f);
    }
  };
  load(kb0);
  // exploration inputs: the draw rows' sigma and SplitMix state, the finish
  // rows' sigma
  float sig_draw[kDrawCalls] = {}, sig_fin[2] = {0.0f, 0.0f};
  uint64_t st_draw[kDrawCalls] = {};
  if (a.noise_state) {
#pragma unroll
    for (int c = 0; c < kDrawCalls; ++c) {
      const int m = blockIdx.x * kHeadRows + warp * (4 * kDrawCalls) + c * 4 + (lane >> 3);
      if (m < a.M) {
        sig_draw[c] = a.sigma[m];
        st_draw[c] = a.noise_state[m];
      }
    }
#pragma unroll
    for (int h = 0; h < 2; ++h) {
      const int m = row0 + g + 8 * h;
      if (kh == 0 && m < a.M) sig_fin[h] = a.sigma[m];
    }
  }
  if (a.wpack) {
    // packed fragments: 16-byte cp.async copies, completed before the barrier below
    for (int e = tid; e < KB * kNT * 32; e += 32 * kHeadWarps)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(ptx::smem_u32(wf + e)),
                   "l"(a.wpack + e)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
  }
  // otherwise stage W fragments (kWU fragments' loads in flight per thread
  // before any is converted)
  constexpr int kWU = 4;
  for (int e0 = a.wpack ? KB * kNT * 32 : tid; e0 < KB * kNT * 32; e0 += kWU * 32 * kHeadWarps) {
    float v[kWU][4];
#pragma unroll
    for (int u = 0; u < kWU; ++u) {
      const int e = e0 + u * 32 * kHeadWarps;
      const int ln = e & 31, nt = (e >> 5) % kNT, kb = (e >> 5) / kNT;
      const int gg = ln >> 2, tt = ln & 3;
      const int n = 8 * nt + gg;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 16 * kb + 4 * tt + q;
        v[u][q] = (e < KB * kNT * 32 && k < K && n < N)
                      ? __ldg(a.w + static_cast<int64_t>(k) * a.ldw + n) : 0.0f;
      }
    }
#pragma unroll
    for (int u = 0; u < kWU; ++u) {
      const int e = e0 + u * 32 * kHeadWarps;
      if (e >= KB * kNT * 32) break;
      if constexpr (k3x) {  // raw fp32: split hi / lo where it is used
        wf[e] = make_float4(v[u][0], v[u][1], v[u][2], v[u][3]);
      } else {
        wf[e] = make_float4(__uint_as_float(tf32_bits(v[u][0])), __uint_as_float(tf32_bits(v[u][1])),
                            __uint_as_float(tf32_bits(v[u][2])), __uint_as_float(tf32_bits(v[u][3])));
      }
    }
  }
  // exploration draws for the block's 64 rows (8 lanes per row, 4 rows per
  // warp per call, 2 calls per warp)
  if (a.noise_state) {
#pragma unroll
    for (int c = 0; c < kDrawCalls; ++c) {
      const int r = warp * (4 * kDrawCalls) + c * 4 + (lane >> 3);  // block row
      const int m = blockIdx.x * kHeadRows + r;
      const bool on = m < a.M && sig_draw[c] > 0.0f;
      group_row_normals<8>(a.noise_state + (m < a.M ? m : 0), st_draw[c], on, N, lane & 7,
                           sz + r * kNT * 8);
    }
  }
  if (a.wpack) asm volatile("cp.async.wait_all;" ::: "memory");
  __syncthreads();  // W fragments (and the draws) staged
  float acc[kNT][4];
#pragma unroll
  for (int nt = 0; nt < kNT; ++nt) acc[nt][0] = acc[nt][1] = acc[nt][2] = acc[nt][3] = 0.0f;
  for (int kb = kb0; kb < kb1; kb += kU) {
    if (kb != kb0) load(kb);
#pragma unroll
    for (int u = 0; u < kU; ++u) {
      if (kb + u >= kb1) break;
      const float xa4[4] = {va[u].x, va[u].y, va[u].z, va[u].w};
      const float xb4[4] = {vb[u].x, vb[u].y, vb[u].z, vb[u].w};
      uint32_t ah[4], bh[4], al[4], bl[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        ah[q] = tf32_bits(xa4[q]);
        bh[q] = tf32_bits(xb4[q]);
        if constexpr (k3x) {
          al[q] = tf32_bits(__fsub_rn(xa4[q], __uint_as_float(ah[q])));
          bl[q] = tf32_bits(__fsub_rn(xb4[q], __uint_as_float(bh[q])));
        }
      }
      const float4* wrow = wf + static_cast<int64_t>(kb + u) * kNT * 32 + lane;
#pragma unroll
      for (int nt = 0; nt < kNT; ++nt) {
        const float4 w = wrow[nt * 32];
        uint32_t w0 = __float_as_uint(w.x), w1 = __float_as_uint(w.y), w2 = __float_as_uint(w.z),
                 w3 = __float_as_uint(w.w);
        if constexpr (k3x) {
          w0 = tf32_bits(w.x);
          w1 = tf32_bits(w.y);
          w2 = tf32_bits(w.z);
          w3 = tf32_bits(w.w);
          const uint32_t l0 = tf32_bits(__fsub_rn(w.x, __uint_as_float(w0)));
          const uint32_t l1 = tf32_bits(__fsub_rn(w.y, __uint_as_float(w1)));
          const uint32_t l2 = tf32_bits(__fsub_rn(w.z, __uint_as_float(w2)));
          const uint32_t l3 = tf32_bits(__fsub_rn(w.w, __uint_as_float(w3)));
          // small terms first, into the same accumulator
          mma_tf32(acc[nt], al[0], bl[0], al[1], bl[1], w0, w1);
          mma_tf32(acc[nt], ah[0], bh[0], ah[1], bh[1], l0, l1);
          mma_tf32(acc[nt], al[2], bl[2], al[3], bl[3], w2, w3);
          mma_tf32(acc[nt], ah[2], bh[2], ah[3], bh[3], l2, l3);
        }
        // k8 #1: logical k t / t+4 -> physical 4t / 4t+1; #2: 4t+2 / 4t+3
        mma_tf32(acc[nt], ah[0], bh[0], ah[1], bh[1], w0, w1);
        mma_tf32(acc[nt], ah[2], bh[2], ah[3], bh[3], w2, w3);
      }
    }
  }
  // K parts: parts 1.. hand their partial sums over shared memory, part 0
  // adds them in fixed order
  if (kh > 0) {
    float* x = xch + static_cast<int64_t>(((kh - 1) * kMT + mt) * 32 + lane) * kNT * 4;
#pragma unroll
    for (int nt = 0; nt < kNT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) x[nt * 4 + q] = acc[nt][q];
  }
  __syncthreads();
  if (kh > 0) return;
#pragma unroll
  for (int j = 0; j < kKP - 1; ++j) {  // (((p0 + p1) + p2) + ...), fixed order
    const float* x = xch + static_cast<int64_t>((j * kMT + mt) * 32 + lane) * kNT * 4;
#pragma unroll
    for (int nt = 0; nt < kNT; ++nt)
#pragma unroll
      for (int q = 0; q < 4; ++q) acc[nt][q] = __fadd_rn(acc[nt][q], x[nt * 4 + q]);
  }
  // finish: lane holds rows g / g + 8, columns 8 nt + 2t, + 1
#pragma unroll
  for (int h = 0; h < 2; ++h) {
    const int m = row0 + g + 8 * h;
    if (m >= a.M) continue;
    const int br = 16 * mt + g + 8 * h;  // block row
    const float sig = sig_fin[h];
#pragma unroll
    for (int nt = 0; nt < kNT; ++nt)
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const int c = 8 * nt + 2 * t + e;
        if (c >= N) continue;
        const float s = acc[nt][2 * h + e];
        if (a.mode == 0) {
          a.out[static_cast<int64_t>(m) * a.ld_out + c] = s;
          continue;
        }
        const float yv = __fadd_rn(s, a.bias[c]);
        const float th = tanhf(yv);
        float act = __fadd_rn(a.mid, __fmul_rn(a.half, th));
        if (a.tanh_out) a.tanh_out[static_cast<int64_t>(m) * a.ld_tanh + c] = th;
        if (a.noise_state) {
          if (sig > 0.0f) act = __fadd_rn(act, __fadd_rn(__fmul_rn(sz[br * kNT * 8 + c], sig), 0.0f));
          if (act < a.low) act = a.low;
          if (act > a.high) act = a.high;
        }
        a.out[static_cast<int64_t>(m) * a.ld_out + c] = act;
      }
  }
}

}  // namespace pqlg::head
