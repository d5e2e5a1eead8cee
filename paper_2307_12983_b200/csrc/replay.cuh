// Device replay path: n-step assembly fused with the ring insert, the state
// ring, and Philox-driven minibatch sampling fused with observation
// normalization.  All are HBM-bound copy kernels: one warp per row, lanes
// stride the row so every access is a coalesced 128-byte segment.
//
// Reference semantics (bit-exact):
//   NStepAssembler::push_step / push_env / emit   nstep.hpp:58-118
//   ReplayBuffer::insert / sample                 replay_buffer.hpp:33-69
//   StateBuffer::insert / sample                  replay_buffer.hpp:93-112
//   RunningNormalizer::apply_stats + normalize_clip  normalizer.hpp:56-70,
//                                                 scalar.hpp:93-106
#pragma once

#include "pdl.cuh"
#include <cstdint>

#include "rng.cuh"

namespace pqlg::replay {

// SoA ring on device (replay_buffer.hpp:79-80); rows padded to `ld_*`.
struct Ring {
  float* obs;
  float* act;
  float* boot;
  float* ret;
  float* eff;
  int64_t ld_obs, ld_act;
  int D, A;
  uint64_t capacity;
  uint64_t* state;  // device: [0] cursor, [1] count
};

struct StateRing {
  float* obs;
  int64_t ld;
  int D;
  uint64_t capacity;
  uint64_t* state;  // [0] cursor, [1] count
};

// Per-env n-step windows (nstep.hpp:120-125).
struct Window {
  float* obs;  // [N*n x ld_obs]
  float* act;  // [N*n x ld_act]
  float* rew;  // [N*n]
  uint32_t* head;
  uint32_t* count;
  int64_t ld_obs, ld_act;
  int N, n;
  float gamma;
};

// StepSlice (messages.hpp:31-35) on device.
struct Slice {
  const float* obs;
  const float* act;
  const float* boot;
  const float* rew;
  const uint8_t* term;
  const uint8_t* trunc;
  int64_t ld_obs, ld_act;
};

// Normalization constants in fp32 (normalizer.hpp:62-66), identity flag.
struct Norm {
  const float* mean;
  const float* inv;
  const int* identity;  // device flag: count <= 1
};

// Destination of a gathered minibatch.  obs/boot rows are normalized.
struct Gather {
  float* obs;
  int64_t ld_obs;
  float* act;  // may alias obs + D (critic input [obs | act])
  int64_t ld_act;
  float* boot;
  int64_t ld_boot;
  float* ret;
  float* eff;
};

constexpr int kScanBlock = 1024;
constexpr int kWarpsPerBlock = 8;

// Warp-cooperative row copy.  With 16-byte aligned rows whose strides leave
// room for the padded tail (wide = true), lanes move float4s; otherwise a
// scalar loop.
__device__ __forceinline__ void copy_row(float* __restrict__ dst, const float* __restrict__ src,
                                         int n, bool wide, int lane) {
  if (wide) {
    const int n4 = (n + 3) >> 2;
    const float4* s4 = reinterpret_cast<const float4*>(src);
    float4* d4 = reinterpret_cast<float4*>(dst);
    for (int j = lane; j < n4; j += 32) d4[j] = s4[j];
  } else {
    for (int d = lane; d < n; d += 32) dst[d] = src[d];
  }
}

// A padded row of up to 256 floats held by one warp: 2 float4 per lane.
struct WarpRow {
  float4 v[2];
};
__device__ __forceinline__ WarpRow load_row(const float* __restrict__ src, int n, int lane) {
  const int n4 = (n + 3) >> 2;
  const float4* s4 = reinterpret_cast<const float4*>(src);
  WarpRow r;
  r.v[0] = lane < n4 ? s4[lane] : make_float4(0.f, 0.f, 0.f, 0.f);
  r.v[1] = lane + 32 < n4 ? s4[lane + 32] : make_float4(0.f, 0.f, 0.f, 0.f);
  return r;
}
__device__ __forceinline__ void store_row(float* __restrict__ dst, const WarpRow& r, int n,
                                          int lane) {
  const int n4 = (n + 3) >> 2;
  float4* d4 = reinterpret_cast<float4*>(dst);
  if (lane < n4) d4[lane] = r.v[0];
  if (lane + 32 < n4) d4[lane + 32] = r.v[1];
}

__device__ __forceinline__ bool aligned16(const void* p, int64_t ld) {
  return ((reinterpret_cast<uintptr_t>(p) & 15) == 0) && ((ld & 3) == 0);
}

__device__ __forceinline__ float normalize1(float x, float mean, float inv) {
  float z = __fmul_rn(__fsub_rn(x, mean), inv);
  if (z > 5.0f) z = 5.0f;
  if (z < -5.0f) z = -5.0f;
  return z;
}

// Emit count of env e for this step (0..n): nstep.hpp:78-92.
__device__ __forceinline__ int emit_count(uint32_t count, int n, bool done) {
  int c = static_cast<int>(count) + 1;
  int emits = 0;
  if (c == n) {
    emits = 1;
    c -= 1;
  }
  if (done) emits += c;
  return emits;
}

// K1: per-env emit counts, block-exclusive offsets and block totals.
static __global__ void nstep_count_kernel(Window w, Slice s, uint32_t* offs, uint32_t* block_sums) {
  pdl::entry();
  __shared__ uint32_t warp_tot[kScanBlock / 32];
  const int e = blockIdx.x * kScanBlock + threadIdx.x;
  uint32_t c = 0;
  if (e < w.N) {
    const bool done = (s.term[e] != 0) || (s.trunc[e] != 0);
    c = static_cast<uint32_t>(emit_count(w.count[e], w.n, done));
  }
  // warp-inclusive scan
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t v = c;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t t = __shfl_up_sync(0xffffffffu, v, d);
    if (lane >= d) v += t;
  }
  if (lane == 31) warp_tot[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint32_t t = warp_tot[lane];
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t u = __shfl_up_sync(0xffffffffu, t, d);
      if (lane >= d) t += u;
    }
    warp_tot[lane] = t;  // inclusive over warps
  }
  __syncthreads();
  const uint32_t warp_prefix = wid ? warp_tot[wid - 1] : 0u;
  if (e < w.N) offs[e] = warp_prefix + v - c;
  if (threadIdx.x == kScanBlock - 1) block_sums[blockIdx.x] = warp_tot[31];
}

// K2: one warp per env.  Writes the new window slot, then emits this step's
// records in reference order straight into the ring.
static __global__ void nstep_emit_kernel(Window w, Slice s, float reward_scale, Ring ring,
                                  const uint32_t* offs, const uint32_t* block_sums,
                                  int n_blocks) {
  pdl::entry();
  const int lane = threadIdx.x & 31;
  const int e = blockIdx.x * kWarpsPerBlock + (threadIdx.x >> 5);
  if (e >= w.N) return;
  // every independent load first (nothing below aliases them until the
  // window write), so their latencies overlap
  const uint32_t h0 = w.head[e], c0 = w.count[e];
  const bool term = s.term[e] != 0;
  const bool done = term || (s.trunc[e] != 0);
  const float rew_e = s.rew[e];
  const uint32_t off_e = offs[e];
  const uint64_t cursor0 = ring.state[0];
  float my_rew = lane < w.n ? w.rew[static_cast<size_t>(e) * w.n + lane] : 0.0f;
  // global offset of this env's first record and the step total
  uint32_t before = 0, total = 0;
  const int my_block = e / kScanBlock;
  for (int b = lane; b < n_blocks; b += 32) {
    const uint32_t v = block_sums[b];
    total += v;
    if (b < my_block) before += v;
  }
#pragma unroll
  for (int d = 16; d > 0; d >>= 1) {
    total += __shfl_xor_sync(0xffffffffu, total, d);
    before += __shfl_xor_sync(0xffffffffu, before, d);
  }
  const uint64_t base = static_cast<uint64_t>(before) + off_e;
  const int n = w.n, D = ring.D, A = ring.A;
  uint32_t h = h0;
  uint32_t c = c0;
  // float4 paths when the slice rows are 16B aligned with padded strides
  const bool wide_o = aligned16(s.obs, s.ld_obs) && aligned16(s.boot, s.ld_obs) &&
                      s.ld_obs >= ((D + 3) & ~3);
  const bool wide_a = aligned16(s.act, s.ld_act) && s.ld_act >= ((A + 3) & ~3);
  // push: window slot (head + count) % n; lane k keeps the window reward of
  // slot k in a register (rewards are read back by shuffle, not from memory)
  const uint32_t slot = (h + c) % n;
  const float new_rew = __fmul_rn(rew_e, reward_scale);
  if (lane == static_cast<int>(slot)) my_rew = new_rew;
  // Common case (padded rows, D <= 256, A <= 128): every row this env moves
  // -- the new obs/act, the window front (the first emitted record's
  // obs/act) and the boot obs -- is loaded before anything is stored, so
  // the warp pays one memory round trip instead of one per row.
  const bool fast = wide_o && wide_a && D <= 256 && A <= 128;
  const bool will_emit = (c + 1 == static_cast<uint32_t>(n)) || done;
  bool first_preloaded = false;
  WarpRow fo{}, fa{}, bo{};
  {
    const size_t wrow = static_cast<size_t>(e) * n + slot;
    if (fast) {
      const WarpRow no = load_row(s.obs + static_cast<size_t>(e) * s.ld_obs, D, lane);
      const WarpRow na = load_row(s.act + static_cast<size_t>(e) * s.ld_act, A, lane);
      if (will_emit) {
        const size_t front = static_cast<size_t>(e) * n + h;
        bo = load_row(s.boot + static_cast<size_t>(e) * s.ld_obs, D, lane);
        if (front == wrow) {  // empty window: the front is the record pushed now
          fo = no;
          fa = na;
        } else {
          fo = load_row(w.obs + front * w.ld_obs, D, lane);
          fa = load_row(w.act + front * w.ld_act, A, lane);
        }
        first_preloaded = true;
      }
      store_row(w.obs + wrow * w.ld_obs, no, D, lane);
      store_row(w.act + wrow * w.ld_act, na, A, lane);
    } else {
      copy_row(w.obs + wrow * w.ld_obs, s.obs + static_cast<size_t>(e) * s.ld_obs, D, wide_o, lane);
      copy_row(w.act + wrow * w.ld_act, s.act + static_cast<size_t>(e) * s.ld_act, A, wide_a, lane);
    }
    if (lane == 0) w.rew[wrow] = new_rew;
  }
  __syncwarp();
  c += 1;

  uint32_t j = 0;
  auto emit = [&](uint32_t m, bool terminated) {
    const bool use_pre = first_preloaded;  // only the step's first record was preloaded
    first_preloaded = false;
    float g = 0.0f, disc = 1.0f;
    for (uint32_t k = 0; k < m; ++k) {
      const float r = __shfl_sync(0xffffffffu, my_rew, static_cast<int>((h + k) % n));
      g = __fadd_rn(g, __fmul_rn(disc, r));
      disc = __fmul_rn(disc, w.gamma);
    }
    const uint64_t rec = base + j++;
    // records overwritten within this same insert are skipped (ring order)
    if (rec + ring.capacity < total) return;
    const uint64_t p = (cursor0 + rec) % ring.capacity;
    const size_t front = static_cast<size_t>(e) * n + h;
    if (use_pre) {  // rows loaded up front (first record of the step)
      store_row(ring.obs + p * ring.ld_obs, fo, D, lane);
      store_row(ring.act + p * ring.ld_act, fa, A, lane);
      store_row(ring.boot + p * ring.ld_obs, bo, D, lane);
    } else {
      // window and ring rows are padded to 16 bytes by construction
      copy_row(ring.obs + p * ring.ld_obs, w.obs + front * w.ld_obs, D, true, lane);
      copy_row(ring.act + p * ring.ld_act, w.act + front * w.ld_act, A, true, lane);
      copy_row(ring.boot + p * ring.ld_obs, s.boot + static_cast<size_t>(e) * s.ld_obs, D, wide_o,
               lane);
    }
    if (lane == 0) {
      ring.ret[p] = g;
      ring.eff[p] = terminated ? 0.0f : disc;
    }
  };

  if (c == static_cast<uint32_t>(n)) {
    emit(n, term);  // terminated && done == terminated
    h = (h + 1) % n;
    c -= 1;
  }
  if (done) {
    while (c > 0) {
      emit(c, term);
      h = (h + 1) % n;
      c -= 1;
    }
    h = 0;
  }
  if (lane == 0) {
    w.head[e] = h;
    w.count[e] = c;
  }
}

// K3: cursor = (cursor + total) % cap; count = min(count + total, cap).
static __global__ void ring_advance_kernel(uint64_t* state, uint64_t capacity, const uint32_t* sums,
                                    int n_sums, uint64_t extra) {
  pdl::entry();
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  uint64_t total = extra;
  for (int b = 0; b < n_sums; ++b) total += sums[b];
  state[0] = (state[0] + total) % capacity;
  const uint64_t c = state[1] + total;
  state[1] = c < capacity ? c : capacity;
}

// Direct insert of an assembled batch (ReplayBuffer::insert).  One warp per
// row; rows that a later row of the same batch overwrites are skipped.
static __global__ void ring_insert_kernel(Ring ring, const float* obs, const float* act,
                                   const float* boot, const float* ret, const float* eff,
                                   int64_t ld_obs, int64_t ld_act, uint64_t n) {
  pdl::entry();
  const int lane = threadIdx.x & 31;
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= n || r + ring.capacity < n) return;
  const uint64_t p = (ring.state[0] + r) % ring.capacity;
  for (int d = lane; d < ring.D; d += 32) {
    ring.obs[p * ring.ld_obs + d] = obs[r * ld_obs + d];
    ring.boot[p * ring.ld_obs + d] = boot[r * ld_obs + d];
  }
  for (int d = lane; d < ring.A; d += 32) ring.act[p * ring.ld_act + d] = act[r * ld_act + d];
  if (lane == 0) {
    ring.ret[p] = ret[r];
    ring.eff[p] = eff[r];
  }
}

static __global__ void state_insert_kernel(StateRing ring, const float* rows, int64_t ld, uint64_t n) {
  pdl::entry();
  const int lane = threadIdx.x & 31;
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= n || r + ring.capacity < n) return;
  const uint64_t p = (ring.state[0] + r) % ring.capacity;
  const bool wide = aligned16(rows, ld) && ld >= ((ring.D + 3) & ~3);
  copy_row(ring.obs + p * ring.ld, rows + r * ld, ring.D, wide, lane);
}

// Synthetic pre-fill: obs/boot ~ N(0,1), act ~ U(-1,1),
// ret ~ 0.1 N(0,1), eff = disc except 1/terminal_every rows (terminal, 0).
// Philox keyed by `seed`; one warp per row.  Used by the benchmarks to fill
// a 5M-record ring without a host round trip.
__device__ __forceinline__ float philox_normal(uint64_t key, uint64_t ctr) {
  const uint64_t x = rng::philox_draw(key, ctr);
  const float u1 = (static_cast<float>(x >> 40) + 0.5f) * 0x1p-24f;
  const float u2 = static_cast<float>((x >> 16) & 0xFFFFFFu) * 0x1p-24f;
  return sqrtf(-2.0f * logf(u1)) * cospif(2.0f * u2);
}

static __global__ void ring_fill_kernel(Ring ring, uint64_t n, uint64_t seed, float disc,
                                        uint32_t terminal_every) {
  pdl::entry();
  const int lane = threadIdx.x & 31;
  const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kWarpsPerBlock + (threadIdx.x >> 5);
  if (r >= n) return;
  const uint64_t p = (ring.state[0] + r) % ring.capacity;
  const uint64_t base = r * 1024;
  for (int d = lane; d < ring.D; d += 32) {
    ring.obs[p * ring.ld_obs + d] = philox_normal(seed, base + d);
    ring.boot[p * ring.ld_obs + d] = philox_normal(seed, base + 512 + d);
  }
  for (int d = lane; d < ring.A; d += 32) {
    const uint64_t x = rng::philox_draw(seed ^ 0x5bd1e995ull, base + d);
    ring.act[p * ring.ld_act + d] = static_cast<float>(x >> 40) * 0x1p-23f - 1.0f;
  }
  if (lane == 0) {
    ring.ret[p] = 0.1f * philox_normal(seed ^ 0x27d4eb2full, r);
    ring.eff[p] = (terminal_every && (r % terminal_every) == 0) ? 0.0f : disc;
  }
}

// ---------------------------------------------------------------- sampling
// Sampler state on device: Philox key, counter, rejection flag.
struct SamplerState {
  uint64_t key;
  uint64_t counter;
  uint32_t reject;
  uint32_t ticket;  // blocks finished in the current sampling launch
};

// idx for row r: host_idx (mt19937-compat mode) or Philox + Lemire.
__device__ __forceinline__ uint64_t sample_index(const SamplerState* ss, const uint64_t* host_idx,
                                                 uint64_t count, uint64_t r, bool& reject) {
  reject = false;
  if (host_idx) return host_idx[r];
  return rng::lemire_step(rng::philox_draw(ss->key, ss->counter + r), count, reject);
}

__device__ __forceinline__ void gather_row(const Ring& ring, const Norm& norm, const Gather& g,
                                           uint64_t i, uint64_t r, int lane) {
  const bool ident = *norm.identity != 0;
  const float* __restrict__ so = ring.obs + i * ring.ld_obs;
  const float* __restrict__ sb = ring.boot + i * ring.ld_obs;
  float* __restrict__ dobs = g.obs + r * g.ld_obs;
  float* __restrict__ dboot = g.boot + r * g.ld_boot;
  int d0 = 0;
  if (ring.D <= 256) {  // all loads of the row in flight before any store
    float x[8], y[8], mu[8], iv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int d = lane + 32 * u;
      x[u] = d < ring.D ? __ldg(so + d) : 0.0f;
      y[u] = d < ring.D ? __ldg(sb + d) : 0.0f;
      mu[u] = (d < ring.D && !ident) ? norm.mean[d] : 0.0f;
      iv[u] = (d < ring.D && !ident) ? norm.inv[d] : 1.0f;
    }
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int d = lane + 32 * u;
      if (d < ring.D) {
        float xx = x[u], yy = y[u];
        if (!ident) {
          xx = normalize1(xx, mu[u], iv[u]);
          yy = normalize1(yy, mu[u], iv[u]);
        }
        dobs[d] = xx;
        dboot[d] = yy;
      }
    }
    d0 = ring.D;
  }
  for (int d = d0 + lane; d < ring.D; d += 32) {
    float x = so[d], y = sb[d];
    if (!ident) {
      const float mu = norm.mean[d], iv = norm.inv[d];
      x = normalize1(x, mu, iv);
      y = normalize1(y, mu, iv);
    }
    dobs[d] = x;
    dboot[d] = y;
  }
  const float* sa = ring.act + i * ring.ld_act;
  float* da = g.act + r * g.ld_act;
  for (int d = lane; d < ring.A; d += 32) da[d] = sa[d];
  if (lane == 0) {
    g.ret[r] = ring.ret[i];
    g.eff[r] = ring.eff[i];
  }
}

// The last block of a sampling launch (atomic ticket in SamplerState::ticket)
// advances the Philox counter by B, or -- when any draw hit Lemire's
// rejection zone (probability ~count/2^64 per draw) -- redoes the whole batch
// sequentially with libstdc++'s redraw loop and advances the counter by the
// draws consumed.  redo(i, r, lane) gathers row r from ring index i.
template <class Redo>
__device__ __forceinline__ void finish_sample(SamplerState* ss, const uint64_t* host_idx,
                                              uint64_t count, uint64_t B, Redo&& redo) {
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(&ss->ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last || threadIdx.x >= 32) return;
  __threadfence();
  const int lane = threadIdx.x;
  const volatile SamplerState* vs = ss;
  if (!host_idx) {
    if (vs->reject == 0) {
      if (lane == 0) ss->counter += B;
    } else {
      uint64_t ctr = ss->counter;
      for (uint64_t r = 0; r < B; ++r) {
        uint64_t i = 0;
        if (lane == 0) {
          bool reject = true;
          while (reject) i = rng::lemire_step(rng::philox_draw(ss->key, ctr++), count, reject);
        }
        i = __shfl_sync(0xffffffffu, i, 0);
        redo(i, r, lane);
      }
      if (lane == 0) {
        ss->counter = ctr;
        ss->reject = 0;
      }
    }
  }
  if (lane == 0) ss->ticket = 0;
}

// ReplayBuffer::sample fused with apply_stats on obs and boot_obs.  A block
// owns kSampleRows rows: its first warp draws their indices (one Philox draw
// per lane, in parallel), then each warp gathers kRowsPerWarp rows with all
// of their loads in flight before any store (the gather is latency-bound:
// random ~850 B rows).  The ticketed finish above ends the launch.
constexpr int kSampleRows = 32;
constexpr int kRowsPerWarp = kSampleRows / kWarpsPerBlock;  // 4

__device__ __forceinline__ void draw_block_indices(const SamplerState* ss,
                                                   const uint64_t* host_idx, uint64_t count,
                                                   uint64_t B, uint64_t* s_idx) {
  if (threadIdx.x < kSampleRows) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kSampleRows + threadIdx.x;
    uint64_t i = 0;
    if (r < B) {
      bool reject = false;
      i = sample_index(ss, host_idx, count, r, reject);
      if (reject) atomicOr(const_cast<uint32_t*>(&ss->reject), 1u);
    }
    s_idx[threadIdx.x] = i;
  }
  __syncthreads();
}

// Index-only sampling (test hook pqlg_k_sample_indices): the sampler's own
// parallel draw and ticketed finish (including the sequential Lemire redo)
// over a virtual live count, the indices written to `out` instead of rows
// being gathered.  With count just above 2^63 about half the draws land in
// the rejection zone, so the redo path runs.
static __global__ void __launch_bounds__(32 * kWarpsPerBlock)
    sample_indices_kernel(SamplerState* ss, uint64_t count, uint64_t B, uint64_t* out) {
  __shared__ uint64_t s_idx[kSampleRows];
  pdl::entry();
  draw_block_indices(ss, nullptr, count, B, s_idx);
  if (threadIdx.x < kSampleRows) {
    const uint64_t r = static_cast<uint64_t>(blockIdx.x) * kSampleRows + threadIdx.x;
    if (r < B) out[r] = s_idx[threadIdx.x];
  }
  finish_sample(ss, nullptr, count, B, [&](uint64_t i, uint64_t r, int ln) {
    if (ln == 0) out[r] = i;
  });
}

static __global__ void __launch_bounds__(32 * kWarpsPerBlock)
    replay_sample_kernel(const __grid_constant__ Ring ring, const __grid_constant__ Norm norm,
                         const __grid_constant__ Gather g, SamplerState* ss,
                         const uint64_t* host_idx, uint64_t B, int early) {
  __shared__ uint64_t s_idx[kSampleRows];
  // early (inside the learner's update graph, where the preceding kernel is
  // the previous update's Adam, which touches none of the sampler state, the
  // ring or the gather buffers): let the next kernel launch and start the
  // gather at once, overlapping that kernel; wait for it only before exiting,
  // so this grid's completion still implies its predecessor's
  if (early) pdl::trigger();
  else pdl::entry();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint64_t count = ring.state[1];
  draw_block_indices(ss, host_idx, count, B, s_idx);
  const uint64_t rb = static_cast<uint64_t>(blockIdx.x) * kSampleRows + w * kRowsPerWarp;
  const bool vec4 = ring.D <= 256 && (ring.ld_obs & 3) == 0 && (g.ld_obs & 3) == 0 &&
                    (g.ld_boot & 3) == 0 &&
                    ((reinterpret_cast<uintptr_t>(ring.obs) | reinterpret_cast<uintptr_t>(ring.boot) |
                      reinterpret_cast<uintptr_t>(g.obs) | reinterpret_cast<uintptr_t>(g.boot)) & 15) == 0;
  if (vec4) {
    // 16-byte rows: lane l gathers quads l and l + 32 of each row (all loads
    // of the warp's rows in flight before any store); the last, partial quad
    // is stored element-wise (the critic input's action columns follow the
    // observation at column D)
    const bool ident = *norm.identity != 0;
    const int Q = (ring.D + 3) >> 2;
    float4 x[kRowsPerWarp][2], y[kRowsPerWarp][2];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t i = s_idx[w * kRowsPerWarp + k];
      const float4* so = reinterpret_cast<const float4*>(ring.obs + i * ring.ld_obs);
      const float4* sb = reinterpret_cast<const float4*>(ring.boot + i * ring.ld_obs);
      const bool ok = rb + k < B;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = lane + 32 * u;
        x[k][u] = (ok && q < Q) ? __ldg(so + q) : make_float4(0.f, 0.f, 0.f, 0.f);
        y[k][u] = (ok && q < Q) ? __ldg(sb + q) : make_float4(0.f, 0.f, 0.f, 0.f);
      }
    }
    float av[kRowsPerWarp], rv[kRowsPerWarp], ev[kRowsPerWarp];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t i = s_idx[w * kRowsPerWarp + k];
      const bool ok = rb + k < B;
      av[k] = (ok && lane < ring.A) ? __ldg(ring.act + i * ring.ld_act + lane) : 0.0f;
      rv[k] = (ok && lane == 0) ? __ldg(ring.ret + i) : 0.0f;
      ev[k] = (ok && lane == 0) ? __ldg(ring.eff + i) : 0.0f;
    }
    float mu[2][4], iv[2][4];
#pragma unroll
    for (int u = 0; u < 2; ++u)
#pragma unroll
      for (int c = 0; c < 4; ++c) {
        const int d = 4 * (lane + 32 * u) + c;
        mu[u][c] = (d < ring.D && !ident) ? norm.mean[d] : 0.0f;
        iv[u][c] = (d < ring.D && !ident) ? norm.inv[d] : 1.0f;
      }
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t r = rb + k;
      if (r >= B) break;
      float* dobs = g.obs + r * g.ld_obs;
      float* dboot = g.boot + r * g.ld_boot;
#pragma unroll
      for (int u = 0; u < 2; ++u) {
        const int q = lane + 32 * u;
        if (q >= Q) continue;
        float xx[4] = {x[k][u].x, x[k][u].y, x[k][u].z, x[k][u].w};
        float yy[4] = {y[k][u].x, y[k][u].y, y[k][u].z, y[k][u].w};
        if (!ident) {
#pragma unroll
          for (int c = 0; c < 4; ++c) {
            xx[c] = normalize1(xx[c], mu[u][c], iv[u][c]);
            yy[c] = normalize1(yy[c], mu[u][c], iv[u][c]);
          }
        }
        const int d0 = 4 * q;
        if (d0 + 4 <= ring.D) {
          *reinterpret_cast<float4*>(dobs + d0) = make_float4(xx[0], xx[1], xx[2], xx[3]);
          *reinterpret_cast<float4*>(dboot + d0) = make_float4(yy[0], yy[1], yy[2], yy[3]);
        } else {
#pragma unroll
          for (int c = 0; c < 4; ++c)
            if (d0 + c < ring.D) {
              dobs[d0 + c] = xx[c];
              dboot[d0 + c] = yy[c];
            }
        }
      }
      if (lane < ring.A) g.act[r * g.ld_act + lane] = av[k];
      if (lane == 0) {
        g.ret[r] = rv[k];
        g.eff[r] = ev[k];
      }
    }
    if (ring.A > 32) {  // wide actions: the generic path for the columns >= 32
      for (int k = 0; k < kRowsPerWarp && rb + k < B; ++k) {
        const uint64_t i = s_idx[w * kRowsPerWarp + k];
        for (int d = 32 + lane; d < ring.A; d += 32)
          g.act[(rb + k) * g.ld_act + d] = ring.act[i * ring.ld_act + d];
      }
    }
  } else if (ring.D <= 256) {
    const bool ident = *norm.identity != 0;
    float x[kRowsPerWarp][8], y[kRowsPerWarp][8];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t i = s_idx[w * kRowsPerWarp + k];
      const float* so = ring.obs + i * ring.ld_obs;
      const float* sb = ring.boot + i * ring.ld_obs;
      const bool ok = rb + k < B;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int d = lane + 32 * u;
        x[k][u] = (ok && d < ring.D) ? __ldg(so + d) : 0.0f;
        y[k][u] = (ok && d < ring.D) ? __ldg(sb + d) : 0.0f;
      }
    }
    float av[kRowsPerWarp], rv[kRowsPerWarp], ev[kRowsPerWarp];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t i = s_idx[w * kRowsPerWarp + k];
      const bool ok = rb + k < B;
      av[k] = (ok && lane < ring.A) ? __ldg(ring.act + i * ring.ld_act + lane) : 0.0f;
      rv[k] = (ok && lane == 0) ? __ldg(ring.ret + i) : 0.0f;
      ev[k] = (ok && lane == 0) ? __ldg(ring.eff + i) : 0.0f;
    }
    float mu[8], iv[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      const int d = lane + 32 * u;
      mu[u] = (d < ring.D && !ident) ? norm.mean[d] : 0.0f;
      iv[u] = (d < ring.D && !ident) ? norm.inv[d] : 1.0f;
    }
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t r = rb + k;
      if (r >= B) break;
      float* dobs = g.obs + r * g.ld_obs;
      float* dboot = g.boot + r * g.ld_boot;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int d = lane + 32 * u;
        if (d < ring.D) {
          float xx = x[k][u], yy = y[k][u];
          if (!ident) {
            xx = normalize1(xx, mu[u], iv[u]);
            yy = normalize1(yy, mu[u], iv[u]);
          }
          dobs[d] = xx;
          dboot[d] = yy;
        }
      }
      if (lane < ring.A) g.act[r * g.ld_act + lane] = av[k];
      if (lane == 0) {
        g.ret[r] = rv[k];
        g.eff[r] = ev[k];
      }
    }
    if (ring.A > 32) {  // wide actions: the generic path for the columns >= 32
      for (int k = 0; k < kRowsPerWarp && rb + k < B; ++k) {
        const uint64_t i = s_idx[w * kRowsPerWarp + k];
        for (int d = 32 + lane; d < ring.A; d += 32)
          g.act[(rb + k) * g.ld_act + d] = ring.act[i * ring.ld_act + d];
      }
    }
  } else {
    for (int k = 0; k < kRowsPerWarp && rb + k < B; ++k)
      gather_row(ring, norm, g, s_idx[w * kRowsPerWarp + k], rb + k, lane);
  }
  finish_sample(ss, host_idx, count, B,
                [&](uint64_t i, uint64_t rr, int ln) { gather_row(ring, norm, g, i, rr, ln); });
  if (early) pdl::wait();
}

__device__ __forceinline__ void gather_state(const StateRing& ring, const Norm& norm, float* out,
                                             int64_t ld_out, uint64_t i, uint64_t r, int lane) {
  const bool ident = *norm.identity != 0;
  const float* so = ring.obs + i * ring.ld;
  float* d = out + r * ld_out;
  for (int k = lane; k < ring.D; k += 32) {
    float x = so[k];
    if (!ident) x = normalize1(x, norm.mean[k], norm.inv[k]);
    d[k] = x;
  }
}

// StateBuffer::sample fused with apply_stats (block layout as above).
static __global__ void __launch_bounds__(32 * kWarpsPerBlock)
    state_sample_kernel(StateRing ring, Norm norm, float* out, int64_t ld_out, SamplerState* ss,
                        const uint64_t* host_idx, uint64_t B, int early) {
  __shared__ uint64_t s_idx[kSampleRows];
  if (early) pdl::trigger();  // as replay_sample_kernel
  else pdl::entry();
  const int lane = threadIdx.x & 31;
  const int w = threadIdx.x >> 5;
  const uint64_t count = ring.state[1];
  draw_block_indices(ss, host_idx, count, B, s_idx);
  const uint64_t rb = static_cast<uint64_t>(blockIdx.x) * kSampleRows + w * kRowsPerWarp;
  if (ring.D <= 256) {
    const bool ident = *norm.identity != 0;
    float x[kRowsPerWarp][8];
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const float* so = ring.obs + s_idx[w * kRowsPerWarp + k] * ring.ld;
      const bool ok = rb + k < B;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int d = lane + 32 * u;
        x[k][u] = (ok && d < ring.D) ? __ldg(so + d) : 0.0f;
      }
    }
#pragma unroll
    for (int k = 0; k < kRowsPerWarp; ++k) {
      const uint64_t r = rb + k;
      if (r >= B) break;
      float* d_out = out + r * ld_out;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int d = lane + 32 * u;
        if (d < ring.D) d_out[d] = ident ? x[k][u] : normalize1(x[k][u], norm.mean[d], norm.inv[d]);
      }
    }
  } else {
    for (int k = 0; k < kRowsPerWarp && rb + k < B; ++k)
      gather_state(ring, norm, out, ld_out, s_idx[w * kRowsPerWarp + k], rb + k, lane);
  }
  finish_sample(ss, host_idx, count, B, [&](uint64_t i, uint64_t rr, int ln) {
    gather_state(ring, norm, out, ld_out, i, rr, ln);
  });
  if (early) pdl::wait();
}

}  // namespace pqlg::replay
