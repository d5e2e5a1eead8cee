// Device restatements of the reference's random streams, bit-exact:
//   splitmix64 / derive_seed              proj/include/pql/rng.hpp:20-30
//   SplitMixEngine                        proj/include/pql/vecenv/vecenv.hpp:33-39
//   uniform_int_distribution<size_t>      libstdc++ bits/uniform_int_dist.h:257-276
//   normal_distribution<float> (polar)    libstdc++ bits/random.tcc:1811-1844
//   generate_canonical<float>             libstdc++ bits/random.tcc:3349-3381
//   logf                                  glibc 2.39 sysdeps/ieee754/flt-32/e_logf.c
// plus Philox4x32-10, the counter-based generator that replaces the
// reference's sequential mt19937_64 for sampling on the GPU.
#pragma once

#include <cstdint>

namespace pqlg::rng {

enum Stream : uint64_t { kEnv = 1, kNoise = 2, kInit = 3, kSample = 4, kEval = 5, kSac = 6 };

__host__ __device__ __forceinline__ uint64_t splitmix64(uint64_t x) {
  x += 0x9e3779b97f4a7c15ull;
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}

__host__ __device__ __forceinline__ uint64_t derive_seed(uint64_t master, uint64_t stream,
                                                         uint64_t index) {
  const uint64_t s = splitmix64(master ^ (stream * 0xd6e8feb86659fd93ull));
  return splitmix64(s ^ splitmix64(index));
}

// Philox4x32-10 draw `counter` of stream `key`: out[0] | out[1] << 32.
__host__ __device__ __forceinline__ uint64_t philox_draw(uint64_t key, uint64_t counter) {
  uint32_t c0 = static_cast<uint32_t>(counter), c1 = static_cast<uint32_t>(counter >> 32);
  uint32_t c2 = 0, c3 = 0;
  uint32_t k0 = static_cast<uint32_t>(key), k1 = static_cast<uint32_t>(key >> 32);
#pragma unroll
  for (int r = 0; r < 10; ++r) {
    if (r > 0) {
      k0 += 0x9E3779B9u;
      k1 += 0xBB67AE85u;
    }
    const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c0;
    const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c2;
    const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c1 ^ k0;
    const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c3 ^ k1;
    c1 = static_cast<uint32_t>(p1);
    c3 = static_cast<uint32_t>(p0);
    c0 = n0;
    c2 = n2;
  }
  return static_cast<uint64_t>(c0) | (static_cast<uint64_t>(c1) << 32);
}

// One Lemire step: returns the index for draw x and sets `reject` when the
// draw falls in the rejection zone (libstdc++ would redraw).
__host__ __device__ __forceinline__ uint64_t lemire_step(uint64_t x, uint64_t range,
                                                         bool& reject) {
#if defined(__CUDA_ARCH__)
  const uint64_t hi = __umul64hi(x, range);
  const uint64_t lo = x * range;
#else
  const unsigned __int128 p = static_cast<unsigned __int128>(x) * range;
  const uint64_t hi = static_cast<uint64_t>(p >> 64), lo = static_cast<uint64_t>(p);
#endif
  reject = false;
  if (lo < range) {
    const uint64_t threshold = (0 - range) % range;
    reject = lo < threshold;
  }
  return hi;
}

// ------------------------------------------------------ glibc 2.39 logf
// Table of glibc e_logf_data.c (LOGF_TABLE_BITS = 4): {invc, logc}.  In
// global memory (read through the L1): a constexpr array indexed by a
// per-lane value would be rebuilt on every call's stack.
__device__ static const double2 kLogfTab[16] = {
    {0x1.661ec79f8f3bep+0, -0x1.57bf7808caadep-2}, {0x1.571ed4aaf883dp+0, -0x1.2bef0a7c06ddbp-2},
    {0x1.49539f0f010bp+0, -0x1.01eae7f513a67p-2},  {0x1.3c995b0b80385p+0, -0x1.b31d8a68224e9p-3},
    {0x1.30d190c8864a5p+0, -0x1.6574f0ac07758p-3}, {0x1.25e227b0b8eap+0, -0x1.1aa2bc79c81p-3},
    {0x1.1bb4a4a1a343fp+0, -0x1.a4e76ce8c0e5ep-4}, {0x1.12358f08ae5bap+0, -0x1.1973c5a611cccp-4},
    {0x1.0953f419900a7p+0, -0x1.252f438e10c1ep-5}, {0x1p+0, 0x0p+0},
    {0x1.e608cfd9a47acp-1, 0x1.aa5aa5df25984p-5},  {0x1.ca4b31f026aap-1, 0x1.c5e53aa362eb4p-4},
    {0x1.b2036576afce6p-1, 0x1.526e57720db08p-3},  {0x1.9c2d163a1aa2dp-1, 0x1.bc2860d22477p-3},
    {0x1.886e6037841edp-1, 0x1.1058bc8a07ee1p-2},  {0x1.767dcf5534862p-1, 0x1.4043057b6ee09p-2}};

__device__ __forceinline__ float glibc_logf(float x) {
  constexpr double kLn2 = 0x1.62e42fefa39efp-1;
  constexpr double A0 = -0x1.00ea348b88334p-2, A1 = 0x1.5575b0be00b6ap-2,
                   A2 = -0x1.ffffef20a4123p-2;
  uint32_t ix = __float_as_uint(x);
  if (ix == 0x3f800000u) return 0.0f;
  if (ix - 0x00800000u >= 0x7f800000u - 0x00800000u) {
    if (ix * 2 == 0) return -__int_as_float(0x7f800000);
    if (ix == 0x7f800000u) return x;
    if ((ix & 0x80000000u) || ix * 2 >= 0xff000000u) return __int_as_float(0x7fc00000);
    ix = __float_as_uint(__fmul_rn(x, 0x1p23f)) - (23u << 23);
  }
  const uint32_t tmp = ix - 0x3f330000u;
  const int i = static_cast<int>((tmp >> 19) & 15u);
  const int k = static_cast<int32_t>(tmp) >> 23;
  const uint32_t iz = ix - (tmp & (0x1ffu << 23));
  const double z = static_cast<double>(__uint_as_float(iz));
  const double2 t = __ldg(&kLogfTab[i]);
  const double r = __dadd_rn(__dmul_rn(z, t.x), -1.0);
  const double y0 = __dadd_rn(t.y, __dmul_rn(static_cast<double>(k), kLn2));
  const double r2 = __dmul_rn(r, r);
  double y = __dadd_rn(__dmul_rn(A1, r), A2);
  y = __dadd_rn(__dmul_rn(A0, r2), y);
  y = __dadd_rn(__dmul_rn(y, r2), __dadd_rn(y0, r));
  return __double2float_rn(y);
}

// generate_canonical<float> over a SplitMixEngine: float(x) * 2^-64, < 1.
__device__ __forceinline__ float canonical_f32(uint64_t& state) {
  const uint64_t x = splitmix64(state++);
  float u = __fmul_rn(__ull2float_rn(x), 0x1p-64f);
  if (u >= 1.0f) u = __uint_as_float(0x3f7fffffu);  // nextafter(1, 0)
  return u;
}

// One polar pair (normal_distribution<float>): returns y*mult, caches x*mult.
__device__ __forceinline__ float polar_pair(uint64_t& state, float& saved) {
  float x, y, r2;
  do {
    x = __double2float_rn(static_cast<double>(__fmul_rn(2.0f, canonical_f32(state))) - 1.0);
    y = __double2float_rn(static_cast<double>(__fmul_rn(2.0f, canonical_f32(state))) - 1.0);
    r2 = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
  } while (r2 > 1.0f || r2 == 0.0f);
  const float mult = __fsqrt_rn(__fdiv_rn(__fmul_rn(-2.0f, glibc_logf(r2)), r2));
  saved = __fmul_rn(x, mult);
  return __fmul_rn(y, mult);
}

// k-th (0-based) set bit of m
__device__ __forceinline__ int nth_set_bit(unsigned int m, int k) {
  for (int i = 0; i < k; ++i) m &= m - 1;
  return __ffs(m) - 1;
}

// A fresh normal_distribution<float> over the row's SplitMix state
// (learners.cpp:89-92), the polar candidates drawn 32 at a time across the
// warp: lane l of round r tries pair r*32 + l (states s + 2(r*32 + l), +1);
// accepted pairs are taken in lane order.  Returns lane d's normal (d < A).
__device__ __forceinline__ float warp_row_normals(uint64_t* state, int A, int lane) {
  const uint64_t s0 = *state;
  const int need = (A + 1) / 2;
  int got = 0;
  float val = 0.0f;
  uint64_t consumed = 0;
  for (int round = 0;; ++round) {
    uint64_t s = s0 + 2 * (static_cast<uint64_t>(round) * 32 + lane);
    const float x = __double2float_rn(
        static_cast<double>(__fmul_rn(2.0f, canonical_f32(s))) - 1.0);
    const float y = __double2float_rn(
        static_cast<double>(__fmul_rn(2.0f, canonical_f32(s))) - 1.0);
    const float r2 = __fadd_rn(__fmul_rn(x, x), __fmul_rn(y, y));
    const bool ok = !(r2 > 1.0f || r2 == 0.0f);
    const unsigned int bal = __ballot_sync(0xffffffffu, ok);
    float vx = 0.0f, vy = 0.0f;
    if (ok) {
      const float mult = __fsqrt_rn(__fdiv_rn(__fmul_rn(-2.0f, glibc_logf(r2)), r2));
      vx = __fmul_rn(x, mult);
      vy = __fmul_rn(y, mult);
    }
    const int n = __popc(bal);
    const int p = lane / 2 - got;  // this lane's pair within this round
    const int owner = (lane < A && p >= 0 && p < n) ? nth_set_bit(bal, p) : 0;
    const float oy = __shfl_sync(0xffffffffu, vy, owner);
    const float ox = __shfl_sync(0xffffffffu, vx, owner);
    if (lane < A && p >= 0 && p < n) val = (lane & 1) ? ox : oy;
    if (got + n >= need) {
      consumed = static_cast<uint64_t>(round) * 32 + nth_set_bit(bal, need - got - 1) + 1;
      break;
    }
    got += n;
  }
  if (lane == 0) *state = s0 + 2 * consumed;
  return val;
}

// uniform() of vecenv.cpp:19-23 (53-bit path), evaluated in double.
__device__ __forceinline__ float env_uniform(uint64_t& state, float lo, float hi) {
  const double u = __dmul_rn(static_cast<double>(splitmix64(state++) >> 11), 0x1.0p-53);
  return __double2float_rn(
      __dadd_rn(static_cast<double>(lo), __dmul_rn(static_cast<double>(__fsub_rn(hi, lo)), u)));
}

}  // namespace pqlg::rng
