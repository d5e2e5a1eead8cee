// The running-normalizer state and the fixed-order finish of its update
// (RunningNormalizer::update + merge, normalizer.hpp:33-50, :73-83), shared by
// the standalone finish launch and the actor's fused policy-head launch.
#pragma once

#include <cstdint>

namespace pqlg::actor {

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

constexpr int kNormFinishWarps = 16;  // logical warps of the fixed summation order
inline int norm_finish_blocks(int D) { return (D + 31) / 32; }

struct NormFinishArgs {
  const double* shift;     // [D] the partials' shift
  int N, D, blocks;        // rows of the batch, columns, partial rows
  const double2* partial;  // [blocks][D] (sum (x - shift), sum (x - shift)^2)
  unsigned int* ticket;
  NormState s;
  int nblk;                // finish blocks (norm_finish_blocks(D))
};

// Finish block `bid` (columns 32 bid ..): partial row k of column c is added
// by logical warp k % 16 in ascending k, the 16 warp sums in order -- the same
// order for any physical warp count dividing 16.  The batch (mean, M2) is then
// merged into the running stats with Chan's formula (or, sharded, written to
// s.batch) and the fp32 apply constants refreshed; the last block advances the
// count.  red: [16][32] double2 of shared memory.  Every thread of the block
// must call it.
__device__ __forceinline__ void norm_finish_block(const NormFinishArgs& f, int bid, double2* red) {
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int c = bid * 32 + lane;
  const int D = f.D, N = f.N, blocks = f.blocks;
  const NormState& s = f.s;
  for (int lw = w; lw < kNormFinishWarps; lw += nw) {
    double a1 = 0.0, a2 = 0.0;
    if (c < D) {
      constexpr int kIn = 4;
      for (int k0 = lw; k0 < blocks; k0 += kNormFinishWarps * kIn) {
        double2 v[kIn];
#pragma unroll
        for (int t = 0; t < kIn; ++t) {
          const int k = k0 + kNormFinishWarps * t;
          v[t] = k < blocks ? __ldcg(f.partial + static_cast<int64_t>(k) * D + c) : make_double2(0.0, 0.0);
        }
#pragma unroll
        for (int t = 0; t < kIn; ++t) {
          a1 += v[t].x;
          a2 += v[t].y;
        }
      }
    }
    red[lw * 32 + lane] = make_double2(a1, a2);
  }
  __syncthreads();
  const int64_t n0i = s.batch ? 0 : *s.count;
  if (w == 0 && c < D) {
    const double nb = static_cast<double>(N);
    const double na = static_cast<double>(n0i);
    const int64_t cnt = n0i + N;
    double t1 = 0.0, t2 = 0.0;
#pragma unroll
    for (int k = 0; k < kNormFinishWarps; ++k) {
      t1 += red[k * 32 + lane].x;
      t2 += red[k * 32 + lane].y;
    }
    const double bmean = f.shift[c] + t1 / nb;
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
    __threadfence();
    // every block read the old count before its ticket: the last one advances it
    if (atomicAdd(f.ticket, 1u) == static_cast<unsigned>(f.nblk) - 1) {
      if (s.batch) {
        s.batch[2 * D] = static_cast<double>(N);
      } else {
        *s.count = n0i + N;
        *s.identity = n0i + N <= 1 ? 1 : 0;
      }
      *f.ticket = 0u;
    }
  }
}

}  // namespace pqlg::actor
