// Host side of the learners' SAC eps stream (sac_kernels.cuh).
#pragma once

#include <cmath>
#include <random>
#include <vector>

#include "common.h"
#include "mlp_host.h"
#include "sac_kernels.cuh"

namespace pqlg {

// B x A standard normals per update: one normal_distribution<float> over
// the Philox URBG keyed derive_seed(seed, sac, learner) (learners.cpp:137,
// :213), or -- mt19937-compat mode -- over the reference's own
// make_rng(seed, sac, learner) stream, drawn on the host and uploaded.
struct EpsStream {
  DevBuf<sac::EpsState> st;
  DevBuf<float> out;
  DevBuf<unsigned int> counts, ticket;
  DevBuf<int64_t> last_j;
  int64_t n = 0;
  int blocks = 0;
  std::mt19937_64 mt;
  std::vector<float> host;

  void init(uint64_t key, int64_t count) {
    n = count;
    const int64_t need = (n + 1) / 2;
    // candidates: need / (pi/4) + 8 sigma + slack (a shortfall is still
    // handled, sequentially, by the emit kernel's last block)
    const double cand = static_cast<double>(need) / 0.7853981633974483 +
                        8.0 * std::sqrt(static_cast<double>(need)) + 64.0;
    blocks = static_cast<int>((static_cast<int64_t>(cand) + sac::kEpsChunk - 1) / sac::kEpsChunk);
    if (blocks < 1) blocks = 1;
    st.alloc(1);
    const sac::EpsState s0{key, 0};
    copy_sync(st.p, &s0, sizeof(s0), cudaMemcpyHostToDevice);
    out.alloc(static_cast<size_t>(n));
    counts.alloc(blocks);
    ticket.alloc(1);
    last_j.alloc(1);
    const int64_t none = -1;
    copy_sync(last_j.p, &none, 8, cudaMemcpyHostToDevice);
    mt.seed(key);
    host.resize(static_cast<size_t>(n));
  }

  void enqueue(cudaStream_t s) const {
    sac::EpsArgs a{st.p, out.p, n, (n + 1) / 2, counts.p, ticket.p, last_j.p};
    launch(sac::eps_count_kernel, dim3(blocks), dim3(sac::kEpsThreads), 0, s, a);
    launch(sac::eps_emit_kernel, dim3(blocks), dim3(sac::kEpsThreads), 0, s, a);
  }

  // The draws depend on nothing but the stream's own counter: fork them onto
  // a side stream (a parallel branch of the captured update graph) so they
  // run beside the sample and the policy GEMMs; join() before the consumer.
  cudaStream_t side = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void fork(cudaStream_t main) {
    if (!side) {
      PQLG_CUDA(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
      PQLG_CUDA(cudaEventCreateWithFlags(&ev_fork, cudaEventDisableTiming));
      PQLG_CUDA(cudaEventCreateWithFlags(&ev_join, cudaEventDisableTiming));
    }
    PQLG_CUDA(cudaEventRecord(ev_fork, main));
    PQLG_CUDA(cudaStreamWaitEvent(side, ev_fork, 0));
    enqueue(side);
    PQLG_CUDA(cudaEventRecord(ev_join, side));
  }
  void join(cudaStream_t main) const {
    if (ev_join) PQLG_CUDA(cudaStreamWaitEvent(main, ev_join, 0));
  }
  ~EpsStream() {
    if (side) {
      cudaStreamSynchronize(side);
      cudaStreamDestroy(side);
      cudaEventDestroy(ev_fork);
      cudaEventDestroy(ev_join);
    }
  }

  // the reference's sequential stream (learners.cpp:171-173)
  void fill_mt(cudaStream_t s) {
    std::normal_distribution<float> gauss(0.0f, 1.0f);
    for (auto& x : host) x = gauss(mt);
    PQLG_CUDA(cudaMemcpyAsync(out.p, host.data(), n * 4, cudaMemcpyHostToDevice, s));
  }
};

// GaussianPolicy::sample's finish over a planned split-K head (2A columns).
inline mlp::Step gauss_finish_step(const mlp::HeadSplit& hs, sac::GaussArgs g, int M, int A) {
  g.part = hs.part.p;
  g.S = hs.splits;
  g.ld_part = hs.ld_part;
  g.M = M;
  g.A = A;
  const int rows_blocks = (M + sac::kFinishWarps - 1) / sac::kFinishWarps;
  const int blocks = rows_blocks < 4 * mlp::kSMs ? rows_blocks : 4 * mlp::kSMs;
  return [g, blocks](cudaStream_t st) {
    launch(sac::gauss_finish_kernel, dim3(blocks), dim3(32 * sac::kFinishWarps), 0, st, g);
  };
}

}  // namespace pqlg
