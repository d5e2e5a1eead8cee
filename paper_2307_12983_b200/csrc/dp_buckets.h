// Data-parallel gradient buckets: in a data-parallel learner
// every layer's gradient is reduced from its split-K partials (fixed order,
// the same finalize arithmetic as the single-GPU path) and summed over the
// ranks by ncclAllReduce as soon as that layer's backward has produced it --
// on a communication branch of the update graph (a side stream forked from
// the learner's stream with an event per bucket), so the transfer of layer
// l overlaps the dgrad / wgrad GEMMs of the layers below it.  The learner
// joins the branch before the full-gradient norm / clip pass.  World 1 gives
// the single-GPU update bit for bit (the reduction order is unchanged).
#pragma once

#include <cstdint>
#include <utility>
#include <vector>

#include "comm.h"
#include "mlp_host.h"
#include "optim.cuh"

namespace pqlg {

class DpBuckets {
 public:
  DpBuckets(pqlg_comm_s* comm, float* grads, int groups, int64_t gstride)
      : comm_(comm), grads_(grads), groups_(groups), gstride_(gstride) {}
  DpBuckets(const DpBuckets&) = delete;
  DpBuckets& operator=(const DpBuckets&) = delete;
  ~DpBuckets() {
    if (side_) {
      cudaStreamSynchronize(side_);
      cudaStreamDestroy(side_);
      cudaEventDestroy(ev_fork_);
      cudaEventDestroy(ev_join_);
    }
  }

  // One bucket: `segs` (finalize segments, reduction only) fill the flat
  // range [lo, hi) of every group, which is then all-reduced; `extra`
  // (nullable, n_extra floats: the loss) rides in the same NCCL group.
  mlp::Step bucket(std::vector<optim::Segment> segs, int64_t lo, int64_t hi, float* extra = nullptr,
                   size_t n_extra = 0) {
    require(!segs.empty() && segs.size() <= static_cast<size_t>(optim::kMaxSegments),
            "dp bucket: 1..kMaxSegments segments");
    optim::FinalizeArgs f{};
    for (size_t i = 0; i < segs.size(); ++i) f.seg[i] = segs[i];
    f.n_seg = static_cast<int>(segs.size());
    f.gstride = gstride_;
    f.grads = grads_;
    f.skip_norm = 1;
    const int fb = optim::plan_finalize(f);
    const int groups = groups_;
    const int64_t gs = gstride_;
    float* g = grads_;
    pqlg_comm_s* c = comm_;
    return [this, f, fb, groups, gs, g, c, lo, hi, extra, n_extra](cudaStream_t st) {
      cudaStream_t s = fork(st);
      launch(optim::finalize_kernel, dim3(dim3(fb, groups)), dim3(optim::kFinalizeThreads), 0, s,
             f);
      nccl_fence(s);
      PQLG_NCCL(ncclGroupStart());
      for (int k = 0; k < groups; ++k) {
        float* p = g + k * gs + lo;
        PQLG_NCCL(ncclAllReduce(p, p, static_cast<size_t>(hi - lo), ncclFloat32, ncclSum,
                                c->nccl, s));
      }
      if (extra && n_extra)
        PQLG_NCCL(ncclAllReduce(extra, extra, n_extra, ncclFloat32, ncclSum, c->nccl, s));
      PQLG_NCCL(ncclGroupEnd());
    };
  }

  // The learner's stream waits for every bucket issued so far.
  mlp::Step join() {
    return [this](cudaStream_t st) {
      if (!side_) return;
      PQLG_CUDA(cudaEventRecord(ev_join_, side_));
      PQLG_CUDA(cudaStreamWaitEvent(st, ev_join_, 0));
    };
  }

 private:
  cudaStream_t fork(cudaStream_t main) {
    if (!side_) {
      PQLG_CUDA(cudaStreamCreateWithFlags(&side_, cudaStreamNonBlocking));
      PQLG_CUDA(cudaEventCreateWithFlags(&ev_fork_, cudaEventDisableTiming));
      PQLG_CUDA(cudaEventCreateWithFlags(&ev_join_, cudaEventDisableTiming));
    }
    PQLG_CUDA(cudaEventRecord(ev_fork_, main));
    PQLG_CUDA(cudaStreamWaitEvent(side_, ev_fork_, 0));
    return side_;
  }

  pqlg_comm_s* comm_;
  float* grads_;
  int groups_;
  int64_t gstride_;
  cudaStream_t side_ = nullptr;
  cudaEvent_t ev_fork_ = nullptr, ev_join_ = nullptr;
};

}  // namespace pqlg
