// NCCL communicator behind pqlg_comm (data-parallel learners).
#pragma once

#include <nccl.h>

#include <string>

#include "common.h"

struct pqlg_comm_s {
  ncclComm_t nccl = nullptr;
  int rank = 0;
  int world = 1;
};

namespace pqlg {

[[noreturn]] inline void throw_nccl(ncclResult_t r, const char* what) {
  throw Error(PQLG_ENCCL, std::string("NCCL error ") + ncclGetErrorString(r) + ": " + what);
}

#define PQLG_NCCL(expr)                                        \
  do {                                                         \
    ncclResult_t _r = (expr);                                  \
    if (_r != ncclSuccess) ::pqlg::throw_nccl(_r, #expr);      \
  } while (0)

// Every kernel of the library lets its successor launch early (PDL,
// pdl.cuh), which is safe among our kernels because each one waits before
// touching memory.  An NCCL kernel launched with programmatic serialization
// would not wait for ours, so each NCCL call is preceded by this empty kernel,
// launched without the PDL attribute: it starts only when everything before
// it has completed, and it never triggers early.
static __global__ void nccl_fence_kernel() {}
inline void nccl_fence(cudaStream_t st) { nccl_fence_kernel<<<1, 32, 0, st>>>(); }

// One grouped in-place sum all-reduce of up to two float buffers (gradients
// and the loss scalar travel in the same NCCL launch).
inline void allreduce_sum(pqlg_comm_s* c, float* a, size_t na, float* b, size_t nb,
                          cudaStream_t st) {
  nccl_fence(st);
  PQLG_NCCL(ncclGroupStart());
  PQLG_NCCL(ncclAllReduce(a, a, na, ncclFloat32, ncclSum, c->nccl, st));
  if (b && nb) PQLG_NCCL(ncclAllReduce(b, b, nb, ncclFloat32, ncclSum, c->nccl, st));
  PQLG_NCCL(ncclGroupEnd());
}

// All-gather of fp64 records (the sharded actor's batch statistics).
inline void allgather_f64(pqlg_comm_s* c, const double* send, double* recv, size_t n,
                          cudaStream_t st) {
  nccl_fence(st);
  PQLG_NCCL(ncclAllGather(send, recv, n, ncclFloat64, c->nccl, st));
}

}  // namespace pqlg
