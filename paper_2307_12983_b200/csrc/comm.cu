// pqlg_comm: the NCCL communicator of the data-parallel learners (config 5,
// SURVEY 8(e)).  One rank per process/GPU; the unique id travels over the
// caller's host channel.
#include <cstring>
#include <memory>

#include "comm.h"

using namespace pqlg;

extern "C" {

int pqlg_comm_unique_id(uint8_t* id_out) {
  return guarded([&] {
    require(id_out != nullptr, "comm_unique_id: null output");
    static_assert(sizeof(ncclUniqueId) == PQLG_COMM_ID_BYTES, "ncclUniqueId size");
    ncclUniqueId id;
    PQLG_NCCL(ncclGetUniqueId(&id));
    std::memcpy(id_out, &id, sizeof(id));
  });
}

int pqlg_comm_init(int rank, int world, const uint8_t* id, pqlg_comm* out) {
  return guarded([&] {
    require(id && out, "comm_init: null argument");
    require(world >= 1 && rank >= 0 && rank < world, "comm_init: rank must be in [0, world)");
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof(uid));
    auto c = std::make_unique<pqlg_comm_s>();
    c->rank = rank;
    c->world = world;
    PQLG_NCCL(ncclCommInitRank(&c->nccl, world, uid, rank));
    *out = c.release();
  });
}

int pqlg_comm_destroy(pqlg_comm c) {
  return guarded([&] {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(c->nccl);
    delete c;
  });
}

int pqlg_comm_rank(pqlg_comm c, int* rank, int* world) {
  return guarded([&] {
    require(c != nullptr, "comm_rank: null comm");
    if (rank) *rank = c->rank;
    if (world) *world = c->world;
  });
}

int pqlg_comm_allreduce_f32(pqlg_comm c, float* buf, uint64_t n, void* stream) {
  return guarded([&] {
    require(c != nullptr, "comm_allreduce: null comm");
    allreduce_sum(c, buf, n, nullptr, 0, static_cast<cudaStream_t>(stream));
  });
}

}  // extern "C"
