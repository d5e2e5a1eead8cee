// C ABI for the device replay objects: ReplayBuffer, NStepAssembler (fused
// with insert) and StateBuffer.  See include/pqlg.h for the reference
// interfaces each entry point replaces.
#include <memory>
#include <vector>

#include "replay_host.h"

namespace pqlg {

using replay::kWarpsPerBlock;

void DeviceNStep::push(const replay::Slice& s, float reward_scale, DeviceReplay& ring,
                       cudaStream_t st) {
  require(ring.D == D && ring.A == A, "nstep: replay schema mismatch");
  launch(replay::nstep_count_kernel, dim3(n_blocks), dim3(replay::kScanBlock), 0, st, window(), s, offs.p,
                                                                      block_sums.p);
  const int warps = N;
  launch(replay::nstep_emit_kernel, dim3((warps + kWarpsPerBlock - 1) / kWarpsPerBlock), dim3(32 * kWarpsPerBlock), 0, st, window(), s, reward_scale, ring.view(), offs.p,
                                       block_sums.p, n_blocks);
  launch(replay::ring_advance_kernel, dim3(1), dim3(32), 0, st, ring.state.p, ring.capacity, block_sums.p,
                                                n_blocks, 0);
}

void DeviceStates::insert(const float* rows, int64_t ld_rows, uint64_t n, cudaStream_t st) {
  if (n == 0) return;
  const uint64_t blocks = (n + kWarpsPerBlock - 1) / kWarpsPerBlock;
  launch(replay::state_insert_kernel, dim3(static_cast<unsigned>(blocks)), dim3(32 * kWarpsPerBlock), 0, st, view(), rows, ld_rows, n);
  launch(replay::ring_advance_kernel, dim3(1), dim3(32), 0, st, state.p, capacity, nullptr, 0, n);
}

void launch_replay_sample(const DeviceReplay& r, const replay::Norm& norm, const replay::Gather& g,
                          replay::SamplerState* ss, const uint64_t* idx_dev, uint64_t B,
                          cudaStream_t st, bool early) {
  const uint64_t blocks = (B + replay::kSampleRows - 1) / replay::kSampleRows;
  launch(replay::replay_sample_kernel, dim3(static_cast<unsigned>(blocks)), dim3(32 * kWarpsPerBlock), 0, st, r.view(), norm, g, ss, idx_dev, B, early ? 1 : 0);
}

void launch_state_sample(const DeviceStates& r, const replay::Norm& norm, float* out,
                         int64_t ld_out, replay::SamplerState* ss, const uint64_t* idx_dev,
                         uint64_t B, cudaStream_t st, bool early) {
  const uint64_t blocks = (B + replay::kSampleRows - 1) / replay::kSampleRows;
  launch(replay::state_sample_kernel, dim3(static_cast<unsigned>(blocks)), dim3(32 * kWarpsPerBlock), 0, st, r.view(), norm, out, ld_out, ss, idx_dev, B, early ? 1 : 0);
}

namespace {
__global__ void norm_consts_kernel(const int64_t* count, const double* mean, const double* m2,
                                   int D, float* mean_f, float* inv_f, int* ident) {
  pdl::entry();
  const int64_t c = *count;
  if (blockIdx.x == 0 && threadIdx.x == 0) *ident = c <= 1 ? 1 : 0;
  if (c <= 1) return;
  for (int j = blockIdx.x * blockDim.x + threadIdx.x; j < D; j += gridDim.x * blockDim.x) {
    mean_f[j] = static_cast<float>(mean[j]);
    const double var = __ddiv_rn(m2[j], static_cast<double>(c));
    inv_f[j] = static_cast<float>(__ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(var, 1e-8))));
  }
}
}  // namespace

void launch_norm_consts(const int64_t* count, const double* mean, const double* m2, int D,
                        float* mean_f, float* inv_f, int* ident, cudaStream_t st) {
  launch(norm_consts_kernel, dim3((D + 255) / 256), dim3(256), 0, st, count, mean, m2, D, mean_f,
         inv_f, ident);
}

void DeviceNorm::set_device(const int64_t* count, const double* m, const double* m2,
                            cudaStream_t st) {
  launch_norm_consts(count, m, m2, D, mean.p, inv.p, ident.p, st);
}

}  // namespace pqlg

// ------------------------------------------------------------------ C ABI
struct pqlg_nstep_s {
  std::unique_ptr<pqlg::DeviceNStep> a;
  cudaStream_t stream;
};
struct pqlg_states_s {
  std::unique_ptr<pqlg::DeviceStates> s;
  pqlg::DeviceNorm norm;
  pqlg::DevBuf<pqlg::replay::SamplerState> ss;
  pqlg::DevBuf<uint64_t> idx;
};

using namespace pqlg;

namespace {
int64_t ld_or(int64_t ld, int64_t dense) { return ld > 0 ? ld : dense; }

// Uploads the generator for one sample call; returns the device index array
// (INDICES mode) or null (PHILOX mode, state in `ss`).
const uint64_t* prepare_rng(const pqlg_rng* rng, uint64_t B, DevBuf<replay::SamplerState>& ss,
                            DevBuf<uint64_t>& idx, cudaStream_t st) {
  require(rng != nullptr, "sample: rng is required");
  if (ss.n == 0) ss.alloc(1);
  if (rng->mode == PQLG_RNG_INDICES) {
    require(rng->host_indices != nullptr, "sample: host_indices required");
    if (idx.n < B) idx.alloc(B);
    PQLG_CUDA(cudaMemcpyAsync(idx.p, rng->host_indices, B * sizeof(uint64_t),
                              cudaMemcpyHostToDevice, st));
    PQLG_CUDA(cudaStreamSynchronize(st));
    return idx.p;
  }
  require(rng->mode == PQLG_RNG_PHILOX, "sample: unknown rng mode");
  replay::SamplerState h{rng->key, rng->counter, 0, 0};
  PQLG_CUDA(cudaMemcpyAsync(ss.p, &h, sizeof(h), cudaMemcpyHostToDevice, st));
  PQLG_CUDA(cudaStreamSynchronize(st));
  return nullptr;
}

void finish_rng(pqlg_rng* rng, DevBuf<replay::SamplerState>& ss, cudaStream_t st) {
  if (rng->mode != PQLG_RNG_PHILOX) {
    PQLG_CUDA(cudaStreamSynchronize(st));
    return;
  }
  replay::SamplerState h{};
  PQLG_CUDA(cudaMemcpyAsync(&h, ss.p, sizeof(h), cudaMemcpyDeviceToHost, st));
  PQLG_CUDA(cudaStreamSynchronize(st));
  rng->counter = h.counter;
}
}  // namespace

extern "C" {

int pqlg_replay_create(uint64_t capacity, int obs_dim, int act_dim, void* stream,
                       pqlg_replay* out) {
  return guarded([&] {
    require(out != nullptr, "replay_create: out is null");
    auto h = std::make_unique<pqlg_replay_s>();
    h->owned = std::make_unique<DeviceReplay>(capacity, obs_dim, act_dim,
                                              static_cast<cudaStream_t>(stream));
    h->r = h->owned.get();
    h->norm.init(obs_dim);
    *out = h.release();
  });
}

int pqlg_replay_destroy(pqlg_replay h) {
  return guarded([&] { delete h; });
}

int pqlg_replay_size(pqlg_replay h, uint64_t* out) {
  return guarded([&] { *out = h->r->size(); });
}

int pqlg_replay_cursor(pqlg_replay h, uint64_t* out) {
  return guarded([&] {
    uint64_t s[2];
    h->r->read_state(s);
    *out = s[0];
  });
}

int pqlg_replay_insert(pqlg_replay h, const pqlg_nstep_batch* b, uint64_t n) {
  return guarded([&] {
    if (n == 0) return;  // replay_buffer.hpp:34
    auto& r = *h->r;
    const int64_t ldo = ld_or(b->ld_obs, r.D), lda = ld_or(b->ld_act, r.A);
    const uint64_t blocks = (n + kWarpsPerBlock - 1) / kWarpsPerBlock;
    launch(replay::ring_insert_kernel, dim3(static_cast<unsigned>(blocks)), dim3(32 * kWarpsPerBlock), 0, r.stream, r.view(), b->obs, b->act, b->boot_obs, b->ret,
                                             b->eff_disc, ldo, lda, n);
    launch(replay::ring_advance_kernel, dim3(1), dim3(32), 0, r.stream, r.state.p, r.capacity, nullptr, 0, n);
  });
}

int pqlg_replay_sample(pqlg_replay h, uint64_t batch, pqlg_rng* rng, uint64_t min_live,
                       const pqlg_norm_stats* norm, pqlg_nstep_batch* o) {
  const int rc = guarded([&] {
    auto& r = *h->r;
    const uint64_t count = r.size();
    if (count < min_live || count == 0) throw Error(PQLG_NOT_READY, "replay: not enough records");
    if (norm) h->norm.set(norm->count, norm->mean, norm->m2, r.stream);
    else h->norm.set_identity(r.stream);
    const uint64_t* idx = prepare_rng(rng, batch, h->ss, h->idx, r.stream);
    replay::Gather g{o->obs, ld_or(o->ld_obs, r.D), o->act, ld_or(o->ld_act, r.A),
                     o->boot_obs, ld_or(o->ld_obs, r.D), o->ret, o->eff_disc};
    launch_replay_sample(r, h->norm.view(), g, h->ss.p, idx, batch, r.stream);
    finish_rng(rng, h->ss, r.stream);
  });
  return rc;
}

int pqlg_k_sample_indices(uint64_t key, uint64_t* counter, uint64_t count, uint64_t batch,
                          uint64_t* out_host, uint32_t* rejected) {
  return guarded([&] {
    require(counter && out_host && count >= 1 && batch >= 1, "sample_indices: bad arguments");
    cudaStream_t st;
    PQLG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    DevBuf<replay::SamplerState> ss(1);
    DevBuf<uint64_t> out(batch);
    const replay::SamplerState s0{key, *counter, 0, 0};
    PQLG_CUDA(cudaMemcpyAsync(ss.p, &s0, sizeof(s0), cudaMemcpyHostToDevice, st));
    const uint64_t blocks = (batch + replay::kSampleRows - 1) / replay::kSampleRows;
    // the reject flag is cleared by the finish: read it through a probe copy
    // taken before (flag state after the draws is what the finish saw)
    launch(replay::sample_indices_kernel, dim3(static_cast<unsigned>(blocks)),
           dim3(32 * kWarpsPerBlock), 0, st, ss.p, count, batch, out.p);
    replay::SamplerState s1{};
    PQLG_CUDA(cudaMemcpyAsync(&s1, ss.p, sizeof(s1), cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaMemcpyAsync(out_host, out.p, batch * 8, cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaStreamSynchronize(st));
    PQLG_CUDA(cudaStreamDestroy(st));
    if (rejected) *rejected = (s1.counter - *counter) > batch ? 1u : 0u;
    *counter = s1.counter;
  });
}

int pqlg_replay_fill_synthetic(pqlg_replay h, uint64_t n, uint64_t seed, float disc,
                               uint32_t terminal_every) {
  return guarded([&] {
    if (n == 0) return;
    auto& r = *h->r;
    const uint64_t blocks = (n + kWarpsPerBlock - 1) / kWarpsPerBlock;
    launch(replay::ring_fill_kernel, dim3(static_cast<unsigned>(blocks)), dim3(32 * kWarpsPerBlock), 0, r.stream, r.view(), n, seed, disc, terminal_every);
    launch(replay::ring_advance_kernel, dim3(1), dim3(32), 0, r.stream, r.state.p, r.capacity, nullptr, 0, n);
  });
}

int pqlg_replay_read_rows(pqlg_replay h, uint64_t i0, uint64_t n, float* obs, float* act,
                          float* boot, float* ret, float* eff) {
  return guarded([&] {
    auto& r = *h->r;
    require(i0 + n <= r.capacity, "read_rows: out of range");
    auto st = r.stream;
    if (obs)
      PQLG_CUDA(cudaMemcpy2DAsync(obs, r.D * sizeof(float), r.obs.p + i0 * r.ld_obs,
                                  r.ld_obs * sizeof(float), r.D * sizeof(float), n,
                                  cudaMemcpyDeviceToHost, st));
    if (act)
      PQLG_CUDA(cudaMemcpy2DAsync(act, r.A * sizeof(float), r.act.p + i0 * r.ld_act,
                                  r.ld_act * sizeof(float), r.A * sizeof(float), n,
                                  cudaMemcpyDeviceToHost, st));
    if (boot)
      PQLG_CUDA(cudaMemcpy2DAsync(boot, r.D * sizeof(float), r.boot.p + i0 * r.ld_obs,
                                  r.ld_obs * sizeof(float), r.D * sizeof(float), n,
                                  cudaMemcpyDeviceToHost, st));
    if (ret)
      PQLG_CUDA(cudaMemcpyAsync(ret, r.ret.p + i0, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    if (eff)
      PQLG_CUDA(cudaMemcpyAsync(eff, r.eff.p + i0, n * sizeof(float), cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaStreamSynchronize(st));
  });
}

int pqlg_nstep_create(int n_envs, int obs_dim, int act_dim, float gamma, int horizon, void* stream,
                      pqlg_nstep* out) {
  return guarded([&] {
    auto h = std::make_unique<pqlg_nstep_s>();
    h->a = std::make_unique<DeviceNStep>(n_envs, obs_dim, act_dim, gamma, horizon);
    h->stream = static_cast<cudaStream_t>(stream);
    *out = h.release();
  });
}

int pqlg_nstep_destroy(pqlg_nstep h) {
  return guarded([&] { delete h; });
}

int pqlg_nstep_push_step(pqlg_nstep h, const pqlg_step_slice* s, float reward_scale,
                         pqlg_replay dst) {
  return guarded([&] {
    auto& a = *h->a;
    replay::Slice sl{s->obs, s->act, s->boot_obs, s->rew, s->term, s->trunc,
                     ld_or(s->ld_obs, a.D), ld_or(s->ld_act, a.A)};
    a.push(sl, reward_scale, *dst->r, h->stream);
  });
}

int pqlg_states_create(uint64_t capacity, int obs_dim, void* stream, pqlg_states* out) {
  return guarded([&] {
    auto h = std::make_unique<pqlg_states_s>();
    h->s = std::make_unique<DeviceStates>(capacity, obs_dim, static_cast<cudaStream_t>(stream));
    h->norm.init(obs_dim);
    *out = h.release();
  });
}

int pqlg_states_destroy(pqlg_states h) {
  return guarded([&] { delete h; });
}

int pqlg_states_size(pqlg_states h, uint64_t* out) {
  return guarded([&] { *out = h->s->size(); });
}

int pqlg_states_insert(pqlg_states h, const float* rows, int64_t ld, uint64_t n) {
  return guarded([&] {
    auto& s = *h->s;
    s.insert(rows, ld_or(ld, s.D), n, s.stream);
  });
}

int pqlg_states_sample(pqlg_states h, uint64_t batch, pqlg_rng* rng, uint64_t min_live,
                       const pqlg_norm_stats* norm, float* out, int64_t ld_out) {
  return guarded([&] {
    auto& s = *h->s;
    const uint64_t count = s.size();
    if (count < min_live || count == 0) throw Error(PQLG_NOT_READY, "states: not enough rows");
    if (norm) h->norm.set(norm->count, norm->mean, norm->m2, s.stream);
    else h->norm.set_identity(s.stream);
    const uint64_t* idx = prepare_rng(rng, batch, h->ss, h->idx, s.stream);
    launch_state_sample(s, h->norm.view(), out, ld_or(ld_out, s.D), h->ss.p, idx, batch,
                        s.stream);
    finish_rng(rng, h->ss, s.stream);
  });
}

}  // extern "C"
