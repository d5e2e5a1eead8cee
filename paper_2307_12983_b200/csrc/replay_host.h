// Host-side owners of the device replay objects (used by the C ABI in
// replay.cu and by the learner cores).
#pragma once

#include <cmath>
#include <memory>
#include <vector>

#include "common.h"
#include "replay.cuh"

namespace pqlg {

// fp32 normalization constants on device (normalizer.hpp:56-70).
// (mean_f, inv_f, identity) from device NormStats, normalizer.hpp:62-66.
void launch_norm_consts(const int64_t* count, const double* mean, const double* m2, int D,
                        float* mean_f, float* inv_f, int* ident, cudaStream_t st);

struct DeviceNorm {
  DevBuf<float> mean, inv;
  DevBuf<int> ident;  // device flag: kernels (and captured graphs) read it at run time
  int D = 0;
  // pinned staging [mean_f D | inv_f D | ident] so set() is asynchronous; the
  // event guards reuse while a previous copy is in flight
  float* stage = nullptr;
  cudaEvent_t staged = nullptr;
  DeviceNorm() = default;
  DeviceNorm(const DeviceNorm&) = delete;
  DeviceNorm& operator=(const DeviceNorm&) = delete;
  ~DeviceNorm() {
    if (staged) {
      cudaEventSynchronize(staged);
      cudaEventDestroy(staged);
    }
    if (stage) cudaFreeHost(stage);
  }
  void init(int dim) {
    D = dim;
    mean.alloc(dim);
    inv.alloc(dim);
    ident.alloc(1);
    PQLG_CUDA(cudaMallocHost(&stage, (2 * static_cast<size_t>(dim) + 1) * sizeof(float)));
    PQLG_CUDA(cudaEventCreateWithFlags(&staged, cudaEventDisableTiming));
    set_identity(nullptr);
    PQLG_CUDA(cudaEventSynchronize(staged));
  }
  void set_identity(cudaStream_t st) {
    PQLG_CUDA(cudaEventSynchronize(staged));
    reinterpret_cast<int*>(stage)[2 * D] = 1;
    PQLG_CUDA(cudaMemcpyAsync(ident.p, stage + 2 * D, sizeof(int), cudaMemcpyHostToDevice, st));
    PQLG_CUDA(cudaEventRecord(staged, st));
  }
  // NormStats -> (mean_f, inv_f) exactly as normalizer.hpp:62-66 (host double).
  void set(int64_t count, const double* m, const double* m2, cudaStream_t st) {
    if (count <= 1) {
      set_identity(st);
      return;
    }
    PQLG_CUDA(cudaEventSynchronize(staged));  // the previous staged copy has landed
    float* mf = stage;
    float* inv_f = stage + D;
    for (int j = 0; j < D; ++j) {
      mf[j] = static_cast<float>(m[j]);
      const double var = m2[j] / static_cast<double>(count);
      inv_f[j] = static_cast<float>(1.0 / std::sqrt(var + 1e-8));
    }
    reinterpret_cast<int*>(stage)[2 * D] = 0;
    PQLG_CUDA(cudaMemcpyAsync(mean.p, mf, D * sizeof(float), cudaMemcpyHostToDevice, st));
    PQLG_CUDA(cudaMemcpyAsync(inv.p, inv_f, D * sizeof(float), cudaMemcpyHostToDevice, st));
    PQLG_CUDA(cudaMemcpyAsync(ident.p, stage + 2 * D, sizeof(int), cudaMemcpyHostToDevice, st));
    PQLG_CUDA(cudaEventRecord(staged, st));
  }
  // The same from device-resident NormStats (count, mean, m2), computed on
  // device in fp64 (IEEE division and sqrt: identical to the host formula),
  // asynchronous on st.
  void set_device(const int64_t* count, const double* m, const double* m2, cudaStream_t st);
  replay::Norm view() const { return replay::Norm{mean.p, inv.p, ident.p}; }
};

struct DeviceReplay {
  int D, A;
  uint64_t capacity;
  int64_t ld_obs, ld_act;
  cudaStream_t stream;
  DevBuf<float> obs, act, boot, ret, eff;
  DevBuf<uint64_t> state;  // cursor, count

  DeviceReplay(uint64_t cap, int obs_dim, int act_dim, cudaStream_t st)
      : D(obs_dim), A(act_dim), capacity(cap), stream(st) {
    require(cap >= 1, "replay: capacity must be >= 1");
    require(obs_dim >= 1 && act_dim >= 1, "replay: dims must be >= 1");
    ld_obs = round_up(D, 4);
    ld_act = round_up(A, 4);
    obs.alloc(cap * ld_obs);
    act.alloc(cap * ld_act);
    boot.alloc(cap * ld_obs);
    ret.alloc(cap);
    eff.alloc(cap);
    state.alloc(2);
  }

  replay::Ring view() const {
    return replay::Ring{obs.p, act.p, boot.p, ret.p, eff.p, ld_obs, ld_act, D, A, capacity, state.p};
  }

  void read_state(uint64_t* cursor_count) const {
    PQLG_CUDA(cudaMemcpyAsync(cursor_count, state.p, 2 * sizeof(uint64_t), cudaMemcpyDeviceToHost,
                              stream));
    PQLG_CUDA(cudaStreamSynchronize(stream));
  }
  uint64_t size() const {
    uint64_t s[2];
    read_state(s);
    return s[1];
  }
};

struct DeviceStates {
  int D;
  uint64_t capacity;
  int64_t ld;
  cudaStream_t stream;
  DevBuf<float> obs;
  DevBuf<uint64_t> state;

  DeviceStates(uint64_t cap, int obs_dim, cudaStream_t st) : D(obs_dim), capacity(cap), stream(st) {
    require(cap >= 1, "state buffer: capacity must be >= 1");
    ld = round_up(D, 4);
    obs.alloc(cap * ld);
    state.alloc(2);
  }
  replay::StateRing view() const { return replay::StateRing{obs.p, ld, D, capacity, state.p}; }
  uint64_t size() const {
    uint64_t s[2];
    PQLG_CUDA(cudaMemcpyAsync(s, state.p, sizeof(s), cudaMemcpyDeviceToHost, stream));
    PQLG_CUDA(cudaStreamSynchronize(stream));
    return s[1];
  }
  void insert(const float* rows, int64_t ld_rows, uint64_t n, cudaStream_t st);
};

struct DeviceNStep {
  int N, D, A, n;
  float gamma;
  int64_t ld_obs, ld_act;
  DevBuf<float> wobs, wact, wrew;
  DevBuf<uint32_t> head, count, offs, block_sums;
  int n_blocks;

  DeviceNStep(int n_envs, int obs_dim, int act_dim, float g, int horizon)
      : N(n_envs), D(obs_dim), A(act_dim), n(horizon), gamma(g) {
    require(horizon >= 1 && horizon <= 32, "nstep: horizon must be in [1, 32]");
    require(n_envs >= 1, "nstep: n_envs must be >= 1");
    ld_obs = round_up(D, 4);
    ld_act = round_up(A, 4);
    wobs.alloc(static_cast<size_t>(N) * n * ld_obs);
    wact.alloc(static_cast<size_t>(N) * n * ld_act);
    wrew.alloc(static_cast<size_t>(N) * n);
    head.alloc(N);
    count.alloc(N);
    offs.alloc(N);
    n_blocks = (N + replay::kScanBlock - 1) / replay::kScanBlock;
    block_sums.alloc(n_blocks);
  }
  replay::Window window() const {
    return replay::Window{wobs.p, wact.p, wrew.p, head.p, count.p, ld_obs, ld_act, N, n, gamma};
  }
  // push_step + insert into `ring` (3 launches on `st`).
  void push(const replay::Slice& s, float reward_scale, DeviceReplay& ring, cudaStream_t st);
};

// Sampling into a gather destination; `ss` lives on device.
void launch_replay_sample(const DeviceReplay& r, const replay::Norm& norm, const replay::Gather& g,
                          replay::SamplerState* ss, const uint64_t* idx_dev, uint64_t B,
                          cudaStream_t st, bool early = false);
void launch_state_sample(const DeviceStates& r, const replay::Norm& norm, float* out,
                         int64_t ld_out, replay::SamplerState* ss, const uint64_t* idx_dev,
                         uint64_t B, cudaStream_t st, bool early = false);

}  // namespace pqlg

// ABI handle: owns its buffer, or views one owned by a learner core.
struct pqlg_replay_s {
  pqlg::DeviceReplay* r = nullptr;
  std::unique_ptr<pqlg::DeviceReplay> owned;
  pqlg::DeviceNorm norm;
  pqlg::DevBuf<pqlg::replay::SamplerState> ss;
  pqlg::DevBuf<uint64_t> idx;
};
