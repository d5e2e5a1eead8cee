// ActorCore (learners.hpp:52-73, learners.cpp:62-116) on one B200: policy
// inference with the mixed-noise head, the running normalizer and the
// synthetic EnvBatch (actor.cu).
#pragma once

#include <memory>
#include <vector>

#include "mlp_host.h"
#include "net.h"

struct pqlg_comm_s;

namespace pqlg {

struct DeviceEnv;

class Actor {
 public:
  // comm (nullable): a sharded actor whose running normalizer is merged over
  // all shards every step (all-gather of the batch statistics)
  Actor(const pqlg_config& cfg, const pqlg_task_dims& dims, cudaStream_t st,
        pqlg_comm_s* comm = nullptr);
  ~Actor();
  void adopt_policy(const float* flat, int64_t version, bool device);
  void rollout_step(pqlg_step_slice* out);
  void rollout_n(int n);
  void norm(int64_t* count, double* mean, double* m2);
  void read_state(int what, void* out);
  // The last rollout_step's StepSlice, dense rows into host buffers (any may
  // be null); synchronizes.
  void read_last_slice(float* obs, float* act, float* boot, float* rew, uint8_t* term,
                       uint8_t* trunc);
  int64_t policy_version() const { return version_; }
  cudaStream_t stream() const { return stream_; }
  // recorded on the actor's stream after every rollout_step (null before the first)
  cudaEvent_t step_event() const { return step_done_; }
  int kernels_per_step();
  // Per-kernel device times of the step graph: one replay runs kSets
  // consecutive steps (every output buffer set once), so the actor's state
  // advances as after kSets rollout steps.
  std::string time_steps(int reps);
  int n_envs() const { return N_; }
  int obs_dim() const { return D_; }
  int64_t param_count() const { return pnet_.params; }
  int64_t snapshot_len() const { return pnet_.params + (sac_ ? 1 : 0); }
  // device views for the pipeline (run_parallel): the running normalizer
  // (owned by the actor, SPEC "Normalizer statistics are owned by the Actor")
  const float* policy_dev() const { return pol_.p; }
  const NetShape& policy_shape() const { return pnet_; }
  // restore the running normalizer (checkpoint load) and re-normalize the
  // current observations for the next policy input
  void set_norm(int64_t count, const double* mean, const double* m2);
  const int64_t* count_dev() const { return count_.p; }
  const double* mean_dev() const { return mean_.p; }
  const double* m2_dev() const { return m2_.p; }

 private:
  void build();
  void enqueue(int cur);

  pqlg_config cfg_;
  pqlg_task_dims dims_;
  cudaStream_t stream_;
  cudaStream_t owned_stream_ = nullptr;
  int N_, D_, A_, Ap_, H_, nh_;
  bool sac_ = false;            // pql_sac: Gaussian policy, no schedule noise
  pqlg_comm_s* comm_ = nullptr; // sharded: normalizer merged across shards
  cudaEvent_t step_done_ = nullptr;
  DevBuf<double> nbatch_, ngather_;
  mlp::HeadSplit head_split_;   // pql_sac: split-K [mean | log_std] head
  int64_t Dp_;
  NetShape pnet_;
  int64_t version_ = 0;
  int cur_ = 0;
  bool stepped_ = false;

  std::unique_ptr<DeviceEnv> env_;
  // Step outputs rotate over kSets buffer sets, so a slice handed out by
  // rollout_step stays valid for two more steps (its consumers -- the
  // learners' ingest -- can overlap the next step on their own streams).
  static constexpr int kSets = 3;
  DevBuf<float> obs_[kSets], boot_[kSets], rew_[kSets], act_[kSets], Xn_;
  DevBuf<uint8_t> term_[kSets], trunc_[kSets];
  DevBuf<float> pol_;
  DevBuf<float> wpack_;  // policy head W in the head kernel's fragment order
  void pack_head();
  void ensure_graphs();  // the per-buffer-set step graphs (rollout_step / rollout_n)
  bool fused_finish_ = false;  // normalizer finish inside the head launch
  actor::NormState norm_state() const;
  std::vector<DevBuf<float>> pact_;
  DevBuf<uint64_t> noise_rng_;
  DevBuf<float> sigma_;
  DevBuf<int64_t> count_;
  // npart_/nshift_: running-normalizer partial sums of the current
  // observations and their shift (written by the previous env step)
  DevBuf<double> mean_, m2_, npart_, nshift_;
  DevBuf<unsigned int> nticket_;
  DevBuf<float> mean_f_, inv_f_;
  DevBuf<int> identity_;
  DevBuf<uint32_t> status_;
  std::vector<mlp::Step> policy_steps_;   // hidden layers
  mlp::Step head_steps_[kSets];           // policy head + noise into act_[set]
  cudaGraphExec_t graph_[kSets] = {nullptr, nullptr, nullptr};
  int kps_ = 0;
};

// evaluate_policy (learners.cpp:280-325) on the synthetic task (actor.cu).
// Evaluator owns the device context (env, policy, buffers, stream) for one
// (config, episodes, eval_seed), allocated once: the metrics loops keep one
// so an evaluation neither allocates nor frees device memory (cudaFree
// synchronises the device, stalling the pipeline's streams).
class Evaluator {
 public:
  Evaluator(const pqlg_config& cfg, const pqlg_task_dims& dims, int episodes, uint64_t eval_seed);
  ~Evaluator();
  Evaluator(const Evaluator&) = delete;
  Evaluator& operator=(const Evaluator&) = delete;
  void run(const float* policy, int64_t count, const double* mean, const double* m2,
           double* returns, double* mean_out, double* stderr_out);

 private:
  struct Impl;
  std::unique_ptr<Impl> p_;
};
// One-shot: a fresh Evaluator.
void evaluate_policy(const pqlg_config& cfg, const pqlg_task_dims& dims, const float* policy,
                     int64_t count, const double* mean, const double* m2, int episodes,
                     uint64_t eval_seed, double* returns, double* mean_out, double* stderr_out);

}  // namespace pqlg
