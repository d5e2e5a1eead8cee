// The three runtime cores (learners.hpp:52-139) as device-resident objects.
#pragma once

#include <array>
#include <memory>
#include <random>
#include <vector>

#include "mlp_host.h"
#include "net.h"
#include "replay_host.h"
#include "sac_host.h"

struct pqlg_comm_s;

namespace pqlg {

class DpBuckets;  // dp_buckets.h

// CriticLearnerCore (learners.hpp:77-106).
class VLearner {
 public:
  // comm (nullable): data-parallel mode, one NCCL all-reduce per update
  VLearner(const pqlg_config& cfg, const pqlg_task_dims& dims, uint64_t init_seed,
           cudaStream_t st, pqlg_comm_s* comm = nullptr);
  ~VLearner();

  void adopt_policy(const float* flat_host, int64_t version);
  // pql_sac: the snapshot's log_alpha travels with the net (messages.hpp:18-19)
  void adopt_policy_sac(const float* flat_host, float log_alpha, int64_t version);
  float log_alpha();
  void adopt_norm(int64_t count, const double* mean, const double* m2);
  // asynchronous device-pointer variants (the run_parallel pipeline); the
  // device snapshot is [net | log_alpha] (snapshot_len floats)
  void adopt_policy_device(const float* flat_dev, int64_t version);
  int64_t snapshot_len() const { return pnet_.params + (sac_ ? 1 : 0); }
  void adopt_norm_device(const int64_t* count, const double* mean, const double* m2) {
    norm_.set_device(count, mean, m2, stream_);
  }
  const float* critic_dev(int k) const { return q_.p + k * Ps_; }
  const NetShape& policy_shape() const { return pnet_; }
  const NetShape& critic_shape() const { return qnet_; }
  int64_t critic_params() const { return qnet_.params; }
  int64_t policy_params() const { return pnet_.params; }
  int64_t lagged_version() const { return lagged_version_; }
  // NormStats last adopted from the host (checkpointing)
  int64_t norm_count_ = 0;
  std::vector<double> norm_mean_, norm_m2_;
  void ingest(const replay::Slice& s);
  void ingest_host(const pqlg_step_slice& host);  // copy-in path for a host StepSlice
  bool ready(int64_t c_a);
  float update();
  void update_n(int n);
  float last_loss();
  void get_params(int which, float* out);
  int64_t param_count(int which) const;
  void set_params(int which, const float* flat_host);
  void debug_read(int what, float* out);
  void set_mt_mode(bool on) { mt_mode_ = on; }
  int kernels_per_update();
  // Per-kernel device times of the update graph (time_in_graph, common.h).
  std::string time_update(int reps);

  DeviceReplay* replay() { return replay_.get(); }
  int obs_dim() const { return D_; }
  int act_dim() const { return A_; }
  cudaStream_t stream() const { return stream_; }
  // Synchronizes; PQLG_ENONFINITE (and clears the sticky status word) if an
  // update since the last check was non-finite.
  int check_status();

 private:
  void build_update();
  void enqueue();
  void prepare_indices();

  pqlg_config cfg_;
  pqlg_task_dims dims_;
  cudaStream_t stream_;
  cudaStream_t owned_stream_ = nullptr;
  pqlg_comm_s* comm_ = nullptr;  // data-parallel communicator (nullable)
  int rank_ = 0, world_ = 1;
  int D_, A_, H_, nh_, B_, Kp_;
  bool dist_ = false;  // PQL-D: categorical (C51) critics with L_ atoms
  bool sac_ = false;   // pql_sac: Gaussian lagged policy, entropy term in the target
  int L_ = 1, Lp_ = 1;
  float reward_scale_, gamma_;
  EpsStream eps_;      // pql_sac eps draws
  std::unique_ptr<DpBuckets> dp_;  // data-parallel gradient buckets (comm_ only)
  DevBuf<float> logp_; // log pi(a'|s+) [B]
  NetShape qnet_, pnet_;
  int64_t Ps_ = 0;  // group stride of the twin-critic parameter blocks
  int64_t lagged_version_ = 0;

  DevBuf<float> q_, qt_, m_, v_, grads_, lagged_;
  DevBuf<float> wpack_;  // lagged policy head W in the head kernel's fragment order
  int wpack_n_ = 0;      // its output columns (act_dim, pql_sac 2 act_dim)
  void lagged_changed();
  mlp::HeadSplit head_split_;  // split-K lagged-policy head
  std::unique_ptr<DeviceReplay> replay_;
  std::unique_ptr<DeviceNStep> nstep_;
  DevBuf<float> in_f_;     // host-ingest staging: obs | act | boot | rew
  DevBuf<uint8_t> in_u8_;  // term | trunc
  DeviceNorm norm_;
  DevBuf<replay::SamplerState> sampler_;
  bool mt_mode_ = false;
  std::mt19937_64 mt_;
  DevBuf<uint64_t> idx_;
  std::vector<uint64_t> idx_host_;

  DevBuf<int64_t> step_;
  DevBuf<float2> bc_;
  DevBuf<uint32_t> status_;
  DevBuf<float> loss_;
  PinnedBuf<uint32_t> hbuf_;  // update(): loss bits + status

  // workspaces
  DevBuf<float> Xon_, Xtg_, ret_, eff_, y_;
  std::vector<DevBuf<float>> pact_;
  std::array<std::vector<DevBuf<float>>, 2> tact_, oact_, G_;
  std::array<std::vector<DevBuf<uint32_t>>, 2> omask_;  // ReLU bitmasks of the online critics
  DevBuf<float> part_t_, part_o_, up_;
  DevBuf<double> block_loss_;
  DevBuf<unsigned int> loss_counter_;
  std::vector<DevBuf<float>> wpart_, colsum_;
  std::vector<int> wsplits_;
  DevBuf<float> head_dw_, head_db_, head_cs_;
  int fin_blocks_ = 0;
  DevBuf<double> block_sq_;
  DevBuf<unsigned int> fin_counter_;
  DevBuf<float> scale_;
  // C51 (PQL-D) head state: atoms, target/online probabilities, expected
  // values, upstream [2][B x Lp], head-bias partials, head weight partials,
  // padded head mirrors (q1, q2, q1_target, q2_target)
  DevBuf<float> atoms_, probs_t_, probs_o_, ev_t_, up51_, db51_, head_wpart_;
  std::array<WeightMirror, 4> heads_;
  int head_splits_ = 0, c51_blocks_ = 0;

  std::vector<mlp::Step> steps_;
  // update graphs: one update, and two back to back (update_n replays the
  // pair, so the second update's sample overlaps the first one's Adam)
  cudaGraphExec_t graph_exec_ = nullptr, graph2_exec_ = nullptr;
  bool capture_ = false;  // steps are being captured into an update graph
  bool graph_checked_ = false;
  int kpu_ = 0;
};

// PolicyLearnerCore (learners.hpp:110-139): the actor gradient through the
// frozen online critic replicas (ddpg_actor_loss, ddpg.hpp:86-118), clip +
// Adam on the policy (learners.cpp:239-270).
class PLearner {
 public:
  PLearner(const pqlg_config& cfg, const pqlg_task_dims& dims, uint64_t init_seed,
           cudaStream_t st, pqlg_comm_s* comm = nullptr);
  ~PLearner();

  void adopt_critics(const float* q1_host, const float* q2_host, int64_t version);
  void adopt_critics_device(const float* q1_dev, const float* q2_dev, int64_t version);
  void adopt_norm(int64_t count, const double* mean, const double* m2);
  void adopt_norm_device(const int64_t* count, const double* mean, const double* m2) {
    norm_.set_device(count, mean, m2, stream_);
  }
  int64_t policy_params() const { return pnet_.params; }
  int64_t critic_params() const { return qnet_.params; }
  // device policy snapshot [net | log_alpha] (pql_sac) as the pipeline moves it
  int64_t snapshot_len() const { return pnet_.params + (sac_ ? 1 : 0); }
  float log_alpha();
  const NetShape& policy_shape() const { return pnet_; }
  const NetShape& critic_shape() const { return qnet_; }
  int64_t norm_count_ = 0;  // NormStats last adopted from the host (checkpointing)
  std::vector<double> norm_mean_, norm_m2_;
  void ingest(const float* states_dev, int64_t ld, uint64_t n);
  void ingest_host(const float* states_host, int64_t ld, uint64_t n);
  bool ready(int64_t c_a);
  float update();
  void update_n(int n);
  float last_loss();
  void get_params(int which, float* out);
  void set_params(int which, const float* flat_host);
  int64_t param_count(int which) const;
  void set_mt_mode(bool on) { mt_mode_ = on; }
  int kernels_per_update();
  // Per-kernel device times of the update graph (time_in_graph, common.h).
  std::string time_update(int reps);
  uint64_t buffer_size() { return states_->size(); }
  const float* policy_dev() const { return pol_.p; }
  int obs_dim() const { return D_; }
  cudaStream_t stream() const { return stream_; }
  int64_t critic_version() const { return critic_version_; }
  int check_status();  // as VLearner::check_status

 private:
  void build_update();
  void enqueue();

  pqlg_config cfg_;
  pqlg_task_dims dims_;
  cudaStream_t stream_;
  cudaStream_t owned_stream_ = nullptr;
  pqlg_comm_s* comm_ = nullptr;  // data-parallel communicator (nullable)
  int rank_ = 0, world_ = 1;
  int D_, A_, Ap_, H_, nh_, B_, Kp_;
  int Ah_ = 0, Ahp_ = 0;  // policy head outputs (A, or 2A for pql_sac) and padded stride
  bool dist_ = false;  // PQL-D actor objective (c51_actor_loss)
  bool sac_ = false;   // pql_sac actor objective + alpha update
  EpsStream eps_;
  DevBuf<float> sd_, logp_;  // pql_sac: +-std [B x Ap], log pi [B]
  int L_ = 1, Lp_ = 1;
  NetShape qnet_, pnet_;
  int64_t Ps_ = 0;
  int64_t critic_version_ = 0;

  DevBuf<float> pol_, m_, v_, grads_, q_;
  WeightMirror head_;
  mlp::HeadSplit head_split_;
  std::unique_ptr<DeviceStates> states_;
  DevBuf<float> in_f_;  // host-ingest staging
  DeviceNorm norm_;
  DevBuf<replay::SamplerState> sampler_;
  bool mt_mode_ = false;
  std::mt19937_64 mt_;
  DevBuf<uint64_t> idx_;
  std::vector<uint64_t> idx_host_;
  DevBuf<int64_t> step_;
  DevBuf<float2> bc_;
  DevBuf<uint32_t> status_;
  DevBuf<float> loss_;
  PinnedBuf<uint32_t> hbuf_;  // update(): loss bits + status

  DevBuf<float> X_, T_, dy_, up_, part_;
  std::vector<DevBuf<float>> pact_, Gp_;
  std::vector<DevBuf<uint32_t>> pmask_;
  std::array<std::vector<DevBuf<float>>, 2> cact_, Gc_;
  std::array<std::vector<DevBuf<uint32_t>>, 2> cmask_;
  std::array<DevBuf<float>, 2> dact_;
  DevBuf<double> block_loss_;
  DevBuf<unsigned int> loss_counter_;
  std::vector<DevBuf<float>> wpart_, colsum_;
  std::vector<int> wsplits_;
  DevBuf<float> head_db_;
  DevBuf<double> block_sq_;
  DevBuf<unsigned int> fin_counter_;
  DevBuf<float> scale_;
  std::unique_ptr<DpBuckets> dp_;  // data-parallel gradient buckets (comm_ only)
  DevBuf<float> atoms_, probs_, ev_, up51_;  // C51 actor objective
  std::array<WeightMirror, 2> heads_;

  DevBuf<float> wpack_;  // policy head W in the head kernel's fragment order
  std::vector<mlp::Step> steps_;
  cudaGraphExec_t graph_exec_ = nullptr, graph2_exec_ = nullptr;  // (as VLearner)
  bool capture_ = false;
  int kpu_ = 0;
};

}  // namespace pqlg
