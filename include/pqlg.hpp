// Header-only C++ layer over the pqlg C ABI (include/pqlg.h): RAII handles
// named after the reference's runtime cores (proj/include/pql/runtime/
// learners.hpp:52-139) that throw the reference's exception types:
//   PQLG_EINVAL                -> std::invalid_argument  (RunConfig::validate)
//   PQLG_ENONFINITE            -> std::runtime_error     (learners.cpp:164, :248)
//   PQLG_NOT_READY             -> std::runtime_error     ("update before warm-up")
//   PQLG_ECUDA / PQLG_ENCCL    -> std::runtime_error
// Only std types cross this header, so a reference build can include it
// without pulling in CUDA (INTEGRATION.md shows the adaptation to pql::rt).
#pragma once

#include <cstdint>
#include <stdexcept>
#include <string>
#include <vector>

#include "pqlg.h"

namespace pqlg {

inline void check(int status) {
  if (status == PQLG_OK) return;
  const std::string msg = pqlg_last_error();
  if (status == PQLG_EINVAL) throw std::invalid_argument(msg);
  throw std::runtime_error(msg);
}

// Reference std::vector<std::uint8_t> flags and MatF rows as plain views.
struct HostSlice {
  const float* obs;
  const float* act;
  const float* boot_obs;
  const float* rew;
  const std::uint8_t* term;
  const std::uint8_t* trunc;
};

// CriticLearnerCore (learners.hpp:77-106).
class VLearner {
 public:
  VLearner(const pqlg_config& cfg, const pqlg_task_dims& dims, std::uint64_t init_seed,
           void* stream = nullptr) {
    check(pqlg_vlearner_create(&cfg, &dims, init_seed, stream, &h_));
  }
  ~VLearner() {
    if (h_) pqlg_vlearner_destroy(h_);
  }
  VLearner(const VLearner&) = delete;
  VLearner& operator=(const VLearner&) = delete;

  void adopt_policy(const std::vector<float>& flat, std::int64_t version) {
    check(pqlg_vlearner_adopt_policy(h_, flat.data(), version));
  }
  void adopt_norm(std::int64_t count, const double* mean, const double* m2) {
    const pqlg_norm_stats n{count, mean, m2};
    check(pqlg_vlearner_adopt_norm(h_, &n));
  }
  void ingest(const pqlg_step_slice& device_views) { check(pqlg_vlearner_ingest(h_, &device_views)); }
  void ingest_host(const HostSlice& s) {
    const pqlg_step_slice v{s.obs, s.act, s.boot_obs, s.rew, s.term, s.trunc, 0, 0};
    check(pqlg_vlearner_ingest_host(h_, &v));
  }
  bool ready(std::int64_t c_a) const {
    int r = 0;
    check(pqlg_vlearner_ready(h_, c_a, &r));
    return r != 0;
  }
  float update() {
    float loss = 0.0f;
    check(pqlg_vlearner_update(h_, &loss));
    return loss;
  }
  void update_n(int n) { check(pqlg_vlearner_update_n(h_, n)); }
  std::int64_t param_count() const {
    std::int64_t n = 0;
    check(pqlg_vlearner_param_count(h_, 0, &n));
    return n;
  }
  // CriticSnapshot{q1, q2} online nets (learners.cpp:190-196)
  void snapshot(std::vector<float>& q1, std::vector<float>& q2) const {
    q1.resize(param_count());
    q2.resize(param_count());
    check(pqlg_vlearner_snapshot(h_, q1.data(), q2.data()));
  }
  std::uint64_t buffer_size() const {
    std::uint64_t n = 0;
    check(pqlg_vlearner_buffer_size(h_, &n));
    return n;
  }
  // which: 0 q1, 1 q2, 2 q1_target, 3 q2_target, 4 lagged policy
  std::int64_t param_count(int which) const {
    std::int64_t n = 0;
    check(pqlg_vlearner_param_count(h_, which, &n));
    return n;
  }
  void set_params(int which, const std::vector<float>& flat) {
    if (static_cast<std::int64_t>(flat.size()) != param_count(which))
      throw std::invalid_argument("set_params: parameter count mismatch");
    check(pqlg_vlearner_set_params(h_, which, flat.data()));
  }
  void get_params(int which, std::vector<float>& flat) const {
    flat.resize(static_cast<std::size_t>(param_count(which)));
    check(pqlg_vlearner_get_params(h_, which, flat.data()));
  }
  // pql_sac: adopt a PolicySnapshot's net and log_alpha (equal-or-newer)
  void adopt_policy_sac(const std::vector<float>& flat, float log_alpha, std::int64_t version) {
    check(pqlg_vlearner_adopt_policy_sac(h_, flat.data(), log_alpha, version));
  }
  void set_sampler(int mode) { check(pqlg_vlearner_set_sampler(h_, mode)); }
  pqlg_vlearner handle() const { return h_; }

 private:
  pqlg_vlearner h_ = nullptr;
};

// PolicyLearnerCore (learners.hpp:110-139).
class PLearner {
 public:
  PLearner(const pqlg_config& cfg, const pqlg_task_dims& dims, std::uint64_t init_seed,
           void* stream = nullptr) {
    check(pqlg_plearner_create(&cfg, &dims, init_seed, stream, &h_));
  }
  ~PLearner() {
    if (h_) pqlg_plearner_destroy(h_);
  }
  PLearner(const PLearner&) = delete;
  PLearner& operator=(const PLearner&) = delete;

  void adopt_critics(const std::vector<float>& q1, const std::vector<float>& q2,
                     std::int64_t version) {
    check(pqlg_plearner_adopt_critics(h_, q1.data(), q2.data(), version));
  }
  void adopt_norm(std::int64_t count, const double* mean, const double* m2) {
    const pqlg_norm_stats n{count, mean, m2};
    check(pqlg_plearner_adopt_norm(h_, &n));
  }
  void ingest(const float* states_dev, std::int64_t ld, std::uint64_t n) {
    check(pqlg_plearner_ingest(h_, states_dev, ld, n));
  }
  void ingest_host(const float* states, std::int64_t ld, std::uint64_t n) {
    check(pqlg_plearner_ingest_host(h_, states, ld, n));
  }
  bool ready(std::int64_t c_a) const {
    int r = 0;
    check(pqlg_plearner_ready(h_, c_a, &r));
    return r != 0;
  }
  float update() {
    float loss = 0.0f;
    check(pqlg_plearner_update(h_, &loss));
    return loss;
  }
  void update_n(int n) { check(pqlg_plearner_update_n(h_, n)); }
  std::vector<float> snapshot() const {
    std::int64_t n = 0;
    check(pqlg_plearner_param_count(h_, 0, &n));
    std::vector<float> flat(static_cast<std::size_t>(n));
    check(pqlg_plearner_snapshot(h_, flat.data()));
    return flat;
  }
  // which: 0 policy, 1 critic replica q1, 2 critic replica q2
  std::int64_t param_count(int which) const {
    std::int64_t n = 0;
    check(pqlg_plearner_param_count(h_, which, &n));
    return n;
  }
  void set_params(int which, const std::vector<float>& flat) {
    if (static_cast<std::int64_t>(flat.size()) != param_count(which))
      throw std::invalid_argument("set_params: parameter count mismatch");
    check(pqlg_plearner_set_params(h_, which, flat.data()));
  }
  void get_params(int which, std::vector<float>& flat) const {
    flat.resize(static_cast<std::size_t>(param_count(which)));
    check(pqlg_plearner_get_params(h_, which, flat.data()));
  }
  float log_alpha() const {
    float a = 0.0f;
    check(pqlg_plearner_log_alpha(h_, &a));
    return a;
  }
  std::uint64_t buffer_size() const {
    std::uint64_t n = 0;
    check(pqlg_plearner_buffer_size(h_, &n));
    return n;
  }
  void set_sampler(int mode) { check(pqlg_plearner_set_sampler(h_, mode)); }
  pqlg_plearner handle() const { return h_; }

 private:
  pqlg_plearner h_ = nullptr;
};

// ActorCore (learners.hpp:52-73) over the synthetic GPU env.
class Actor {
 public:
  Actor(const pqlg_config& cfg, const pqlg_task_dims& dims, void* stream = nullptr) {
    check(pqlg_actor_create(&cfg, &dims, stream, &h_));
  }
  ~Actor() {
    if (h_) pqlg_actor_destroy(h_);
  }
  Actor(const Actor&) = delete;
  Actor& operator=(const Actor&) = delete;

  void adopt_policy(const std::vector<float>& flat, std::int64_t version) {
    check(pqlg_actor_adopt_policy(h_, flat.data(), version));
  }
  // device views valid until the next rollout_step
  pqlg_step_slice rollout_step() {
    pqlg_step_slice s{};
    check(pqlg_actor_rollout_step(h_, &s));
    return s;
  }
  std::int64_t policy_version() const {
    std::int64_t v = 0;
    check(pqlg_actor_policy_version(h_, &v));
    return v;
  }
  // the last rollout_step's StepSlice into host rows (any pointer may be null)
  void read_slice(float* obs, float* act, float* boot_obs, float* rew, std::uint8_t* term,
                  std::uint8_t* trunc) const {
    check(pqlg_actor_read_slice(h_, obs, act, boot_obs, rew, term, trunc));
  }
  // running NormStats (mean / m2 sized obs_dim)
  std::int64_t norm(double* mean, double* m2) const {
    std::int64_t count = 0;
    check(pqlg_actor_norm(h_, &count, mean, m2));
    return count;
  }
  pqlg_actor handle() const { return h_; }

 private:
  pqlg_actor h_ = nullptr;
};

}  // namespace pqlg
