// ref_harness.cpp -- extern "C" entry points into the UNMODIFIED reference
// (/root/reference/proj), compiled by `make -C oracle ref` into
// oracle/_ref/libpqlref.so.  TEST INFRASTRUCTURE ONLY: used to pin the CPU
// restatement (pql_oracle.c), to generate tests/golden fixtures, and as the
// timed CPU baseline (bench.py --impl reference).  Every function below just
// drives the reference's own classes/functions in the order the reference's
// runtime cores use them (proj/src/runtime/learners.cpp).
#include <cmath>
#include <cstdint>
#include <cstring>
#include <memory>
#include <random>
#include <stdexcept>
#include <vector>

#include "pql/agents/c51.hpp"
#include "pql/agents/ddpg.hpp"
#include "pql/agents/sac.hpp"
#include "pql/explore/noise.hpp"
#include "pql/funcapprox/checkpoint.hpp"
#include "pql/funcapprox/normalizer.hpp"
#include "pql/funcapprox/optim.hpp"
#include "pql/kernels/kernels.hpp"
#include "pql/replay/nstep.hpp"
#include "pql/replay/replay_buffer.hpp"
#include "pql/rng.hpp"
#include "pql/runtime/learners.hpp"
#include "pql/runtime/metrics.hpp"
#include "pql/sched/ratio_gate.hpp"
#include "pql/vecenv/vecenv.hpp"

using namespace pql;

#define REF_API extern "C" __attribute__((visibility("default")))

namespace {

fa::Mlp<float> make_mlp(const size_t* sizes, size_t n_layers, const float* flat) {
  std::vector<std::size_t> s(sizes, sizes + n_layers + 1);
  std::vector<fa::Act> acts(n_layers, fa::Act::relu);
  acts.back() = fa::Act::identity;
  auto net = fa::Mlp<float>::zeros(s, acts);
  if (flat) std::memcpy(net.flat.data(), flat, net.flat.size() * sizeof(float));
  return net;
}

MatF make_mat(const float* p, size_t rows, size_t cols) {
  MatF m(rows, cols);
  if (p) std::memcpy(m.data(), p, rows * cols * sizeof(float));
  return m;
}

replay::NStepBatch<float> make_batch(const float* obs, const float* act, const float* boot,
                                     const float* ret, const float* eff, size_t B, size_t D,
                                     size_t A) {
  replay::NStepBatch<float> b;
  b.obs = make_mat(obs, B, D);
  b.act = make_mat(act, B, A);
  b.boot_obs = make_mat(boot, B, D);
  b.ret.assign(ret, ret + B);
  b.eff_disc.assign(eff, eff + B);
  return b;
}

fa::NormStats make_stats(int64_t count, const double* mean, const double* m2, size_t D) {
  fa::NormStats s;
  s.count = count;
  s.mean.assign(mean, mean + D);
  s.m2.assign(m2, m2 + D);
  return s;
}

}  // namespace

// ------------------------------------------------- Philox URBG
// Random123 Philox4x32-10 (the published algorithm; the device uses the same
// rounds and constants, rng.cuh) as a UniformRandomBitGenerator: draw k is
// the 64-bit (out0 | out1 << 32) of philox(key, ctr + k).  Driving libstdc++'s
// own uniform_int_distribution<size_t> -- the call of ReplayBuffer::sample
// (replay_buffer.hpp:58-60) -- with it defines the device sampler's indices.
namespace {
struct PhiloxURBG {
  using result_type = uint64_t;
  uint64_t key, ctr;
  static constexpr result_type min() { return 0; }
  static constexpr result_type max() { return ~result_type(0); }
  result_type operator()() {
    uint32_t c[4] = {static_cast<uint32_t>(ctr), static_cast<uint32_t>(ctr >> 32), 0u, 0u};
    uint32_t k[2] = {static_cast<uint32_t>(key), static_cast<uint32_t>(key >> 32)};
    for (int round = 0; round < 10; ++round) {
      const uint64_t p0 = static_cast<uint64_t>(0xD2511F53u) * c[0];
      const uint64_t p1 = static_cast<uint64_t>(0xCD9E8D57u) * c[2];
      const uint32_t n0 = static_cast<uint32_t>(p1 >> 32) ^ c[1] ^ k[0];
      const uint32_t n2 = static_cast<uint32_t>(p0 >> 32) ^ c[3] ^ k[1];
      c[0] = n0;
      c[1] = static_cast<uint32_t>(p1);
      c[2] = n2;
      c[3] = static_cast<uint32_t>(p0);
      k[0] += 0x9E3779B9u;
      k[1] += 0xBB67AE85u;
    }
    ++ctr;
    return static_cast<uint64_t>(c[0]) | (static_cast<uint64_t>(c[1]) << 32);
  }
};
}  // namespace

// B draws of std::uniform_int_distribution<size_t>(0, count-1) over PhiloxURBG;
// returns the advanced counter.
REF_API uint64_t ref_sample_indices_philox(uint64_t key, uint64_t counter, uint64_t count,
                                           size_t B, uint64_t* out) {
  PhiloxURBG g{key, counter};
  std::uniform_int_distribution<std::size_t> pick(0, count - 1);
  for (size_t r = 0; r < B; ++r) out[r] = pick(g);
  return g.ctr;
}

// RatioGate::may_proceed (ratio_gate.hpp:44-60), compiled from the reference
REF_API int ref_ratio_may_proceed(int proc, int64_t ca, int64_t cv, int64_t cp, double beta_av,
                                  double beta_pv, double slack_a, double slack_p,
                                  double slack_v, int64_t warm_up, int free_running) {
  sched::RatioConfig c;
  c.beta_av = beta_av;
  c.beta_pv = beta_pv;
  c.slack_a = slack_a;
  c.slack_p = slack_p;
  c.slack_v = slack_v;
  c.warm_up = warm_up;
  c.free_running = free_running != 0;
  const sched::Proc p = proc == 0 ? sched::Proc::actor
                        : proc == 1 ? sched::Proc::vlearner
                                    : sched::Proc::plearner;
  return sched::RatioGate::may_proceed(p, ca, cv, cp, c) ? 1 : 0;
}

// ------------------------------------------------------------ backend
// kernels::set_backend (kernels.hpp:17-20): 0 scalar (op-order ground truth),
// 1 avx2 (the default on this CPU; FMA-reassociated affine kernels).
REF_API void ref_set_backend(int b) {
  kernels::set_backend(b == 0 ? kernels::Backend::scalar : kernels::Backend::avx2);
}
REF_API int ref_active_backend() {
  return kernels::active_backend() == kernels::Backend::scalar ? 0 : 1;
}

// ---------------------------------------------------------------- rng
REF_API uint64_t ref_derive_seed(uint64_t master, uint64_t stream, uint64_t index) {
  return derive_seed(master, static_cast<RngStream>(stream), index);
}

REF_API void ref_mt64_draws(uint64_t seed, size_t n, uint64_t* out) {
  std::mt19937_64 g(seed);
  for (size_t i = 0; i < n; ++i) out[i] = g();
}

// Indices drawn by n_calls successive ReplayBuffer::sample(B) calls of a
// learner whose sample_rng_ = make_rng(seed, sample, learner)
// (learners.cpp:136, :212).  Row i of the buffer carries ret = i.
REF_API void ref_sample_indices(uint64_t seed, uint64_t learner, uint64_t count, size_t B,
                                size_t n_calls, uint64_t* out) {
  replay::ReplayBuffer buf(count, 1, 1);
  replay::NStepBatch<float> b;
  b.obs.resize(count, 1);
  b.act.resize(count, 1);
  b.boot_obs.resize(count, 1);
  b.ret.resize(count);
  b.eff_disc.assign(count, 0.0f);
  for (size_t i = 0; i < count; ++i) b.ret[i] = static_cast<float>(i);
  buf.insert(b);
  auto rng = make_rng(seed, RngStream::sample, learner);
  for (size_t c = 0; c < n_calls; ++c) {
    auto s = buf.sample(B, rng, 1);
    for (size_t r = 0; r < B; ++r) out[c * B + r] = static_cast<uint64_t>(s->ret[r]);
  }
}

// ---------------------------------------------------------- n-step + ring
// T steps of NStepAssembler::push_step (rewards already scaled) followed by
// ReplayBuffer::insert into a ring of capacity cap.  Returns total emitted
// rows; emitted rows are written up to max_rows; ring obs/ret are dumped via
// the public obs_row / ret_at accessors (replay_buffer.hpp:71-73).
REF_API size_t ref_nstep_replay(size_t T, size_t N, size_t D, size_t A, float gamma, size_t n,
                                size_t cap, const float* obs, const float* act, const float* boot,
                                const float* rew, const uint8_t* term, const uint8_t* trunc,
                                uint64_t* emit_counts, float* e_obs, float* e_act, float* e_boot,
                                float* e_ret, float* e_eff, size_t max_rows, float* ring_obs,
                                float* ring_ret, uint64_t* cursor_count) {
  replay::NStepAssembler<float> as(N, D, A, gamma, n);
  replay::ReplayBuffer buf(cap, D, A);
  replay::NStepBatch<float> out;
  size_t total = 0;
  for (size_t t = 0; t < T; ++t) {
    MatF o = make_mat(obs + t * N * D, N, D), a = make_mat(act + t * N * A, N, A),
         bo = make_mat(boot + t * N * D, N, D);
    out.clear();
    as.push_step(o, a, std::span<const float>(rew + t * N, N),
                 std::span<const uint8_t>(term + t * N, N),
                 std::span<const uint8_t>(trunc + t * N, N), bo, out);
    emit_counts[t] = out.size();
    for (size_t r = 0; r < out.size() && total + r < max_rows; ++r) {
      const size_t k = total + r;
      std::memcpy(e_obs + k * D, out.obs.row(r), D * sizeof(float));
      std::memcpy(e_act + k * A, out.act.row(r), A * sizeof(float));
      std::memcpy(e_boot + k * D, out.boot_obs.row(r), D * sizeof(float));
      e_ret[k] = out.ret[r];
      e_eff[k] = out.eff_disc[r];
    }
    total += out.size();
    buf.insert(out);
  }
  for (size_t i = 0; i < cap; ++i) {
    std::memcpy(ring_obs + i * D, buf.obs_row(i), D * sizeof(float));
    ring_ret[i] = buf.ret_at(i);
  }
  cursor_count[0] = buf.cursor();
  cursor_count[1] = buf.size();
  return total;
}

// StateBuffer insert of T batches of N rows, then n_calls sample(B) with
// make_rng(seed, sample, 2) (learners.cpp:212).
REF_API void ref_state_buffer(size_t cap, size_t D, size_t T, size_t N, const float* rows,
                              uint64_t seed, size_t B, size_t n_calls, float* out,
                              uint64_t* count_out) {
  replay::StateBuffer sb(cap, D);
  for (size_t t = 0; t < T; ++t) sb.insert(make_mat(rows + t * N * D, N, D));
  auto rng = make_rng(seed, RngStream::sample, 2);
  for (size_t c = 0; c < n_calls; ++c) {
    auto s = sb.sample(B, rng, 1);
    std::memcpy(out + c * B * D, s->data(), B * D * sizeof(float));
  }
  *count_out = sb.size();
}

// ------------------------------------------------------------- normalizer
REF_API void ref_normalizer(size_t D, size_t n_batches, const size_t* rows, const float* data,
                            int64_t* count_out, double* mean_out, double* m2_out, const float* x,
                            size_t Bx, float* xn_out) {
  fa::RunningNormalizer norm(D);
  size_t off = 0;
  for (size_t i = 0; i < n_batches; ++i) {
    norm.update(make_mat(data + off * D, rows[i], D));
    off += rows[i];
  }
  const auto& s = norm.stats();
  *count_out = s.count;
  std::memcpy(mean_out, s.mean.data(), D * sizeof(double));
  std::memcpy(m2_out, s.m2.data(), D * sizeof(double));
  MatF xn = norm.apply(make_mat(x, Bx, D));
  std::memcpy(xn_out, xn.data(), Bx * D * sizeof(float));
}

REF_API void ref_normalize_apply(int64_t count, const double* mean, const double* m2, size_t D,
                                 const float* x, size_t B, float* out) {
  MatF r = fa::RunningNormalizer::apply_stats(make_stats(count, mean, m2, D), make_mat(x, B, D));
  std::memcpy(out, r.data(), B * D * sizeof(float));
}

// ------------------------------------------------------------------ optim
REF_API int ref_adam_step(float* p, const float* g, float* m, float* v, size_t n, int64_t t,
                          float lr) {
  std::vector<float> params(p, p + n), grads(g, g + n);
  fa::AdamState<float> st(n);
  st.m.assign(m, m + n);
  st.v.assign(v, v + n);
  st.t = t;
  try {
    fa::adam_step(params, grads, st, lr);
  } catch (const std::exception&) {
    return -2;
  }
  std::memcpy(p, params.data(), n * sizeof(float));
  std::memcpy(m, st.m.data(), n * sizeof(float));
  std::memcpy(v, st.v.data(), n * sizeof(float));
  return 0;
}

REF_API void ref_clip_global_norm(float* g, size_t n, float max_norm) {
  std::vector<float> v(g, g + n);
  fa::clip_global_norm(v, max_norm);
  std::memcpy(g, v.data(), n * sizeof(float));
}

REF_API double ref_sum_squares(const float* x, size_t n) { return kernels::sum_squares(x, n); }

REF_API void ref_soft_update(float* target, const float* online, size_t n, float tau) {
  std::vector<float> t(target, target + n), o(online, online + n);
  fa::soft_update(t, o, tau);
  std::memcpy(target, t.data(), n * sizeof(float));
}

// ------------------------------------------------------------------ noise
REF_API void ref_build_schedule(float smin, float smax, size_t n, float* out) {
  auto s = explore::build_schedule(smin, smax, n);
  std::memcpy(out, s.sigma.data(), n * sizeof(float));
}

// `steps` successive apply_noise calls with the actor's per-env noise
// streams (learners.cpp:74-75); actions [steps][N][A] are perturbed in place.
REF_API void ref_apply_noise(float smin, float smax, size_t N, size_t A, uint64_t seed,
                             size_t steps, float low, float high, float* actions) {
  auto sched = explore::build_schedule(smin, smax, N);
  std::vector<env::SplitMixEngine> rngs(N);
  for (size_t i = 0; i < N; ++i) rngs[i].state = derive_seed(seed, RngStream::noise, i);
  for (size_t s = 0; s < steps; ++s) {
    MatF a = make_mat(actions + s * N * A, N, A);
    explore::apply_noise(a, sched, low, high, rngs);
    std::memcpy(actions + s * N * A, a.data(), N * A * sizeof(float));
  }
}

// -------------------------------------------------------------------- MLP
REF_API void ref_mlp_forward(const float* flat, const size_t* sizes, size_t n_layers,
                             const float* in, size_t B, float* out) {
  auto net = make_mlp(sizes, n_layers, flat);
  MatF y = fa::forward(net, make_mat(in, B, sizes[0]));
  std::memcpy(out, y.data(), B * sizes[n_layers] * sizeof(float));
}

REF_API void ref_mlp_backward(const float* flat, const size_t* sizes, size_t n_layers,
                              const float* in, const float* upstream, size_t B, float* grads,
                              float* dinput) {
  auto net = make_mlp(sizes, n_layers, flat);
  fa::ForwardCache<float> cache;
  fa::forward(net, make_mat(in, B, sizes[0]), &cache);
  std::vector<float> g;
  MatF din;
  fa::backward(net, cache, make_mat(upstream, B, sizes[n_layers]), g, dinput ? &din : nullptr);
  std::memcpy(grads, g.data(), g.size() * sizeof(float));
  if (dinput) std::memcpy(dinput, din.data(), B * sizes[0] * sizeof(float));
}

// Orthogonal init exactly as PolicyHandle::create (learners.cpp:17-33) and
// CriticPair::create (critic.hpp:16-26).
REF_API void ref_init_mlp(const size_t* sizes, size_t n_layers, uint64_t rng_seed,
                          float hidden_gain, float final_gain, size_t n_nets, float* out) {
  std::mt19937_64 rng(rng_seed);
  for (size_t k = 0; k < n_nets; ++k) {
    auto net = make_mlp(sizes, n_layers, nullptr);
    fa::init_orthogonal(net, rng, hidden_gain, final_gain);
    std::memcpy(out + k * net.flat.size(), net.flat.data(), net.flat.size() * sizeof(float));
  }
}

// ----------------------------------------------------------------- agents
namespace {
agents::DeterministicPolicy<float> make_policy(const float* flat, const size_t* sizes,
                                               size_t n_layers, float low, float high) {
  agents::DeterministicPolicy<float> p;
  p.net = make_mlp(sizes, n_layers, flat);
  p.low = low;
  p.high = high;
  return p;
}
agents::CriticPair<float> make_pair(const float* q1, const float* q2, const float* q1t,
                                    const float* q2t, const size_t* sizes, size_t n_layers) {
  agents::CriticPair<float> c;
  c.q1 = make_mlp(sizes, n_layers, q1);
  c.q2 = make_mlp(sizes, n_layers, q2);
  c.q1_target = make_mlp(sizes, n_layers, q1t ? q1t : q1);
  c.q2_target = make_mlp(sizes, n_layers, q2t ? q2t : q2);
  return c;
}
}  // namespace

REF_API int ref_ddpg_critic_loss(const float* pol, const size_t* psizes, const float* q1,
                                 const float* q2, const float* q1t, const float* q2t,
                                 const size_t* qsizes, size_t n_layers, const float* obs_norm,
                                 const float* act, const float* boot_norm, const float* ret,
                                 const float* eff, size_t B, size_t D, size_t A, float low,
                                 float high, float* loss, float* y, float* dq1, float* dq2) {
  auto policy = make_policy(pol, psizes, n_layers, low, high);
  auto pair = make_pair(q1, q2, q1t, q2t, qsizes, n_layers);
  auto batch = make_batch(obs_norm, act, boot_norm, ret, eff, B, D, A);
  try {
    if (y) {
      auto yy = agents::ddpg_critic_target(batch, policy, pair);
      std::memcpy(y, yy.data(), B * sizeof(float));
    }
    auto r = agents::ddpg_critic_loss(batch, policy, pair);
    *loss = r.loss;
    std::memcpy(dq1, r.dq1.data(), r.dq1.size() * sizeof(float));
    std::memcpy(dq2, r.dq2.data(), r.dq2.size() * sizeof(float));
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API int ref_ddpg_actor_loss(const float* pol, const size_t* psizes, const float* q1,
                                const float* q2, const size_t* qsizes, size_t n_layers,
                                const float* states, size_t B, size_t D, float low, float high,
                                float* loss, float* dpolicy) {
  auto policy = make_policy(pol, psizes, n_layers, low, high);
  auto pair = make_pair(q1, q2, nullptr, nullptr, qsizes, n_layers);
  try {
    auto r = agents::ddpg_actor_loss(make_mat(states, B, D), policy, pair);
    *loss = r.loss;
    std::memcpy(dpolicy, r.dpolicy.data(), r.dpolicy.size() * sizeof(float));
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API int ref_c51_project(const float* probs, const float* ret, const float* eff, size_t B,
                            size_t L, float vmin, float vmax, float* out) {
  auto head = agents::CategoricalHead<float>::create(L, vmin, vmax);
  try {
    MatF q = agents::c51_project<float>(make_mat(probs, B, L), std::span<const float>(ret, B),
                                        std::span<const float>(eff, B), head);
    std::memcpy(out, q.data(), B * L * sizeof(float));
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API void ref_c51_atoms(size_t L, float vmin, float vmax, float* out) {
  auto head = agents::CategoricalHead<float>::create(L, vmin, vmax);
  std::memcpy(out, head.atoms.data(), L * sizeof(float));
}

REF_API int ref_c51_critic_loss(const float* pol, const size_t* psizes, const float* q1,
                                const float* q2, const float* q1t, const float* q2t,
                                const size_t* qsizes, size_t n_layers, const float* obs_norm,
                                const float* act, const float* boot_norm, const float* ret,
                                const float* eff, size_t B, size_t D, size_t A, float low,
                                float high, size_t L, float vmin, float vmax, float* loss,
                                float* dq1, float* dq2) {
  auto policy = make_policy(pol, psizes, n_layers, low, high);
  auto pair = make_pair(q1, q2, q1t, q2t, qsizes, n_layers);
  auto batch = make_batch(obs_norm, act, boot_norm, ret, eff, B, D, A);
  auto head = agents::CategoricalHead<float>::create(L, vmin, vmax);
  try {
    auto r = agents::c51_critic_loss(batch, policy, pair, head);
    *loss = r.loss;
    std::memcpy(dq1, r.dq1.data(), r.dq1.size() * sizeof(float));
    std::memcpy(dq2, r.dq2.data(), r.dq2.size() * sizeof(float));
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API int ref_c51_actor_loss(const float* pol, const size_t* psizes, const float* q1,
                               const float* q2, const size_t* qsizes, size_t n_layers,
                               const float* states, size_t B, size_t D, float low, float high,
                               size_t L, float vmin, float vmax, float* loss, float* dpolicy) {
  auto policy = make_policy(pol, psizes, n_layers, low, high);
  auto pair = make_pair(q1, q2, nullptr, nullptr, qsizes, n_layers);
  auto head = agents::CategoricalHead<float>::create(L, vmin, vmax);
  try {
    auto r = agents::c51_actor_loss(make_mat(states, B, D), policy, pair, head);
    *loss = r.loss;
    std::memcpy(dpolicy, r.dpolicy.data(), r.dpolicy.size() * sizeof(float));
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

// ----------------------------------------------- V-learner update (agents)
// One CriticLearnerCore::update (learners.cpp:157-188) for an arbitrary
// depth of network, composed from the reference's own replay / normalizer /
// agents / optim calls in the same order.  State arrays are updated in place.
struct RefCritic {
  size_t D, A, n_layers, B;
  std::vector<size_t> qsizes, psizes;
  float low = -1.0f, high = 1.0f, lr = 5e-4f, tau = 0.05f;
  int distributional = 0;
  size_t n_atoms = 51;
  float vmin = -10.0f, vmax = 10.0f;
  agents::CriticPair<float> critics;
  fa::AdamState<float> adam_q1, adam_q2;
  agents::DeterministicPolicy<float> lagged;
  int sac = 0;  // algo 2: pql_sac (GaussianPolicy lagged, eps stream, alpha)
  agents::GaussianPolicy<float> lagged_g;
  float log_alpha = 0.0f;
  std::mt19937_64 eps_rng;
  fa::NormStats norm;
  std::unique_ptr<replay::ReplayBuffer> buffer;
  std::mt19937_64 sample_rng;
};

REF_API void* ref_vupdate_create(size_t D, size_t A, size_t hidden, size_t n_hidden, size_t B,
                                 size_t capacity, uint64_t seed, const float* q1, const float* q2,
                                 const float* policy, int distributional, size_t n_atoms,
                                 float vmin, float vmax) {
  auto* r = new RefCritic();
  r->D = D; r->A = A; r->B = B; r->n_layers = n_hidden + 1;
  r->sac = distributional == 2;  // `distributional` doubles as algo: 0 ddpg, 1 c51, 2 sac
  if (r->sac) distributional = 0;
  r->distributional = distributional; r->n_atoms = n_atoms; r->vmin = vmin; r->vmax = vmax;
  r->qsizes.push_back(D + A);
  r->psizes.push_back(D);
  for (size_t i = 0; i < n_hidden; ++i) {
    r->qsizes.push_back(hidden);
    r->psizes.push_back(hidden);
  }
  r->qsizes.push_back(distributional ? n_atoms : 1);
  r->psizes.push_back(r->sac ? 2 * A : A);
  r->critics = make_pair(q1, q2, nullptr, nullptr, r->qsizes.data(), r->n_layers);
  r->adam_q1 = fa::AdamState<float>(r->critics.q1.param_count());
  r->adam_q2 = fa::AdamState<float>(r->critics.q2.param_count());
  if (r->sac) {
    r->lagged_g.net = make_mlp(r->psizes.data(), r->n_layers, policy);
    r->eps_rng = make_rng(seed, RngStream::sac, 1);  // learners.cpp:137
  } else {
    r->lagged = make_policy(policy, r->psizes.data(), r->n_layers, -1.0f, 1.0f);
  }
  r->buffer = std::make_unique<replay::ReplayBuffer>(capacity, D, A);
  r->sample_rng = make_rng(seed, RngStream::sample, 1);
  return r;
}

REF_API void ref_vupdate_destroy(void* h) { delete static_cast<RefCritic*>(h); }

REF_API void ref_vupdate_insert(void* h, const float* obs, const float* act, const float* boot,
                                const float* ret, const float* eff, size_t n) {
  auto* r = static_cast<RefCritic*>(h);
  r->buffer->insert(make_batch(obs, act, boot, ret, eff, n, r->D, r->A));
}

REF_API void ref_vupdate_adopt_norm(void* h, int64_t count, const double* mean, const double* m2) {
  auto* r = static_cast<RefCritic*>(h);
  r->norm = make_stats(count, mean, m2, r->D);
}

REF_API int ref_vupdate_step(void* h, float* loss_out) {
  auto* r = static_cast<RefCritic*>(h);
  try {
    auto sampled = r->buffer->sample(r->B, r->sample_rng, r->B);
    if (!sampled) return 1;
    auto& batch = *sampled;
    batch.obs = fa::RunningNormalizer::apply_stats(r->norm, batch.obs);
    batch.boot_obs = fa::RunningNormalizer::apply_stats(r->norm, batch.boot_obs);
    agents::CriticLossResult<float> res;
    if (r->sac) {  // learners.cpp:168-176
      MatF eps(batch.size(), r->A);
      std::normal_distribution<float> gauss(0.0f, 1.0f);
      for (std::size_t k = 0; k < eps.size(); ++k) eps.data()[k] = gauss(r->eps_rng);
      res = agents::sac_critic_loss(batch, r->lagged_g, r->critics, std::exp(r->log_alpha), eps);
    } else if (r->distributional) {
      auto head = agents::CategoricalHead<float>::create(r->n_atoms, r->vmin, r->vmax);
      res = agents::c51_critic_loss(batch, r->lagged, r->critics, head);
    } else {
      res = agents::ddpg_critic_loss(batch, r->lagged, r->critics);
    }
    fa::clip_global_norm(res.dq1, 0.5f);
    fa::clip_global_norm(res.dq2, 0.5f);
    fa::adam_step(r->critics.q1.flat, res.dq1, r->adam_q1, r->lr);
    fa::adam_step(r->critics.q2.flat, res.dq2, r->adam_q2, r->lr);
    r->critics.soft_update_targets(r->tau);
    *loss_out = res.loss;
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API void ref_vupdate_set_log_alpha(void* h, float log_alpha) {
  static_cast<RefCritic*>(h)->log_alpha = log_alpha;
}

// which: 0 q1, 1 q2, 2 q1_target, 3 q2_target
REF_API void ref_vupdate_params(void* h, int which, float* out) {
  auto* r = static_cast<RefCritic*>(h);
  const auto& c = r->critics;
  const fa::Mlp<float>* nets[4] = {&c.q1, &c.q2, &c.q1_target, &c.q2_target};
  std::memcpy(out, nets[which]->flat.data(), nets[which]->flat.size() * sizeof(float));
}

// ----------------------------------------------- P-learner update (agents)
struct RefPolicy {
  size_t D, A, n_layers, B;
  std::vector<size_t> qsizes, psizes;
  float low = -1.0f, high = 1.0f, lr = 5e-4f;
  int distributional = 0;
  size_t n_atoms = 51;
  float vmin = -10.0f, vmax = 10.0f;
  agents::DeterministicPolicy<float> policy;
  int sac = 0;
  agents::GaussianPolicy<float> policy_g;
  agents::EntropyCoef<float> alpha;
  std::vector<float> alpha_param;
  fa::AdamState<float> adam_alpha;
  std::mt19937_64 eps_rng;
  fa::AdamState<float> adam;
  agents::CriticPair<float> critics;
  fa::NormStats norm;
  std::unique_ptr<replay::StateBuffer> states;
  std::mt19937_64 sample_rng;
};

REF_API void* ref_pupdate_create(size_t D, size_t A, size_t hidden, size_t n_hidden, size_t B,
                                 size_t capacity, uint64_t seed, const float* policy,
                                 const float* q1, const float* q2, int distributional,
                                 size_t n_atoms, float vmin, float vmax) {
  auto* r = new RefPolicy();
  r->D = D; r->A = A; r->B = B; r->n_layers = n_hidden + 1;
  r->sac = distributional == 2;  // algo: 0 ddpg, 1 c51, 2 sac
  if (r->sac) distributional = 0;
  r->distributional = distributional; r->n_atoms = n_atoms; r->vmin = vmin; r->vmax = vmax;
  r->qsizes.push_back(D + A);
  r->psizes.push_back(D);
  for (size_t i = 0; i < n_hidden; ++i) {
    r->qsizes.push_back(hidden);
    r->psizes.push_back(hidden);
  }
  r->qsizes.push_back(distributional ? n_atoms : 1);
  r->psizes.push_back(r->sac ? 2 * A : A);
  if (r->sac) {  // learners.cpp:213-219
    r->policy_g.net = make_mlp(r->psizes.data(), r->n_layers, policy);
    r->adam = fa::AdamState<float>(r->policy_g.net.param_count());
    r->alpha.target_entropy = -float(A);
    r->alpha_param.assign(1, 0.0f);
    r->adam_alpha = fa::AdamState<float>(1);
    r->eps_rng = make_rng(seed, RngStream::sac, 2);
  } else {
    r->policy = make_policy(policy, r->psizes.data(), r->n_layers, -1.0f, 1.0f);
    r->adam = fa::AdamState<float>(r->policy.net.param_count());
  }
  r->critics = make_pair(q1, q2, nullptr, nullptr, r->qsizes.data(), r->n_layers);
  r->states = std::make_unique<replay::StateBuffer>(capacity, D);
  r->sample_rng = make_rng(seed, RngStream::sample, 2);
  return r;
}

REF_API void ref_pupdate_destroy(void* h) { delete static_cast<RefPolicy*>(h); }

REF_API void ref_pupdate_insert(void* h, const float* rows, size_t n) {
  auto* r = static_cast<RefPolicy*>(h);
  r->states->insert(make_mat(rows, n, r->D));
}

REF_API void ref_pupdate_adopt_norm(void* h, int64_t count, const double* mean, const double* m2) {
  auto* r = static_cast<RefPolicy*>(h);
  r->norm = make_stats(count, mean, m2, r->D);
}

REF_API int ref_pupdate_step(void* h, float* loss_out) {
  auto* r = static_cast<RefPolicy*>(h);
  try {
    auto sampled = r->states->sample(r->B, r->sample_rng, r->B);
    if (!sampled) return 1;
    MatF states = fa::RunningNormalizer::apply_stats(r->norm, *sampled);
    float loss;
    std::vector<float> dpolicy;
    if (r->sac) {  // learners.cpp:246-258
      MatF eps(states.rows(), r->A);
      std::normal_distribution<float> gauss(0.0f, 1.0f);
      for (std::size_t k = 0; k < eps.size(); ++k) eps.data()[k] = gauss(r->eps_rng);
      r->alpha.log_alpha = r->alpha_param[0];
      auto res = agents::sac_actor_loss(states, r->policy_g, r->critics, r->alpha.alpha(), eps);
      loss = res.loss;
      dpolicy = std::move(res.dpolicy);
      auto ares = agents::sac_alpha_loss(res.mean_logp, r->alpha);
      std::vector<float> dalpha{ares.dlog_alpha};
      fa::adam_step(r->alpha_param, dalpha, r->adam_alpha, r->lr);
      fa::clip_global_norm(dpolicy, 0.5f);
      fa::adam_step(r->policy_g.net.flat, dpolicy, r->adam, r->lr);
      *loss_out = loss;
      return 0;
    }
    if (r->distributional) {
      auto head = agents::CategoricalHead<float>::create(r->n_atoms, r->vmin, r->vmax);
      auto res = agents::c51_actor_loss(states, r->policy, r->critics, head);
      loss = res.loss;
      dpolicy = std::move(res.dpolicy);
    } else {
      auto res = agents::ddpg_actor_loss(states, r->policy, r->critics);
      loss = res.loss;
      dpolicy = std::move(res.dpolicy);
    }
    fa::clip_global_norm(dpolicy, 0.5f);
    fa::adam_step(r->policy.net.flat, dpolicy, r->adam, r->lr);
    *loss_out = loss;
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API void ref_pupdate_params(void* h, float* out) {
  auto* r = static_cast<RefPolicy*>(h);
  const auto& net = r->sac ? r->policy_g.net : r->policy.net;
  std::memcpy(out, net.flat.data(), net.flat.size() * sizeof(float));
}

REF_API float ref_pupdate_log_alpha(void* h) {
  auto* r = static_cast<RefPolicy*>(h);
  return r->sac ? r->alpha_param[0] : 0.0f;
}

// --------------------------------------------------- actor step (agents)
// ActorCore::rollout_step (learners.cpp:80-116) composed from the
// reference's normalizer / DeterministicPolicy / apply_noise, with the
// environment step supplied by the caller (the synthetic env lives in the
// restatement; EnvBatch's tasks have other dims).  Phase 1: raw obs ->
// noisy actions (+ normalizer update after acting is phase 2).
struct RefActor {
  size_t N, D, A, n_layers;
  std::vector<size_t> psizes;
  agents::DeterministicPolicy<float> policy;
  fa::RunningNormalizer normalizer;
  explore::NoiseSchedule schedule;
  std::vector<env::SplitMixEngine> noise_rng;
  int sac = 0;
  agents::GaussianPolicy<float> policy_g;
};

REF_API void* ref_actor_create(size_t N, size_t D, size_t A, size_t hidden, size_t n_hidden,
                               uint64_t seed, const float* policy, float smin, float smax) {
  auto* r = new RefActor();
  r->N = N; r->D = D; r->A = A; r->n_layers = n_hidden + 1;
  r->psizes.push_back(D);
  for (size_t i = 0; i < n_hidden; ++i) r->psizes.push_back(hidden);
  r->psizes.push_back(A);
  r->policy = make_policy(policy, r->psizes.data(), r->n_layers, -1.0f, 1.0f);
  r->normalizer = fa::RunningNormalizer(D);
  r->schedule = explore::build_schedule(smin, smax, N);
  r->noise_rng.resize(N);
  for (size_t i = 0; i < N; ++i) r->noise_rng[i].state = derive_seed(seed, RngStream::noise, i);
  return r;
}

// The stochastic (pql_sac) actor: GaussianPolicy with [mean | log_std] head.
REF_API void* ref_actor_create_sac(size_t N, size_t D, size_t A, size_t hidden, size_t n_hidden,
                                   uint64_t seed, const float* policy) {
  auto* r = static_cast<RefActor*>(ref_actor_create(N, D, A, hidden, n_hidden, seed, nullptr,
                                                    0.05f, 0.8f));
  r->sac = 1;
  std::vector<size_t> ps(r->psizes);
  ps.back() = 2 * A;
  r->policy_g.net = make_mlp(ps.data(), r->n_layers, policy);
  return r;
}

// n draws of one normal_distribution<float>(0, 1) over make_rng(seed, stream, index)
REF_API void ref_normals(uint64_t seed, uint64_t stream, uint64_t index, size_t n, float* out) {
  auto rng = make_rng(seed, static_cast<RngStream>(stream), index);
  std::normal_distribution<float> gauss(0.0f, 1.0f);
  for (size_t k = 0; k < n; ++k) out[k] = gauss(rng);
}

// GaussianPolicy::sample (policy.hpp:77-107) and its backward (:121-152)
// for one batch: act [B x A], logp [B], and dpolicy for (dact, dlogp).
REF_API int ref_gauss_sample(const float* pol, const size_t* psizes, size_t n_layers,
                             const float* obs, const float* eps, size_t B, const float* dact,
                             const float* dlogp, float* act, float* logp, float* dpolicy) {
  agents::GaussianPolicy<float> p;
  p.net = make_mlp(psizes, n_layers, pol);
  const size_t A = psizes[n_layers] / 2;
  try {
    auto s = p.sample(make_mat(obs, B, psizes[0]), make_mat(eps, B, A));
    std::memcpy(act, s.act.data(), B * A * sizeof(float));
    std::memcpy(logp, s.logp.data(), B * sizeof(float));
    if (dpolicy) {
      std::vector<float> g;
      p.backward(s, make_mat(dact, B, A), std::vector<float>(dlogp, dlogp + B), g);
      std::memcpy(dpolicy, g.data(), g.size() * sizeof(float));
    }
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

REF_API void ref_actor_destroy(void* h) { delete static_cast<RefActor*>(h); }

REF_API void ref_actor_act(void* h, const float* obs, float* actions) {
  auto* r = static_cast<RefActor*>(h);
  MatF o = make_mat(obs, r->N, r->D);
  MatF obs_norm = r->normalizer.apply(o);
  if (r->sac) {  // learners.cpp:87-94: a fresh normal_distribution per env
    MatF eps(r->N, r->A);
    for (std::size_t i = 0; i < r->N; ++i) {
      std::normal_distribution<float> gauss(0.0f, 1.0f);
      for (std::size_t d = 0; d < r->A; ++d) eps(i, d) = gauss(r->noise_rng[i]);
    }
    MatF a = r->policy_g.sample(obs_norm, eps).act;
    std::memcpy(actions, a.data(), r->N * r->A * sizeof(float));
    return;
  }
  MatF a = r->policy.act(obs_norm);
  explore::apply_noise(a, r->schedule, r->policy.low, r->policy.high, r->noise_rng);
  std::memcpy(actions, a.data(), r->N * r->A * sizeof(float));
}

REF_API void ref_actor_observe(void* h, const float* obs) {
  auto* r = static_cast<RefActor*>(h);
  r->normalizer.update(make_mat(obs, r->N, r->D));
}

REF_API void ref_actor_stats(void* h, int64_t* count, double* mean, double* m2) {
  auto* r = static_cast<RefActor*>(h);
  const auto& s = r->normalizer.stats();
  *count = s.count;
  std::memcpy(mean, s.mean.data(), r->D * sizeof(double));
  std::memcpy(m2, s.m2.data(), r->D * sizeof(double));
}

// --------------------------------------------------- CriticLearnerCore
// The reference's own runtime core (2 hidden layers of cfg.hidden), used for
// config 1 end to end: ingest (n-step + insert, learners.cpp:144-151) and
// update (learners.cpp:157-188).
struct RefVCore {
  RunConfig cfg;
  size_t D = 0, A = 0;
  std::unique_ptr<rt::CriticLearnerCore> core;
};

REF_API void* ref_vcore_create(size_t n_envs, size_t batch, size_t capacity, size_t hidden,
                               size_t D, size_t A, uint64_t seed, uint64_t init_seed,
                               float reward_scale, int distributional) {
  auto* r = new RefVCore();
  r->cfg.n_envs = n_envs;
  r->cfg.batch_size = batch;
  r->cfg.buffer_capacity = capacity;
  r->cfg.hidden = hidden;
  r->cfg.seed = seed;
  r->cfg.reward_scale = reward_scale;
  r->cfg.algo = distributional ? agents::Algo::pql_d : agents::Algo::pql_ddpg;
  r->D = D;
  r->A = A;
  rt::TaskDims dims{D, A, -1.0f, 1.0f};
  r->core = std::make_unique<rt::CriticLearnerCore>(r->cfg, dims, std::mt19937_64(init_seed));
  return r;
}

REF_API void ref_vcore_destroy(void* h) { delete static_cast<RefVCore*>(h); }

REF_API void ref_vcore_ingest(void* h, const float* obs, const float* act, const float* boot,
                              const float* rew, const uint8_t* term, const uint8_t* trunc) {
  auto* r = static_cast<RefVCore*>(h);
  const size_t N = r->cfg.n_envs;
  rt::StepSlice s;
  s.obs = make_mat(obs, N, r->D);
  s.act = make_mat(act, N, r->A);
  s.boot_obs = make_mat(boot, N, r->D);
  s.rew.assign(rew, rew + N);
  s.term.assign(term, term + N);
  s.trunc.assign(trunc, trunc + N);
  r->core->ingest(s);
}

REF_API int ref_vcore_ready(void* h, int64_t c_a) {
  return static_cast<RefVCore*>(h)->core->ready(c_a) ? 1 : 0;
}

REF_API size_t ref_vcore_buffer_size(void* h) {
  return static_cast<RefVCore*>(h)->core->buffer_size();
}

REF_API void ref_vcore_adopt_norm(void* h, int64_t count, const double* mean, const double* m2) {
  auto* r = static_cast<RefVCore*>(h);
  r->core->adopt_norm(make_stats(count, mean, m2, r->D));
}

REF_API void ref_vcore_adopt_policy(void* h, const float* flat, int64_t version) {
  auto* r = static_cast<RefVCore*>(h);
  rt::PolicySnapshot snap;
  snap.version = version;
  const size_t sizes[4] = {r->D, r->cfg.hidden, r->cfg.hidden, r->A};
  snap.net = make_mlp(sizes, 3, flat);
  r->core->adopt_policy(snap);
}

REF_API int ref_vcore_update(void* h, float* loss) {
  auto* r = static_cast<RefVCore*>(h);
  try {
    *loss = r->core->update();
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

// which: 0 q1, 1 q2, 2 q1_target, 3 q2_target
REF_API void ref_vcore_params(void* h, int which, float* out) {
  auto* r = static_cast<RefVCore*>(h);
  const auto& c = r->core->critics();
  const fa::Mlp<float>* nets[4] = {&c.q1, &c.q2, &c.q1_target, &c.q2_target};
  std::memcpy(out, nets[which]->flat.data(), nets[which]->flat.size() * sizeof(float));
}

// make_snapshot(version) (learners.cpp:190-196): the online nets
REF_API void ref_vcore_snapshot(void* h, int64_t version, float* q1, float* q2) {
  auto* r = static_cast<RefVCore*>(h);
  const rt::CriticSnapshot s = r->core->make_snapshot(version);
  std::memcpy(q1, s.q1.flat.data(), s.q1.flat.size() * sizeof(float));
  std::memcpy(q2, s.q2.flat.data(), s.q2.flat.size() * sizeof(float));
}

// --------------------------------------------------- PolicyLearnerCore
// The reference's own runtime core (learners.cpp:202-274): ingest (the
// StateBuffer insert), adopt_critics / adopt_norm, ready, update, snapshot.
struct RefPCore {
  RunConfig cfg;
  size_t D = 0, A = 0;
  std::unique_ptr<rt::PolicyLearnerCore> core;
};

REF_API void* ref_pcore_create(size_t batch, size_t capacity, size_t hidden, size_t D, size_t A,
                               uint64_t seed, uint64_t init_seed, int algo) {
  auto* r = new RefPCore();
  r->cfg.batch_size = batch;
  r->cfg.buffer_capacity = capacity;
  r->cfg.hidden = hidden;
  r->cfg.seed = seed;
  r->cfg.algo = algo == 1 ? agents::Algo::pql_d
                : algo == 2 ? agents::Algo::pql_sac
                            : agents::Algo::pql_ddpg;
  r->D = D;
  r->A = A;
  rt::TaskDims dims{D, A, -1.0f, 1.0f};
  r->core = std::make_unique<rt::PolicyLearnerCore>(r->cfg, dims, std::mt19937_64(init_seed));
  return r;
}

REF_API void ref_pcore_destroy(void* h) { delete static_cast<RefPCore*>(h); }

REF_API void ref_pcore_ingest(void* h, const float* states, size_t n) {
  auto* r = static_cast<RefPCore*>(h);
  r->core->ingest(make_mat(states, n, r->D));
}

REF_API int ref_pcore_ready(void* h, int64_t c_a) {
  return static_cast<RefPCore*>(h)->core->ready(c_a) ? 1 : 0;
}

REF_API size_t ref_pcore_buffer_size(void* h) {
  return static_cast<RefPCore*>(h)->core->buffer_size();
}

REF_API void ref_pcore_adopt_norm(void* h, int64_t count, const double* mean, const double* m2) {
  auto* r = static_cast<RefPCore*>(h);
  r->core->adopt_norm(make_stats(count, mean, m2, r->D));
}

REF_API void ref_pcore_adopt_critics(void* h, const float* q1, const float* q2, int64_t version) {
  auto* r = static_cast<RefPCore*>(h);
  const size_t L = agents::is_distributional(r->cfg.algo) ? r->cfg.n_atoms : 1;
  const size_t sizes[4] = {r->D + r->A, r->cfg.hidden, r->cfg.hidden, L};
  rt::CriticSnapshot snap;
  snap.version = version;
  snap.q1 = make_mlp(sizes, 3, q1);
  snap.q2 = make_mlp(sizes, 3, q2);
  r->core->adopt_critics(snap);
}

REF_API int ref_pcore_update(void* h, float* loss) {
  auto* r = static_cast<RefPCore*>(h);
  try {
    *loss = r->core->update();
  } catch (const std::exception&) {
    return -2;
  }
  return 0;
}

// make_snapshot(version) (learners.cpp:272-274): the policy net + log_alpha
REF_API size_t ref_pcore_snapshot(void* h, int64_t version, float* flat, float* log_alpha) {
  auto* r = static_cast<RefPCore*>(h);
  const rt::PolicySnapshot s = r->core->make_snapshot(version);
  if (flat) std::memcpy(flat, s.net.flat.data(), s.net.flat.size() * sizeof(float));
  if (log_alpha) *log_alpha = s.log_alpha;
  return s.net.flat.size();
}

REF_API void ref_policy_init(size_t D, size_t A, size_t hidden, uint64_t seed, float* out) {
  RunConfig cfg;
  cfg.hidden = hidden;
  cfg.seed = seed;
  rt::TaskDims dims{D, A, -1.0f, 1.0f};
  auto rng = make_rng(seed, RngStream::init, 0);
  auto p = rt::PolicyHandle::create(cfg, dims, rng);
  std::memcpy(out, p.net().flat.data(), p.net().flat.size() * sizeof(float));
}

// ------------------------------------------------------------ checkpoints
// fa::save_checkpoint / load_checkpoint (src/funcapprox/checkpoint.cpp):
// nets given as (name, n_layers, sizes[n_layers + 1], flat) with ReLU hidden
// layers and an identity output layer (the Mlp shapes of learners.cpp).
REF_API int ref_checkpoint_save(const char* path, int n_nets, const char* const* names,
                                const size_t* n_layers, const size_t* const* sizes,
                                const float* const* flats, int64_t count, const double* mean,
                                const double* m2, size_t dim) {
  try {
    fa::Checkpoint c;
    for (int k = 0; k < n_nets; ++k)
      c.nets.emplace_back(names[k], make_mlp(sizes[k], n_layers[k], flats[k]));
    c.norm = make_stats(count, mean, m2, dim);
    fa::save_checkpoint(path, c);
    return 0;
  } catch (...) {
    return -1;
  }
}

// Parameters of every net concatenated in file order; returns the net count
// (or -1); *n_params / *dim report sizes when the output pointers are null.
REF_API int ref_checkpoint_load(const char* path, float* flat_out, size_t* n_params,
                                int64_t* count, double* mean, double* m2, size_t* dim) {
  try {
    const fa::Checkpoint c = fa::load_checkpoint(path);
    size_t total = 0;
    for (const auto& [name, net] : c.nets) {
      if (flat_out) std::memcpy(flat_out + total, net.flat.data(), net.flat.size() * 4);
      total += net.flat.size();
    }
    *n_params = total;
    *dim = c.norm.dim();
    *count = c.norm.count;
    if (mean) std::memcpy(mean, c.norm.mean.data(), c.norm.dim() * 8);
    if (m2) std::memcpy(m2, c.norm.m2.data(), c.norm.dim() * 8);
    return static_cast<int>(c.nets.size());
  } catch (...) {
    return -1;
  }
}

// ------------------------------------------------------------ metrics CSV
// rt::MetricsWriter (metrics.cpp:8-29): rows given as 9 doubles each in the
// MetricsRow field order (the integer fields rounded).
REF_API int ref_metrics_write(const char* path, const double* rows, size_t n) {
  try {
    rt::MetricsWriter w(path);
    for (size_t i = 0; i < n; ++i) {
      const double* r = rows + 9 * i;
      rt::MetricsRow m;
      m.wall_clock_s = r[0];
      m.env_steps = static_cast<std::int64_t>(r[1]);
      m.c_a = static_cast<std::int64_t>(r[2]);
      m.c_v = static_cast<std::int64_t>(r[3]);
      m.c_p = static_cast<std::int64_t>(r[4]);
      m.eval_return_mean = r[5];
      m.eval_return_stderr = r[6];
      m.critic_loss_ema = r[7];
      m.actor_loss_ema = r[8];
      w.append(m);
    }
  } catch (...) {
    return -1;
  }
  return 0;
}

// ================================================ the synthetic task
// SyntheticEnv is an EnvBatch subclass built through the reference's
// protected constructor and its three virtuals (vecenv.hpp:62-69), so the
// reference's own EnvBatch::reset_all / step (vecenv.cpp:73-106: non-finite
// check, episode counter, time limit, terminal observation, auto-reset,
// truncation flags) and its per-env SplitMix streams (derive_seed(seed, env,
// i), vecenv.cpp:66) run on the synthetic dynamics:
//   s' = clamp(0.95 s + 0.05 (M clamp(a, lo, hi)), +-10)     d-ascending sums
//   reward = -(sum s'^2 / D + 0.01 sum a^2 / A)              float mul/add only
//   terminal when |s'_0| > 9; reset draws s ~ U(-1, 1) on the 53-bit path
//   M[d][k] = 2 u - 1, u = (splitmix64(derive_seed(seed, env, 2^40) + d A + k) >> 11) 2^-53
// `make_env` is the link seam: vecenv.cpp is compiled with
// -Dmake_env=pql_ref_make_env_builtin (oracle/Makefile), and the definition
// below returns a SyntheticEnv while g_synth.on is set (so the reference's
// ActorCore constructor and evaluate_policy build it), else the builtin task.
namespace pql::env {
std::unique_ptr<EnvBatch> pql_ref_make_env_builtin(TaskId task, std::size_t n_envs,
                                                   std::uint64_t seed);
}

namespace {

struct SynthSpec {
  bool on = false;
  size_t D = 0, A = 0, max_len = 1000;
  float low = -1.0f, high = 1.0f;
};
SynthSpec g_synth;

// vecenv.cpp:19-23 (file-local there): the reset draw on the 53-bit path
float synth_uniform(env::SplitMixEngine& rng, float lo, float hi) {
  const double u = static_cast<double>(rng() >> 11) * 0x1.0p-53;
  return static_cast<float>(lo + (hi - lo) * u);
}

class SyntheticEnv final : public env::EnvBatch {
 public:
  SyntheticEnv(size_t n, uint64_t seed, const SynthSpec& sp)
      : EnvBatch(env::TaskId::pendulum /* tag only */, n, seed, sp.D, sp.A, sp.low, sp.high,
                 sp.max_len, 1.0f),
        s_(n * sp.D, 0.0f),
        M_(sp.D * sp.A) {
    const uint64_t mseed = derive_seed(seed, RngStream::env, 1ull << 40);
    for (size_t d = 0; d < sp.D; ++d)
      for (size_t k = 0; k < sp.A; ++k) {
        const uint64_t u = splitmix64(mseed + d * sp.A + k);
        M_[d * sp.A + k] = static_cast<float>(static_cast<double>(u >> 11) * 0x1.0p-53 * 2.0 - 1.0);
      }
  }
  // staggered time limits, episode_step = i mod max_len
  void stagger() {
    for (size_t i = 0; i < n_envs_; ++i)
      episode_step_[i] = static_cast<int64_t>(i % max_episode_len_);
  }

 private:
  void reset_row(size_t i) override {
    for (size_t d = 0; d < obs_dim_; ++d) s_[i * obs_dim_ + d] = synth_uniform(rng(i), -1.0f, 1.0f);
  }
  bool step_row(size_t i, const float* action, float& reward) override {
    const size_t D = obs_dim_, A = act_dim_;
    float a[256];
    float aa = 0.0f;
    for (size_t k = 0; k < A; ++k) {
      float u = action[k];
      u = u < action_low_ ? action_low_ : (u > action_high_ ? action_high_ : u);
      a[k] = u;
      aa = aa + u * u;
    }
    float* s = s_.data() + i * D;
    float ss = 0.0f;
    for (size_t d = 0; d < D; ++d) {
      float ma = 0.0f;
      for (size_t k = 0; k < A; ++k) ma = ma + M_[d * A + k] * a[k];
      float v = 0.95f * s[d] + 0.05f * ma;
      v = v < -10.0f ? -10.0f : (v > 10.0f ? 10.0f : v);
      s[d] = v;
      ss = ss + v * v;
    }
    reward = -(ss / static_cast<float>(D) + 0.01f * (aa / static_cast<float>(A)));
    return std::fabs(s[0]) > 9.0f;
  }
  void observe_row(size_t i, float* obs) const override {
    std::memcpy(obs, s_.data() + i * obs_dim_, obs_dim_ * sizeof(float));
  }

  std::vector<float> s_, M_;
};

}  // namespace

namespace pql::env {
std::unique_ptr<EnvBatch> make_env(TaskId task, std::size_t n_envs, std::uint64_t seed) {
  if (g_synth.on) {
    if (n_envs == 0) throw std::invalid_argument("make_env: n_envs must be >= 1");
    return std::make_unique<SyntheticEnv>(n_envs, seed, g_synth);
  }
  return pql_ref_make_env_builtin(task, n_envs, seed);
}
}  // namespace pql::env

namespace {
std::unique_ptr<env::EnvBatch> make_synth(size_t n, size_t D, size_t A, uint64_t seed,
                                          size_t max_len, float low, float high) {
  g_synth = SynthSpec{true, D, A, max_len, low, high};
  auto e = env::make_env(env::TaskId::pendulum, n, seed);
  g_synth.on = false;
  return e;
}
}  // namespace

// The synthetic EnvBatch on its own: make_env + reset_all (+ stagger);
// writes the initial observations.
REF_API void* ref_synth_env_create(size_t n, size_t D, size_t A, uint64_t seed, size_t max_len,
                                   float low, float high, int stagger, float* obs0) {
  auto e = make_synth(n, D, A, seed, max_len, low, high);
  MatF o = e->reset_all();
  if (stagger) static_cast<SyntheticEnv&>(*e).stagger();
  if (obs0) std::memcpy(obs0, o.data(), n * D * sizeof(float));
  return e.release();
}

REF_API void ref_synth_env_destroy(void* h) { delete static_cast<env::EnvBatch*>(h); }

// EnvBatch::step (vecenv.cpp:84-106); -2 on the non-finite-action throw
REF_API int ref_synth_env_step(void* h, const float* act, float* next_obs, float* terminal_obs,
                               float* rew, uint8_t* dones, uint8_t* trunc) {
  auto* e = static_cast<env::EnvBatch*>(h);
  const size_t N = e->n_envs(), D = e->obs_dim();
  try {
    const auto& r = e->step(make_mat(act, N, e->act_dim()));
    std::memcpy(next_obs, r.next_observations.data(), N * D * sizeof(float));
    // rows without a done keep whatever the buffer held (valid iff dones[i])
    for (size_t i = 0; i < N; ++i)
      if (r.dones[i]) std::memcpy(terminal_obs + i * D, r.terminal_observations.row(i), D * 4);
    std::memcpy(rew, r.rewards.data(), N * sizeof(float));
    std::memcpy(dones, r.dones.data(), N);
    std::memcpy(trunc, r.truncated.data(), N);
  } catch (const std::runtime_error&) {
    return -2;
  }
  return 0;
}

REF_API void ref_synth_env_episode_steps(void* h, int64_t* out) {
  auto* e = static_cast<env::EnvBatch*>(h);
  std::memcpy(out, e->episode_step().data(), e->n_envs() * sizeof(int64_t));
}

// ---------------------------------------- rt::ActorCore on the synthetic task
// The reference's own ActorCore (learners.cpp:62-116) -- constructor (env,
// reset_all, PolicyHandle::create with make_rng(seed, init, 0), noise
// schedule, per-env noise streams) and rollout_step -- with make_env
// returning the synthetic task.  Its policy is PolicyHandle::create's: two
// hidden layers of `hidden` (learners.cpp:22-23).
struct RefActorCore {
  RunConfig cfg;
  std::unique_ptr<rt::ActorCore> core;
  size_t N = 0, D = 0, A = 0;
};

REF_API void* ref_actor_core_create(size_t n_envs, size_t D, size_t A, size_t hidden,
                                    uint64_t seed, double sigma_min, double sigma_max,
                                    double sigma_fixed, size_t max_len, int sac) {
  auto* r = new RefActorCore();
  r->cfg.n_envs = n_envs;
  r->cfg.hidden = hidden;
  r->cfg.seed = seed;
  r->cfg.sigma_min = sigma_min;
  r->cfg.sigma_max = sigma_max;
  r->cfg.sigma_fixed = sigma_fixed;
  r->cfg.algo = sac ? agents::Algo::pql_sac : agents::Algo::pql_ddpg;
  r->N = n_envs;
  r->D = D;
  r->A = A;
  g_synth = SynthSpec{true, D, A, max_len, -1.0f, 1.0f};
  r->core = std::make_unique<rt::ActorCore>(r->cfg, rt::TaskDims{D, A, -1.0f, 1.0f});
  g_synth.on = false;
  static_cast<SyntheticEnv&>(r->core->envs()).stagger();
  return r;
}

REF_API void ref_actor_core_destroy(void* h) { delete static_cast<RefActorCore*>(h); }

// One rollout_step: the StepSlice (obs, act, boot_obs, rew, term, trunc).
REF_API int ref_actor_core_step(void* h, float* obs, float* act, float* boot, float* rew,
                                uint8_t* term, uint8_t* trunc) {
  auto* r = static_cast<RefActorCore*>(h);
  try {
    const rt::StepSlice s = r->core->rollout_step();
    if (obs) std::memcpy(obs, s.obs.data(), r->N * r->D * sizeof(float));
    if (act) std::memcpy(act, s.act.data(), r->N * r->A * sizeof(float));
    if (boot) std::memcpy(boot, s.boot_obs.data(), r->N * r->D * sizeof(float));
    if (rew) std::memcpy(rew, s.rew.data(), r->N * sizeof(float));
    if (term) std::memcpy(term, s.term.data(), r->N);
    if (trunc) std::memcpy(trunc, s.trunc.data(), r->N);
  } catch (const std::runtime_error&) {
    return -2;
  }
  return 0;
}

REF_API void ref_actor_core_norm(void* h, int64_t* count, double* mean, double* m2) {
  auto* r = static_cast<RefActorCore*>(h);
  const auto& s = r->core->norm();
  *count = s.count;
  std::memcpy(mean, s.mean.data(), r->D * sizeof(double));
  std::memcpy(m2, s.m2.data(), r->D * sizeof(double));
}

REF_API size_t ref_actor_core_policy(void* h, float* out) {
  auto* r = static_cast<RefActorCore*>(h);
  const auto& flat = r->core->policy().net().flat;
  if (out) std::memcpy(out, flat.data(), flat.size() * sizeof(float));
  return flat.size();
}

REF_API void ref_actor_core_episode_steps(void* h, int64_t* out) {
  auto* r = static_cast<RefActorCore*>(h);
  std::memcpy(out, r->core->envs().episode_step().data(), r->N * sizeof(int64_t));
}

// --------------------------------------- rt::evaluate_policy on the synthetic task
// learners.cpp:280-325 as written, with make_env returning the synthetic
// task (fresh episodes, no stagger).  The snapshot's net may have any depth.
REF_API int ref_evaluate_synth(const float* pol, const size_t* psizes, size_t n_layers, int sac,
                               int64_t count, const double* mean, const double* m2,
                               size_t episodes, uint64_t eval_seed, size_t max_len, float low,
                               float high, double* mean_out, double* stderr_out) {
  rt::PolicySnapshot snap;
  snap.net = make_mlp(psizes, n_layers, pol);
  snap.stochastic = sac != 0;
  const size_t D = psizes[0];
  const size_t A = sac ? psizes[n_layers] / 2 : psizes[n_layers];
  snap.norm = make_stats(count, mean, m2, D);
  g_synth = SynthSpec{true, D, A, max_len, low, high};
  try {
    const rt::EvalResult r = rt::evaluate_policy(snap, env::TaskId::pendulum, episodes, eval_seed);
    g_synth.on = false;
    *mean_out = r.mean;
    *stderr_out = r.stderr_mean;
  } catch (const std::invalid_argument&) {
    g_synth.on = false;
    return -1;
  } catch (const std::runtime_error&) {
    g_synth.on = false;
    return -2;
  }
  return 0;
}
