// run_parallel on one B200: the three
// PQL processes -- Actor, V-learner, P-learner -- as three host threads, each
// driving its core on its own CUDA stream, paced by counter gating and
// talking only through bounded channels and latest-wins snapshot slots.
//
//   reference                                   here
//   sched::RatioGate (ratio_gate.hpp:17-112)    Gate (same proceed rule, same counters)
//   rt::BoundedChannel (mailbox.hpp:13-63)      Channel<Batch>: host FIFO of descriptors of
//                                               device-resident data slots
//   rt::LatestSlot (mailbox.hpp:67-84)          SnapshotPool: 3 device buffers + events,
//                                               latest-wins, readers never block writers
//   DataBatch / StateBatch (messages.hpp:37-49) one DataSlot per actor iteration: H
//                                               StepSlices, the actor's normalizer, the
//                                               policy it used and the newest critic
//                                               snapshot (hub topology)
//
// All data stays on the device; the host threads only exchange slot indices,
// versions and CUDA events (cudaStreamWaitEvent orders the streams).
#include <algorithm>
#include <atomic>
#include <chrono>
#include <condition_variable>
#include <deque>
#include <cmath>
#include <map>
#include <memory>
#include <mutex>
#include <optional>
#include <string>
#include <thread>
#include <vector>

#include "actor.h"
#include "learner.h"
#include "metrics.h"

namespace pqlg {
namespace {

enum Proc { kActor = 0, kVLearner = 1, kPLearner = 2 };

// RatioGate::may_proceed (ratio_gate.hpp:44-60).
bool may_proceed(int p, int64_t ca, int64_t cv, int64_t cp, const pqlg_ratio_config& c) {
  if (c.free_running) return true;
  if (ca < c.warm_up) return true;
  switch (p) {
    case kActor:
      return static_cast<double>(ca) + 1.0 <= c.beta_av * static_cast<double>(cv) + c.slack_a;
    case kPLearner:
      return static_cast<double>(cp) + 1.0 <= c.beta_pv * static_cast<double>(cv) + c.slack_p;
    case kVLearner:  // must not outrun available data
      return static_cast<double>(cv) + 1.0 <= static_cast<double>(ca) / c.beta_av + c.slack_v;
  }
  return true;
}

class Gate {
 public:
  explicit Gate(const pqlg_ratio_config& c) : cfg_(c) {}
  int64_t count(int p) const { return c_[p].load(std::memory_order_relaxed); }
  bool may(int p) const { return may_proceed(p, count(0), count(1), count(2), cfg_); }
  // wait_turn_for: true = proceed; false = timed out or stopped
  bool wait_for(int p, std::chrono::microseconds t) {
    std::unique_lock<std::mutex> lk(mu_);
    return cv_.wait_for(lk, t, [&] { return stop_ || may(p); }) && !stop_;
  }
  void record(int p, int64_t n) {
    c_[p].fetch_add(n, std::memory_order_relaxed);
    std::lock_guard<std::mutex> lk(mu_);
    cv_.notify_all();
  }
  void shutdown() {
    std::lock_guard<std::mutex> lk(mu_);
    stop_ = true;
    cv_.notify_all();
  }
  bool stopped() {
    std::lock_guard<std::mutex> lk(mu_);
    return stop_;
  }

 private:
  pqlg_ratio_config cfg_;
  std::atomic<int64_t> c_[3]{{0}, {0}, {0}};
  std::mutex mu_;
  std::condition_variable cv_;
  bool stop_ = false;
};

struct Batch {
  int64_t seq;
  int slot;
  int64_t policy_version;
  int64_t critic_version;  // 0: no critic snapshot yet
};

// BoundedChannel (mailbox.hpp:13-63): push blocks while full; close wakes all.
class Channel {
 public:
  explicit Channel(size_t cap) : cap_(cap) {}
  bool push(const Batch& b) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_push_.wait(lk, [&] { return closed_ || q_.size() < cap_; });
    if (closed_) return false;
    q_.push_back(b);
    cv_pop_.notify_one();
    return true;
  }
  std::optional<Batch> pop_wait(std::chrono::microseconds t) {
    std::unique_lock<std::mutex> lk(mu_);
    cv_pop_.wait_for(lk, t, [&] { return closed_ || !q_.empty(); });
    if (q_.empty()) return std::nullopt;
    Batch b = q_.front();
    q_.pop_front();
    cv_push_.notify_one();
    return b;
  }
  void close() {
    std::lock_guard<std::mutex> lk(mu_);
    closed_ = true;
    cv_push_.notify_all();
    cv_pop_.notify_all();
  }

 private:
  size_t cap_;
  std::mutex mu_;
  std::condition_variable cv_push_, cv_pop_;
  std::deque<Batch> q_;
  bool closed_ = false;
};

// LatestSlot (mailbox.hpp:67-84) for device snapshots: the publisher writes
// buffer (latest + 1) % 3 after waiting (on its stream) for the last reader of
// that buffer; a reader copies the latest buffer under the lock and records
// its read event before releasing it, so no buffer is overwritten mid-read.
struct SnapshotPool {
  DevBuf<float> buf[3];
  cudaEvent_t written[3] = {}, read[3] = {};
  int64_t version = 0;
  int latest = -1;
  std::mutex mu;
  void init(size_t floats) {
    for (int k = 0; k < 3; ++k) {
      buf[k].alloc(floats);
      PQLG_CUDA(cudaEventCreateWithFlags(&written[k], cudaEventDisableTiming));
      PQLG_CUDA(cudaEventCreateWithFlags(&read[k], cudaEventDisableTiming));
    }
  }
  ~SnapshotPool() {
    for (int k = 0; k < 3; ++k) {
      if (written[k]) cudaEventDestroy(written[k]);
      if (read[k]) cudaEventDestroy(read[k]);
    }
  }
  // copy(dst_buffer, stream) enqueues the writes of the snapshot
  template <class F>
  int64_t publish(cudaStream_t st, F&& copy) {
    std::lock_guard<std::mutex> lk(mu);
    const int k = (latest + 1) % 3;
    PQLG_CUDA(cudaStreamWaitEvent(st, read[k], 0));
    copy(buf[k].p, st);
    PQLG_CUDA(cudaEventRecord(written[k], st));
    latest = k;
    return ++version;
  }
  // read(src_buffer, version, stream) enqueues the reads when newer than have
  template <class F>
  int64_t take_if_newer(int64_t have, cudaStream_t st, F&& read_fn) {
    std::lock_guard<std::mutex> lk(mu);
    if (latest < 0 || version <= have) return have;
    PQLG_CUDA(cudaStreamWaitEvent(st, written[latest], 0));
    read_fn(buf[latest].p, version, st);
    PQLG_CUDA(cudaEventRecord(read[latest], st));
    return version;
  }
  int64_t newest() {
    std::lock_guard<std::mutex> lk(mu);
    return version;
  }
};

}  // namespace

class Pipeline {
 public:
  Pipeline(const pqlg_config& cfg, const pqlg_task_dims& dims, const pqlg_ratio_config& rc,
           uint64_t init_seed)
      : cfg_(cfg), dims_(dims), rc_(rc), gate_(rc) {
    require(rc.horizon >= 1 && rc.channel_capacity >= 1 && rc.publish_every >= 1,
            "pipeline: horizon, channel_capacity and publish_every must be >= 1");
    require(rc.beta_av > 0 && rc.beta_pv > 0, "pipeline: ratios must be positive");
    PQLG_CUDA(cudaGetDevice(&device_));
    for (auto* s : {&sa_, &sv_, &sp_}) PQLG_CUDA(cudaStreamCreateWithFlags(s, cudaStreamNonBlocking));
    actor_ = std::make_unique<Actor>(cfg, dims, sa_);
    v_ = std::make_unique<VLearner>(cfg, dims, init_seed, sv_);
    p_ = std::make_unique<PLearner>(cfg, dims, init_seed, sp_);
    N_ = cfg.n_envs;
    D_ = dims.obs_dim;
    A_ = dims.act_dim;
    Dp_ = round_up(D_, 4);
    Ap_ = round_up(A_, 4);
    H_ = rc.horizon;
    const int64_t Pp = p_->snapshot_len(), Pq = p_->critic_params();  // [net | log_alpha]
    pol_pool_.init(Pp);
    crit_pool_.init(2 * Pq);
    // one slot per in-flight actor iteration: both channels full + one being
    // filled + one being consumed per learner
    const int n_slots = 2 * rc.channel_capacity + 3;
    slots_.resize(n_slots);
    for (int k = 0; k < n_slots; ++k) {
      Slot& s = slots_[k];
      s.obs.alloc(static_cast<size_t>(H_) * N_ * Dp_);
      s.boot.alloc(static_cast<size_t>(H_) * N_ * Dp_);
      s.act.alloc(static_cast<size_t>(H_) * N_ * Ap_);
      s.rew.alloc(static_cast<size_t>(H_) * N_);
      s.flags.alloc(2ull * H_ * N_);
      s.count.alloc(1);
      s.mean.alloc(D_);
      s.m2.alloc(D_);
      s.pol.alloc(Pp);
      s.crit.alloc(2 * Pq);
      PQLG_CUDA(cudaEventCreateWithFlags(&s.filled, cudaEventDisableTiming));
      PQLG_CUDA(cudaEventCreateWithFlags(&s.done_v, cudaEventDisableTiming));
      PQLG_CUDA(cudaEventCreateWithFlags(&s.done_p, cudaEventDisableTiming));
      free_.push_back(k);
    }
    PQLG_CUDA(cudaDeviceSynchronize());
  }

  ~Pipeline() {
    for (auto& s : slots_) {
      cudaEventDestroy(s.filled);
      cudaEventDestroy(s.done_v);
      cudaEventDestroy(s.done_p);
    }
    actor_.reset();
    v_.reset();
    p_.reset();
    for (auto s : {sa_, sv_, sp_}) {
      cudaStreamSynchronize(s);
      cudaStreamDestroy(s);
    }
  }

  // the evaluator + metrics writer
  void set_metrics(const pqlg_metrics_config& m) {
    require(!ran_, "pipeline: set_metrics before run()");
    if (!m.path) {
      writer_.reset();
      evaluator_.reset();
      return;
    }
    require(m.interval_s > 0.0 && m.eval_episodes >= 1 && m.ema >= 0.0 && m.ema < 1.0,
            "pipeline: metrics needs interval_s > 0, eval_episodes >= 1, 0 <= ema < 1");
    mcfg_ = m;
    closs_ema_.f = aloss_ema_.f = m.ema;
    writer_ = std::make_unique<MetricsWriter>(m.path);
    evaluator_ = std::make_unique<Evaluator>(cfg_, dims_, m.eval_episodes, m.eval_seed);
  }

  void record_snapshots(bool on) { record_snapshots_ = on; }

  // After run(): the P-learner's critic replicas against the snapshot the
  // V-learner published under the version the P-learner holds (version 0:
  // the replicas it was created with, compared with nothing: diff -1).
  void check_critics(int64_t* p_version, double* max_abs_diff) {
    require(ran_, "pipeline: check_critics after run()");
    require(record_snapshots_, "pipeline: check_critics needs record_snapshots before run()");
    const int64_t Pq = p_->critic_params();
    *p_version = p_->critic_version();
    *max_abs_diff = -1.0;
    std::lock_guard<std::mutex> lk(hist_mu_);
    auto it = crit_hist_.find(*p_version);
    if (it == crit_hist_.end()) return;
    std::vector<float> got(2 * Pq);
    p_->get_params(1, got.data());
    p_->get_params(2, got.data() + Pq);
    double mx = 0.0;
    for (int64_t i = 0; i < 2 * Pq; ++i)
      mx = std::max(mx, std::fabs(static_cast<double>(got[i]) - it->second[i]));
    *max_abs_diff = mx;
  }

  pqlg_run_report run(int64_t actor_steps, double max_seconds) {
    require(!ran_, "pipeline: run() may be called once per pipeline");
    ran_ = true;
    ch_v_ = std::make_unique<Channel>(rc_.channel_capacity);
    ch_p_ = std::make_unique<Channel>(rc_.channel_capacity);
    const auto t0 = std::chrono::steady_clock::now();
    std::thread ta([&] { guard_thread([&] { actor_loop(); }); });
    std::thread tv([&] { guard_thread([&] { vlearner_loop(); }); });
    std::thread tp([&] { guard_thread([&] { plearner_loop(); }); });
    t0_ = t0;
    std::thread te;
    if (writer_) te = std::thread([&] { guard_thread([&] { evaluator_loop(); }); });
    while (true) {
      std::this_thread::sleep_for(std::chrono::microseconds(200));
      const double el = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
      if (failed_.load() || gate_.count(kActor) >= actor_steps || el >= max_seconds) break;
    }
    // clean shutdown: the actor finishes its iteration (its pushes complete
    // while the learners keep draining), then the learners drain what is
    // queued and stop -- every batch sent is consumed exactly once
    stop_actor_ = true;
    {
      std::lock_guard<std::mutex> lk(ev_mu_);
      ev_stop_ = true;
      ev_cv_.notify_all();
    }
    ta.join();
    if (te.joinable()) te.join();
    stop_all();
    tv.join();
    tp.join();
    if (failed_.load()) {
      // a sticky device error would make a checked sync throw first and
      // replace the worker's error: drain the streams, ignoring errors
      for (auto s : {sa_, sv_, sp_}) (void)cudaStreamSynchronize(s);
      set_last_error(error_);
      throw Error(err_status_, error_);
    }
    for (auto s : {sa_, sv_, sp_}) PQLG_CUDA(cudaStreamSynchronize(s));
    if (writer_) {  // final metrics row (run_parallel returns final metrics)
      snapshot_for_eval();
      append_row();
    }
    pqlg_run_report r{};
    r.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.c_a = gate_.count(kActor);
    r.c_v = gate_.count(kVLearner);
    r.c_p = gate_.count(kPLearner);
    r.env_steps = r.c_a * N_;
    r.ratio_av = r.c_v ? static_cast<double>(r.c_a) / r.c_v : 0.0;
    r.ratio_pv = r.c_v ? static_cast<double>(r.c_p) / r.c_v : 0.0;
    r.batches_sent = sent_;
    r.batches_consumed_v = stats_[0].consumed;
    r.batches_consumed_p = stats_[1].consumed;
    r.seq_duplicates = stats_[0].dups + stats_[1].dups;
    r.seq_gaps = stats_[0].gaps + stats_[1].gaps;
    r.max_policy_staleness = max_stale_;
    r.policy_version = pol_pool_.newest();
    r.critic_version = crit_pool_.newest();
    r.last_critic_loss = last_closs_;
    r.last_actor_loss = last_aloss_;
    r.ok = 1;
    return r;
  }

 private:
  struct Slot {
    DevBuf<float> obs, boot, act, rew, pol, crit;
    DevBuf<uint8_t> flags;  // term [H x N] | trunc [H x N]
    DevBuf<int64_t> count;
    DevBuf<double> mean, m2;
    cudaEvent_t filled = nullptr, done_v = nullptr, done_p = nullptr;
    int pending = 0;  // consumers still to release it
  };
  bool record_snapshots_ = false;
  std::mutex hist_mu_;
  std::map<int64_t, std::vector<float>> crit_hist_;
  struct ConsumerStats {
    int64_t expect = 0, consumed = 0, dups = 0, gaps = 0;
  };

  template <class F>
  void guard_thread(F&& f) {
    try {
      PQLG_CUDA(cudaSetDevice(device_));  // the CUDA device is per host thread
      f();
    } catch (const Error& e) {
      fail(e.status, e.what());
    } catch (const std::exception& e) {
      fail(PQLG_EINVAL, e.what());
    }
  }
  void fail(int status, const std::string& msg) {
    {
      std::lock_guard<std::mutex> lk(err_mu_);
      if (!failed_.load()) {
        error_ = "run_parallel: " + msg;
        err_status_ = status;
      }
    }
    failed_ = true;
    stop_all();
  }
  void stop_all() {
    gate_.shutdown();
    if (ch_v_) ch_v_->close();
    if (ch_p_) ch_p_->close();
    std::lock_guard<std::mutex> lk(slot_mu_);
    stopping_ = true;
    slot_cv_.notify_all();
  }

  int take_slot() {
    std::unique_lock<std::mutex> lk(slot_mu_);
    slot_cv_.wait(lk, [&] { return stopping_ || !free_.empty(); });
    if (stopping_) return -1;
    const int k = free_.front();
    free_.pop_front();
    slots_[k].pending = 2;
    return k;
  }
  void release_slot(int k) {
    std::lock_guard<std::mutex> lk(slot_mu_);
    if (--slots_[k].pending == 0) {
      free_.push_back(k);
      slot_cv_.notify_all();
    }
  }

  // ---- Actor (Alg. 1, SPEC run_actor): fetch the newest policy, roll out H
  // steps, send (transitions, policy, normalizer) to the V-learner and
  // (states, critic snapshot, normalizer) to the P-learner, gate.
  void actor_loop() {
    int64_t seq = 0, crit_have = 0;
    const int64_t Pp = p_->snapshot_len(), Pq = p_->critic_params();  // [net | log_alpha]
    while (true) {
      bool go = false;
      while (!go) {
        if (gate_.stopped() || stop_actor_.load()) return;
        serve_eval();
        go = gate_.wait_for(kActor, std::chrono::microseconds(2000));
      }
      const int k = take_slot();
      if (k < 0) return;
      Slot& s = slots_[k];
      PQLG_CUDA(cudaStreamWaitEvent(sa_, s.done_v, 0));
      PQLG_CUDA(cudaStreamWaitEvent(sa_, s.done_p, 0));
      // newest policy snapshot (P-learner -> actor)
      pol_pool_.take_if_newer(actor_->policy_version(), sa_,
                              [&](const float* src, int64_t ver, cudaStream_t st) {
                                (void)st;
                                actor_->adopt_policy(src, ver, true);
                              });
      max_stale_ = std::max(max_stale_, pol_pool_.newest() - actor_->policy_version());
      for (int h = 0; h < H_; ++h) {
        pqlg_step_slice v{};
        actor_->rollout_step(&v);
        const size_t ro = static_cast<size_t>(h) * N_;
        auto cp2 = [&](float* dst, int64_t ldd, const float* src, int64_t lds, int w) {
          PQLG_CUDA(cudaMemcpy2DAsync(dst, ldd * 4, src, lds * 4, w * 4, N_,
                                      cudaMemcpyDeviceToDevice, sa_));
        };
        cp2(s.obs.p + ro * Dp_, Dp_, v.obs, v.ld_obs, D_);
        cp2(s.boot.p + ro * Dp_, Dp_, v.boot_obs, v.ld_obs, D_);
        cp2(s.act.p + ro * Ap_, Ap_, v.act, v.ld_act, A_);
        PQLG_CUDA(cudaMemcpyAsync(s.rew.p + ro, v.rew, N_ * 4, cudaMemcpyDeviceToDevice, sa_));
        PQLG_CUDA(cudaMemcpyAsync(s.flags.p + ro, v.term, N_, cudaMemcpyDeviceToDevice, sa_));
        PQLG_CUDA(cudaMemcpyAsync(s.flags.p + static_cast<size_t>(H_) * N_ + ro, v.trunc, N_,
                                  cudaMemcpyDeviceToDevice, sa_));
      }
      // normalizer (owned by the actor) and the policy the data came from
      PQLG_CUDA(cudaMemcpyAsync(s.count.p, actor_->count_dev(), 8, cudaMemcpyDeviceToDevice, sa_));
      PQLG_CUDA(cudaMemcpyAsync(s.mean.p, actor_->mean_dev(), D_ * 8, cudaMemcpyDeviceToDevice, sa_));
      PQLG_CUDA(cudaMemcpyAsync(s.m2.p, actor_->m2_dev(), D_ * 8, cudaMemcpyDeviceToDevice, sa_));
      PQLG_CUDA(cudaMemcpyAsync(s.pol.p, actor_->policy_dev(), Pp * 4, cudaMemcpyDeviceToDevice, sa_));
      // newest critic snapshot (V-learner -> actor -> P-learner).  Only a slot
      // that received a copy in this iteration carries a critic version: a
      // reused slot's s.crit holds an older snapshot (or nothing), which the
      // P-learner's equal-or-newer rule would otherwise adopt.
      bool fresh = false;
      crit_have = crit_pool_.take_if_newer(crit_have, sa_,
                                           [&](const float* src, int64_t, cudaStream_t st) {
                                             PQLG_CUDA(cudaMemcpyAsync(s.crit.p, src, 2 * Pq * 4,
                                                                       cudaMemcpyDeviceToDevice, st));
                                             fresh = true;
                                           });
      PQLG_CUDA(cudaEventRecord(s.filled, sa_));
      const Batch b{seq++, k, actor_->policy_version(), fresh ? crit_have : 0};
      if (!ch_v_->push(b) || !ch_p_->push(b)) return;
      ++sent_;
      gate_.record(kActor, H_);
    }
  }

  void note_seq(ConsumerStats& st, int64_t seq) {
    if (seq < st.expect) ++st.dups;
    else if (seq > st.expect) st.gaps += seq - st.expect;
    st.expect = std::max(st.expect, seq + 1);
    ++st.consumed;
  }

  // ---- V-learner (Alg. 3, SPEC run_vlearner): drain data into the replay
  // buffer, hard-update the lagged policy, update the critics, publish a
  // critic snapshot every K_pub updates, gate.
  void vlearner_loop() {
    ConsumerStats& st = stats_[0];
    int64_t updates = 0;
    const int64_t Pq = v_->critic_params();
    bool have_batch = false;  // replay size >= B (monotone: checked until true)
    auto ready = [&] {
      if (gate_.count(kActor) < cfg_.warm_up) return false;
      if (!have_batch) have_batch = v_->ready(gate_.count(kActor));
      return have_batch;
    };
    auto drain = [&](std::chrono::microseconds first_wait) {
      auto b = ch_v_->pop_wait(first_wait);
      while (b) {
        Slot& s = slots_[b->slot];
        note_seq(st, b->seq);
        PQLG_CUDA(cudaStreamWaitEvent(sv_, s.filled, 0));
        for (int h = 0; h < H_; ++h) {
          const size_t ro = static_cast<size_t>(h) * N_;
          replay::Slice sl{s.obs.p + ro * Dp_, s.act.p + ro * Ap_, s.boot.p + ro * Dp_,
                           s.rew.p + ro, s.flags.p + ro,
                           s.flags.p + static_cast<size_t>(H_) * N_ + ro, Dp_, Ap_};
          v_->ingest(sl);
        }
        v_->adopt_norm_device(s.count.p, s.mean.p, s.m2.p);
        v_->adopt_policy_device(s.pol.p, b->policy_version);
        PQLG_CUDA(cudaEventRecord(s.done_v, sv_));
        release_slot(b->slot);
        b = ch_v_->pop_wait(std::chrono::microseconds(0));
      }
    };
    while (!gate_.stopped()) {
      drain(std::chrono::microseconds(ready() ? 0 : 2000));
      if (!ready()) continue;
      if (!gate_.wait_for(kVLearner, std::chrono::microseconds(1000))) continue;
      v_->update_n(1);
      // the status word after every update: a non-finite update aborts the
      // run before it is counted or drives the gate (SPEC: abort)
      if (v_->check_status() != PQLG_OK)
        throw Error(PQLG_ENONFINITE, "critic update: non-finite target / loss / gradient");
      gate_.record(kVLearner, 1);
      if (++updates % rc_.publish_every == 0) {
        last_closs_ = v_->last_loss();  // throws on a non-finite update (SPEC: abort)
        {
          std::lock_guard<std::mutex> lk(ema_mu_);
          closs_ema_.add(last_closs_);
        }
        const int64_t ver = crit_pool_.publish(sv_, [&](float* dst, cudaStream_t stm) {
          PQLG_CUDA(cudaMemcpyAsync(dst, v_->critic_dev(0), Pq * 4, cudaMemcpyDeviceToDevice, stm));
          PQLG_CUDA(cudaMemcpyAsync(dst + Pq, v_->critic_dev(1), Pq * 4, cudaMemcpyDeviceToDevice,
                                    stm));
        });
        if (record_snapshots_) {  // test hook: host copy of every published snapshot
          std::vector<float> h(2 * Pq);
          PQLG_CUDA(cudaMemcpyAsync(h.data(), v_->critic_dev(0), Pq * 4, cudaMemcpyDeviceToHost, sv_));
          PQLG_CUDA(cudaMemcpyAsync(h.data() + Pq, v_->critic_dev(1), Pq * 4,
                                    cudaMemcpyDeviceToHost, sv_));
          PQLG_CUDA(cudaStreamSynchronize(sv_));
          std::lock_guard<std::mutex> lk(hist_mu_);
          crit_hist_[ver] = std::move(h);
        }
      }
    }
    drain(std::chrono::microseconds(0));  // closed channel: already-queued batches still drain
  }

  // ---- P-learner (Alg. 2, SPEC run_plearner)
  void plearner_loop() {
    ConsumerStats& st = stats_[1];
    int64_t updates = 0;
    const int64_t Pq = p_->critic_params(), Pp = p_->snapshot_len();
    bool have_batch = false;
    auto ready = [&] {
      if (gate_.count(kActor) < cfg_.warm_up) return false;
      if (!have_batch) have_batch = p_->ready(gate_.count(kActor));
      return have_batch;
    };
    auto drain = [&](std::chrono::microseconds first_wait) {
      auto b = ch_p_->pop_wait(first_wait);
      while (b) {
        Slot& s = slots_[b->slot];
        note_seq(st, b->seq);
        PQLG_CUDA(cudaStreamWaitEvent(sp_, s.filled, 0));
        p_->ingest(s.obs.p, Dp_, static_cast<uint64_t>(H_) * N_);
        p_->adopt_norm_device(s.count.p, s.mean.p, s.m2.p);
        if (b->critic_version > 0)
          p_->adopt_critics_device(s.crit.p, s.crit.p + Pq, b->critic_version);
        PQLG_CUDA(cudaEventRecord(s.done_p, sp_));
        release_slot(b->slot);
        b = ch_p_->pop_wait(std::chrono::microseconds(0));
      }
    };
    while (!gate_.stopped()) {
      drain(std::chrono::microseconds(ready() ? 0 : 2000));
      if (!ready()) continue;
      if (!gate_.wait_for(kPLearner, std::chrono::microseconds(1000))) continue;
      p_->update_n(1);
      if (p_->check_status() != PQLG_OK)
        throw Error(PQLG_ENONFINITE, "actor update: non-finite loss / gradient");
      gate_.record(kPLearner, 1);
      if (++updates % rc_.publish_every == 0) {
        last_aloss_ = p_->last_loss();
        {
          std::lock_guard<std::mutex> lk(ema_mu_);
          aloss_ema_.add(last_aloss_);
        }
        pol_pool_.publish(sp_, [&](float* dst, cudaStream_t stm) {
          PQLG_CUDA(cudaMemcpyAsync(dst, p_->policy_dev(), Pp * 4, cudaMemcpyDeviceToDevice, stm));
        });
      }
    }
    drain(std::chrono::microseconds(0));
  }

  // The actor thread copies its policy + normalizer to the host on request,
  // between rollouts (stream order makes the snapshot consistent).
  void serve_eval() {
    if (!ev_req_.load()) return;
    snapshot_for_eval();
    std::lock_guard<std::mutex> lk(ev_mu_);
    ev_req_ = false;
    ev_ready_ = true;
    ev_cv_.notify_all();
  }
  void snapshot_for_eval() {
    ev_pol_.resize(static_cast<size_t>(actor_->param_count()));
    ev_mean_.resize(D_);
    ev_m2_.resize(D_);
    PQLG_CUDA(cudaMemcpyAsync(ev_pol_.data(), actor_->policy_dev(), ev_pol_.size() * 4,
                              cudaMemcpyDeviceToHost, sa_));
    PQLG_CUDA(cudaMemcpyAsync(&ev_count_, actor_->count_dev(), 8, cudaMemcpyDeviceToHost, sa_));
    PQLG_CUDA(cudaMemcpyAsync(ev_mean_.data(), actor_->mean_dev(), D_ * 8, cudaMemcpyDeviceToHost, sa_));
    PQLG_CUDA(cudaMemcpyAsync(ev_m2_.data(), actor_->m2_dev(), D_ * 8, cudaMemcpyDeviceToHost, sa_));
    PQLG_CUDA(cudaStreamSynchronize(sa_));
  }
  void append_row() {
    double mu = 0.0, se = 0.0;
    evaluator_->run(ev_pol_.data(), ev_count_, ev_mean_.data(), ev_m2_.data(), nullptr, &mu, &se);
    pqlg_metrics_row r{};
    r.wall_clock_s =
        std::chrono::duration<double>(std::chrono::steady_clock::now() - t0_).count();
    r.c_a = gate_.count(kActor);
    r.c_v = gate_.count(kVLearner);
    r.c_p = gate_.count(kPLearner);
    r.env_steps = r.c_a * N_;
    r.eval_return_mean = mu;
    r.eval_return_stderr = se;
    {
      std::lock_guard<std::mutex> lk(ema_mu_);
      r.critic_loss_ema = closs_ema_.v;
      r.actor_loss_ema = aloss_ema_.v;
    }
    writer_->append(r);
    ++rows_;
  }
  // every interval_s: ask the actor for a snapshot, evaluate it, append a row
  void evaluator_loop() {
    auto next = t0_ + std::chrono::duration_cast<std::chrono::steady_clock::duration>(
                          std::chrono::duration<double>(mcfg_.interval_s));
    while (true) {
      std::unique_lock<std::mutex> lk(ev_mu_);
      if (ev_cv_.wait_until(lk, next, [&] { return ev_stop_; })) return;
      ev_req_ = true;
      ev_ready_ = false;
      ev_cv_.wait(lk, [&] { return ev_ready_ || ev_stop_; });
      if (!ev_ready_) return;
      lk.unlock();
      append_row();
      next += std::chrono::duration_cast<std::chrono::steady_clock::duration>(
          std::chrono::duration<double>(mcfg_.interval_s));
    }
  }

  pqlg_config cfg_;
  pqlg_task_dims dims_;
  pqlg_ratio_config rc_;
  Gate gate_;
  int device_ = 0;
  cudaStream_t sa_ = nullptr, sv_ = nullptr, sp_ = nullptr;
  std::unique_ptr<Actor> actor_;
  std::unique_ptr<VLearner> v_;
  std::unique_ptr<PLearner> p_;
  int N_, D_, A_, H_;
  int64_t Dp_, Ap_;
  SnapshotPool pol_pool_, crit_pool_;
  std::vector<Slot> slots_;
  std::deque<int> free_;
  std::mutex slot_mu_;
  std::condition_variable slot_cv_;
  bool stopping_ = false;
  std::unique_ptr<Channel> ch_v_, ch_p_;
  ConsumerStats stats_[2];
  int64_t sent_ = 0, max_stale_ = 0;
  float last_closs_ = 0.0f, last_aloss_ = 0.0f;
  bool ran_ = false;
  std::atomic<bool> failed_{false}, stop_actor_{false};
  // metrics / evaluator
  pqlg_metrics_config mcfg_{};
  std::unique_ptr<MetricsWriter> writer_;
  std::unique_ptr<Evaluator> evaluator_;  // allocated once at set_metrics
  std::mutex ema_mu_;
  Ema closs_ema_, aloss_ema_;
  std::chrono::steady_clock::time_point t0_;
  std::mutex ev_mu_;
  std::condition_variable ev_cv_;
  std::atomic<bool> ev_req_{false};
  bool ev_ready_ = false, ev_stop_ = false;
  std::vector<float> ev_pol_;
  int64_t ev_count_ = 0;
  std::vector<double> ev_mean_, ev_m2_;
  int64_t rows_ = 0;
  std::mutex err_mu_;
  std::string error_;
  int err_status_ = PQLG_OK;
};

// run_synchronous: the same cores, one stream, one host
// thread, Algorithm order.  Deterministic: every update replays the same
// graphs on the same stream with Philox streams, so two runs with one seed
// produce identical parameters, losses and metrics (wall clock aside).
pqlg_run_report run_synchronous(const pqlg_config& cfg, const pqlg_task_dims& dims,
                                const pqlg_ratio_config& rc, uint64_t init_seed,
                                int64_t actor_steps, const pqlg_metrics_config* mc) {
  require(rc.horizon >= 1 && rc.publish_every >= 1, "run_synchronous: horizon, publish_every >= 1");
  require(rc.beta_av > 0 && rc.beta_pv > 0, "run_synchronous: ratios must be positive");
  std::unique_ptr<MetricsWriter> writer;
  Ema closs, aloss;
  if (mc && mc->path) {
    require(mc->every_actor_steps >= 1 && mc->eval_episodes >= 1 && mc->ema >= 0.0 && mc->ema < 1.0,
            "run_synchronous: metrics needs every_actor_steps >= 1, eval_episodes >= 1, 0 <= ema < 1");
    closs.f = aloss.f = mc->ema;
    writer = std::make_unique<MetricsWriter>(mc->path);
  }
  std::unique_ptr<Evaluator> evaluator;
  if (writer) evaluator = std::make_unique<Evaluator>(cfg, dims, mc->eval_episodes, mc->eval_seed);
  cudaStream_t st;
  PQLG_CUDA(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
  struct StreamGuard {
    cudaStream_t s;
    ~StreamGuard() { cudaStreamSynchronize(s); cudaStreamDestroy(s); }
  } guard{st};
  Actor actor(cfg, dims, st);
  VLearner v(cfg, dims, init_seed, st);
  PLearner p(cfg, dims, init_seed, st);
  const int N = cfg.n_envs, D = dims.obs_dim, H = rc.horizon;
  const int64_t Pq = v.critic_params(), Pp = p.snapshot_len();
  (void)Pq;
  const auto t0 = std::chrono::steady_clock::now();
  int64_t ca = 0, cv = 0, cp = 0, pol_ver = 0, crit_ver = 0, next_eval = 0;
  float last_c = 0.0f, last_a = 0.0f;
  std::vector<float> pol(static_cast<size_t>(actor.param_count()));
  std::vector<double> mean(D), m2(D);
  auto row = [&] {
    int64_t count = 0;
    PQLG_CUDA(cudaMemcpyAsync(pol.data(), actor.policy_dev(), pol.size() * 4,
                              cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaMemcpyAsync(&count, actor.count_dev(), 8, cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaMemcpyAsync(mean.data(), actor.mean_dev(), D * 8, cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaMemcpyAsync(m2.data(), actor.m2_dev(), D * 8, cudaMemcpyDeviceToHost, st));
    PQLG_CUDA(cudaStreamSynchronize(st));
    double mu = 0.0, se = 0.0;
    evaluator->run(pol.data(), count, mean.data(), m2.data(), nullptr, &mu, &se);
    pqlg_metrics_row r{};
    r.wall_clock_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    r.env_steps = ca * N;
    r.c_a = ca;
    r.c_v = cv;
    r.c_p = cp;
    r.eval_return_mean = mu;
    r.eval_return_stderr = se;
    r.critic_loss_ema = closs.v;
    r.actor_loss_ema = aloss.v;
    writer->append(r);
  };
  if (writer) next_eval = mc->every_actor_steps;
  const int64_t n_v = static_cast<int64_t>(std::llround(H / rc.beta_av));
  require(n_v >= 1, "run_synchronous: horizon / beta_av rounds to zero critic updates per "
                    "iteration (beta_av must be <= 2 * horizon)");
  while (ca < actor_steps) {
    // Alg. 1: roll out H steps, send the transitions / states to the learners
    for (int h = 0; h < H; ++h) {
      pqlg_step_slice sl{};
      actor.rollout_step(&sl);
      v.ingest(replay::Slice{sl.obs, sl.act, sl.boot_obs, sl.rew, sl.term, sl.trunc, sl.ld_obs,
                             sl.ld_act});
      p.ingest(sl.obs, sl.ld_obs, static_cast<uint64_t>(N));
    }
    ca += H;
    // the actor's normalizer travels with the data
    v.adopt_norm_device(actor.count_dev(), actor.mean_dev(), actor.m2_dev());
    p.adopt_norm_device(actor.count_dev(), actor.mean_dev(), actor.m2_dev());
    if (ca >= rc.warm_up && v.ready(ca) && p.ready(ca)) {
      // Alg. 3 / 2: H / beta_av critic updates, policy updates interleaved so
      // that c_p stays at beta_pv * c_v
      for (int64_t k = 0; k < n_v; ++k) {
        v.update_n(1);
        ++cv;
        if (cv % rc.publish_every == 0) {  // critic snapshot -> P-learner
          last_c = v.last_loss();
          closs.add(last_c);
          p.adopt_critics_device(v.critic_dev(0), v.critic_dev(1), ++crit_ver);
        }
        while (static_cast<double>(cp) + 1.0 <= rc.beta_pv * static_cast<double>(cv)) {
          p.update_n(1);
          ++cp;
          if (cp % rc.publish_every == 0) {  // policy snapshot -> actor -> V-learner
            last_a = p.last_loss();
            aloss.add(last_a);
            ++pol_ver;
            actor.adopt_policy(p.policy_dev(), pol_ver, true);
            v.adopt_policy_device(p.policy_dev(), pol_ver);
          }
        }
      }
    }
    if (writer && ca >= next_eval) {
      row();
      next_eval += mc->every_actor_steps;
    }
  }
  PQLG_CUDA(cudaStreamSynchronize(st));
  if (writer) row();
  pqlg_run_report r{};
  r.ok = 1;
  r.wall_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  r.c_a = ca;
  r.c_v = cv;
  r.c_p = cp;
  r.env_steps = ca * N;
  r.ratio_av = cv ? static_cast<double>(ca) / cv : 0.0;
  r.ratio_pv = cv ? static_cast<double>(cp) / cv : 0.0;
  r.policy_version = pol_ver;
  r.critic_version = crit_ver;
  r.last_critic_loss = cv ? v.last_loss() : 0.0f;
  r.last_actor_loss = cp ? p.last_loss() : 0.0f;
  (void)Pp;
  return r;
}

}  // namespace pqlg

struct pqlg_pipeline_s {
  std::unique_ptr<pqlg::Pipeline> p;
};

using namespace pqlg;

extern "C" {

void pqlg_ratio_config_default(pqlg_ratio_config* c) {
  // RatioConfig defaults (ratio_gate.hpp:17-25) + SPEC.md:486-492
  *c = pqlg_ratio_config{};
  c->beta_av = 1.0 / 8.0;
  c->beta_pv = 1.0 / 2.0;
  c->slack_a = 4.0;
  c->slack_p = 1.0;
  c->slack_v = 1.0;
  c->warm_up = 32;
  c->free_running = 0;
  c->horizon = 4;
  c->channel_capacity = 8;
  c->publish_every = 8;
}

int pqlg_ratio_may_proceed(int proc, int64_t c_a, int64_t c_v, int64_t c_p,
                           const pqlg_ratio_config* cfg) {
  if (!cfg || proc < 0 || proc > 2) return -1;
  return may_proceed(proc, c_a, c_v, c_p, *cfg) ? 1 : 0;
}

int pqlg_pipeline_create(const pqlg_config* cfg, const pqlg_task_dims* dims,
                         const pqlg_ratio_config* rc, uint64_t init_rng_seed, pqlg_pipeline* out) {
  return guarded([&] {
    require(cfg && dims && rc && out, "pipeline_create: null argument");
    auto h = std::make_unique<pqlg_pipeline_s>();
    h->p = std::make_unique<Pipeline>(*cfg, *dims, *rc, init_rng_seed);
    *out = h.release();
  });
}

int pqlg_pipeline_run(pqlg_pipeline h, int64_t actor_steps, double max_seconds,
                      pqlg_run_report* out) {
  return guarded([&] {
    require(h && out, "pipeline_run: null argument");
    *out = h->p->run(actor_steps, max_seconds);
  });
}

int pqlg_pipeline_record_snapshots(pqlg_pipeline h, int on) {
  return guarded([&] {
    require(h, "pipeline_record_snapshots: null handle");
    h->p->record_snapshots(on != 0);
  });
}

int pqlg_pipeline_check_critics(pqlg_pipeline h, int64_t* p_version, double* max_abs_diff) {
  return guarded([&] {
    require(h && p_version && max_abs_diff, "pipeline_check_critics: null argument");
    h->p->check_critics(p_version, max_abs_diff);
  });
}

int pqlg_pipeline_destroy(pqlg_pipeline h) {
  return guarded([&] { delete h; });
}

int pqlg_pipeline_set_metrics(pqlg_pipeline h, const pqlg_metrics_config* m) {
  return guarded([&] {
    require(h && m, "pipeline_set_metrics: null argument");
    h->p->set_metrics(*m);
  });
}

int pqlg_run_synchronous(const pqlg_config* cfg, const pqlg_task_dims* dims,
                         const pqlg_ratio_config* rc, uint64_t init_rng_seed, int64_t actor_steps,
                         const pqlg_metrics_config* metrics, pqlg_run_report* out) {
  return guarded([&] {
    require(cfg && dims && rc && out, "run_synchronous: null argument");
    *out = run_synchronous(*cfg, *dims, *rc, init_rng_seed, actor_steps, metrics);
  });
}

}  // extern "C"
