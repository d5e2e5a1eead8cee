// Actor: ActorCore::rollout_step (proj/include/pql/runtime/learners.hpp:52-73,
// proj/src/runtime/learners.cpp:62-116) on one B200, with the synthetic GPU
// environment behind the EnvBatch contract (vecenv.hpp:44-81).
//
// One step = normalize (stats of step t-1) -> policy (tcgen05 GEMMs) whose
// head epilogue squashes, adds the per-env mixed exploration noise and clamps
// -> env step kernel (auto-reset, terminal obs, truncation) -> StepSlice
// views -> running-normalizer update over the step's observations.
#include <cmath>
#include <cstdlib>
#include <memory>
#include <random>
#include <vector>

#include "actor.h"
#include "comm.h"
#include "actor_kernels.cuh"
#include "learner.h"

namespace pqlg {

// Host copy of the synthetic task's fixed coupling matrix (SURVEY 8(d)
// synthetic env): M[d][k] = 2 * (splitmix64(derive_seed(seed, env, 2^40) +
// d*A + k) >> 11) * 2^-53 - 1.
static std::vector<float> coupling_matrix(uint64_t seed, int D, int A) {
  std::vector<float> M(static_cast<size_t>(D) * A);
  const uint64_t mseed = rng::derive_seed(seed, rng::kEnv, 1ull << 40);
  for (int d = 0; d < D; ++d)
    for (int k = 0; k < A; ++k) {
      const uint64_t u = rng::splitmix64(mseed + static_cast<uint64_t>(d) * A + k);
      M[static_cast<size_t>(d) * A + k] =
          static_cast<float>(static_cast<double>(u >> 11) * 0x1.0p-53 * 2.0 - 1.0);
    }
  return M;
}

// Synthetic EnvBatch on device (also exposed through pqlg_env_*).
struct DeviceEnv {
  int N, D, A, max_len, offset;
  int64_t ld;
  float low, high;
  DevBuf<float> s, M, MT;
  DevBuf<int64_t> ep;
  DevBuf<uint64_t> rng;

  DeviceEnv(int n, int obs_dim, int act_dim, uint64_t seed, int max_episode_len, int env_offset,
            float lo, float hi)
      : N(n), D(obs_dim), A(act_dim), max_len(max_episode_len), offset(env_offset), low(lo),
        high(hi) {
    require(n >= 1, "make_env: n_envs must be >= 1");  // vecenv.cpp:57
    require(max_episode_len >= 1, "env: max_episode_len must be >= 1");
    ld = round_up(D, 4);
    s.alloc(static_cast<size_t>(N) * ld);
    auto m = coupling_matrix(seed, D, A);
    M.alloc(m.size());
    copy_sync(M.p, m.data(), m.size() * 4, cudaMemcpyHostToDevice);
    if (A <= actor::kMaxA && D <= actor::kMaxD) {
      const auto t = actor::env_transpose_M(m, D, A);
      MT.alloc(t.size());
      copy_sync(MT.p, t.data(), t.size() * 4, cudaMemcpyHostToDevice);
    }
    ep.alloc(N);
    std::vector<uint64_t> r(N);
    for (int i = 0; i < N; ++i) r[i] = rng::derive_seed(seed, rng::kEnv, offset + i);
    rng.alloc(N);
    copy_sync(rng.p, r.data(), N * 8, cudaMemcpyHostToDevice);
  }
  actor::EnvState view() const {
    return actor::EnvState{s.p, ld, s.p, ld, M.p, reinterpret_cast<const float4*>(MT.p), ep.p, rng.p,
                           N, D, A, max_len, low, high, 1.0f};
  }
  void reset(float* obs, int64_t ld_obs, cudaStream_t st) {
    launch(actor::env_reset_kernel, dim3((N + actor::kEnvWarps - 1) / actor::kEnvWarps), dim3(32 * actor::kEnvWarps), 0, st, view(), obs, ld_obs, offset);
  }
  // persistent grid: as many blocks as fit (occupancy), at most one per tile
  template <int kSlots>
  void step_as(const float* act, int64_t ld_act, const actor::StepOut& o, cudaStream_t st,
               const actor::NextNorm& nn, const float* cur, int64_t ld_cur,
               const actor::NormPartialOut& np) {
    actor::EnvState v = view();
    if (cur) {  // the caller's obs buffers hold the state: read cur, write next_obs only
      v.s = nullptr;
      v.s_in = cur;
      v.ld_in = ld_cur;
    }
    require(v.ld_in % 4 == 0 && (reinterpret_cast<uintptr_t>(v.s_in) & 15) == 0,
            "env: state rows must be 16-byte aligned");
    const int tiles = (N + actor::kEnvTile - 1) / actor::kEnvTile;
    // the bulk path: one 16-byte row stride for state, boot, next obs and
    // normalised next obs (the actor's Dp-wide buffers)
    const bool rows16 = o.ld_obs == v.ld_in && (!nn.out || nn.ld_out == v.ld_in) &&
                        (!v.s || v.ld == v.ld_in) &&
                        ((reinterpret_cast<uintptr_t>(o.next_obs) | reinterpret_cast<uintptr_t>(o.boot) |
                          reinterpret_cast<uintptr_t>(nn.out) | reinterpret_cast<uintptr_t>(v.s)) & 15) == 0;
    if (rows16 && actor::env_tma_ok(act, ld_act, D, A, v.ld_in)) {
      // TMA-fed persistent kernel, one CTA per SM (tma_grid(): the actor's
      // normalizer partial count)
      auto kern = actor::env_step_tma_kernel<kSlots>;
      const size_t smem = actor::env_tma_smem(A, kSlots, v.ld_in, ld_act);
      static size_t configured = 0;
      if (configured < smem) {
        PQLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       static_cast<int>(smem)));
        configured = smem;
      }
#ifdef PQLG_ENV_TRACE
      if (std::getenv("PQLG_ENV_NOPART")) {  // A/B only: no normalizer partials
        launch(kern, dim3(tma_grid()), dim3(actor::kEnvTmaThreads), smem, st, v, act, ld_act, o, nn,
               actor::NormPartialOut{});
        return;
      }
#endif
      launch(kern, dim3(tma_grid()), dim3(actor::kEnvTmaThreads), smem, st, v, act, ld_act, o, nn,
             np);
      return;
    }
    require(!np.partial, "env: normalizer partials need the TMA step (16-byte rows)");
    auto kern = actor::env_step_kernel<kSlots>;
    const size_t smem = actor::env_step_smem(D, A, kSlots);
    static int per_sm = 0;
    static size_t per_sm_smem = 0;
    if (per_sm == 0 || per_sm_smem != smem) {
      PQLG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                     200 * 1024));
      PQLG_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern,
                                                              32 * actor::kEnvWarps, smem));
      if (per_sm < 1) per_sm = 1;
      per_sm_smem = smem;
    }
    const int blocks = std::min(tiles, per_sm * mlp::kSMs);
    launch(kern, dim3(blocks), dim3(32 * actor::kEnvWarps), smem, st, v, act, ld_act, o, nn);
  }
  // blocks of the TMA step = partial sums it writes (one per SM, <= tiles)
  int tma_grid() const {
    const int tiles = (N + actor::kEnvTile - 1) / actor::kEnvTile;
    return std::min(tiles, mlp::kSMs);
  }
  // cur: optional obs buffer holding the current state (the actor's double
  // buffer); then the internal state array is neither read nor written.
  // np: optional running-normalizer partials of the next observations.
  void step(const float* act, int64_t ld_act, const actor::StepOut& o, cudaStream_t st,
            const actor::NextNorm& nn = actor::NextNorm{}, const float* cur = nullptr,
            int64_t ld_cur = 0, const actor::NormPartialOut& np = actor::NormPartialOut{}) {
    require(A <= actor::kMaxA, "env: act_dim > 32 not supported");
    require(D <= actor::kMaxD, "env: obs_dim > 256 not supported");
    if ((D + 3) / 4 <= 32) step_as<1>(act, ld_act, o, st, nn, cur, ld_cur, np);
    else step_as<2>(act, ld_act, o, st, nn, cur, ld_cur, np);
  }
};

Actor::Actor(const pqlg_config& cfg, const pqlg_task_dims& dims, cudaStream_t st,
             pqlg_comm_s* comm)
    : cfg_(cfg), dims_(dims), stream_(st), comm_(comm) {
  if (!stream_) {
    PQLG_CUDA(cudaStreamCreateWithFlags(&owned_stream_, cudaStreamNonBlocking));
    stream_ = owned_stream_;
  }
  require(cfg.precision == PQLG_PREC_TF32 || cfg.precision == PQLG_PREC_3XTF32,
          "actor: unknown precision");
  require(cfg.algo == PQLG_ALGO_DDPG || cfg.algo == PQLG_ALGO_C51 || cfg.algo == PQLG_ALGO_SAC,
          "actor: unknown algo");
  sac_ = cfg.algo == PQLG_ALGO_SAC;
  require(!sac_ || dims.act_dim <= 32, "actor: pql_sac needs act_dim <= 32");
  require(cfg.hidden_layers >= 1 && cfg.hidden >= 32 && cfg.hidden % 32 == 0,
          "actor: hidden width must be a multiple of 32");
  N_ = cfg.n_envs;
  D_ = dims.obs_dim;
  A_ = dims.act_dim;
  Ap_ = static_cast<int>(round_up(A_, 4));
  H_ = cfg.hidden;
  nh_ = cfg.hidden_layers;
  Dp_ = round_up(D_, 4);
  std::vector<int> ps{D_};
  for (int i = 0; i < nh_; ++i) ps.push_back(H_);
  ps.push_back(sac_ ? 2 * A_ : A_);  // GaussianPolicy: [mean | log_std] (learners.cpp:20-22)
  pnet_ = NetShape::make(ps);

  // policy: PolicyHandle::create with make_rng(seed, init, 0) (learners.cpp:69)
  std::mt19937_64 prng(rng::derive_seed(cfg.seed, rng::kInit, 0));
  std::vector<float> pol;
  init_orthogonal(pnet_, pol, prng, static_cast<float>(std::sqrt(2.0)), 1e-2f);
  pol_.alloc(snapshot_len());  // [net | log_alpha] for pql_sac (log_alpha unused here)
  copy_sync(pol_.p, pol.data(), pol.size() * 4, cudaMemcpyHostToDevice);

  // exploration: build_schedule over the global env count (noise.hpp:23-42;
  // a sharded actor takes its slice of the one global schedule), per-env
  // SplitMix streams derive_seed(seed, noise, global i) (learners.cpp:74-75)
  const int n_total = cfg.envs_total > 0 ? cfg.envs_total : N_;
  require(cfg.env_offset + N_ <= n_total, "actor: env_offset + n_envs exceeds envs_total");
  std::vector<float> sig(N_);
  for (int i = 0; i < N_; ++i) {
    const int gi = cfg.env_offset + i;
    const float smin = static_cast<float>(cfg.sigma_min), smax = static_cast<float>(cfg.sigma_max);
    float v;
    if (cfg.sigma_fixed >= 0.0) v = static_cast<float>(cfg.sigma_fixed);  // build_fixed_schedule
    else if (n_total == 1 || gi == 0) v = smin;
    else if (gi == n_total - 1) v = smax;
    else {
      const double lo = smin, span = static_cast<double>(smax) - smin;
      v = static_cast<float>(lo + (static_cast<double>(gi) / (n_total - 1)) * span);
    }
    sig[i] = v;
  }
  sigma_.alloc(N_);
  copy_sync(sigma_.p, sig.data(), N_ * 4, cudaMemcpyHostToDevice);
  std::vector<uint64_t> nr(N_);
  for (int i = 0; i < N_; ++i) nr[i] = rng::derive_seed(cfg.seed, rng::kNoise, cfg.env_offset + i);
  noise_rng_.alloc(N_);
  copy_sync(noise_rng_.p, nr.data(), N_ * 8, cudaMemcpyHostToDevice);

  // environment + initial observations (make_env -> reset_all, learners.cpp:66-68)
  env_ = std::make_unique<DeviceEnv>(N_, D_, A_, cfg.seed, cfg.max_episode_len, cfg.env_offset,
                                     dims.low, dims.high);
  for (int k = 0; k < kSets; ++k) {
    obs_[k].alloc(static_cast<size_t>(N_) * Dp_);
    boot_[k].alloc(static_cast<size_t>(N_) * Dp_);
    rew_[k].alloc(N_);
    term_[k].alloc(N_);
    trunc_[k].alloc(N_);
    act_[k].alloc(static_cast<size_t>(N_) * Ap_);
  }
  Xn_.alloc(static_cast<size_t>(N_) * Dp_);
  env_->reset(obs_[0].p, Dp_, stream_);

  // normalizer (count 0 -> identity)
  count_.alloc(1);
  mean_.alloc(D_);
  m2_.alloc(D_);
  mean_f_.alloc(D_);
  inv_f_.alloc(D_);
  identity_.alloc(1);
  const int one = 1;
  copy_sync(identity_.p, &one, 4, cudaMemcpyHostToDevice);
  npart_.alloc(static_cast<size_t>(actor::kNormBlocks) * D_ * 2);
  if (comm_) {
    require(D_ <= 1024, "actor: sharded normalizer needs obs_dim <= 1024");
    nbatch_.alloc(2 * static_cast<size_t>(D_) + 1);
    ngather_.alloc(static_cast<size_t>(comm_->world) * (2 * D_ + 1));
  }
  nticket_.alloc(actor::norm_tickets(D_));
  nshift_.alloc(D_);
  status_.alloc(1);
  // the first step's normalizer partials (later steps get them from the env
  // step that produced their observations)
  actor::norm_partial(obs_[0].p, Dp_, N_, D_, env_->tma_grid(), npart_.p, nshift_.p, stream_);
  // first policy input: apply_stats with count 0 is the identity
  launch(actor::normalize_kernel, dim3(4 * mlp::kSMs), dim3(256), 0, stream_, obs_[0].p, Dp_, Xn_.p, Dp_,
                                                               mean_f_.p, inv_f_.p, identity_.p,
                                                               N_, D_);
  {
    gemm::PrecisionScope prec(cfg.precision == PQLG_PREC_3XTF32);
    build();
  }
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

Actor::~Actor() {
  if (step_done_) cudaEventDestroy(step_done_);
  for (auto& g : graph_)
    if (g) cudaGraphExecDestroy(g);
  if (owned_stream_) {
    cudaStreamSynchronize(owned_stream_);
    cudaStreamDestroy(owned_stream_);
  }
}

void Actor::build() {
  const int N = N_, D = D_, A = A_, H = H_, nh = nh_;
  const int bnH = mlp::bn_for(H);
  pact_.resize(nh);
  for (auto& b : pact_) b.alloc(static_cast<size_t>(N) * H);
  const float* in = Xn_.p;
  int64_t ld = Dp_;
  int K = D;
  for (int l = 0; l < nh; ++l) {
    epi::Hidden e{};
    e.bias[0] = e.bias[1] = pol_.p + pnet_.b_off[l];
    e.bn = bnH;
    e.M = N;
    e.N = H;
    e.store = 1;
    const float* W = pol_.p + pnet_.w_off[l];
    policy_steps_.push_back(mlp::fwd(in, in, ld, W, W, N, H, K, 1, e, 0, pact_[l].p, pact_[l].p, H));
    in = pact_[l].p;
    ld = H;
    K = H;
  }
  if (sac_) {
    // GaussianPolicy::sample with a fresh normal_distribution per env over
    // its noise stream (learners.cpp:87-94): split-K head + sampling finish
    // packed head weights and the normalizer finish ride in the head launch
    // (as for the deterministic head below)
    head::RowsArgs base{};
    wpack_.alloc(static_cast<size_t>(mlp::head_pack_elems(2 * A, H)) * 4);
    base.wpack = reinterpret_cast<const float4*>(wpack_.p);
    pack_head();
    base.fin = actor::norm_finish_args(nshift_.p, N, D_, env_->tma_grid(), npart_.p, nticket_.p,
                                       norm_state());
    fused_finish_ = true;
    auto gemm = mlp::head_raw_step(head_split_, in, ld, pol_.p + pnet_.w_off[nh], N, 2 * A, H,
                                   base);
    sac::GaussArgs g{};
    g.bias = pol_.p + pnet_.b_off[nh];
    g.rng = noise_rng_.p;
    g.ld_act = Ap_;
    g.mid = (dims_.low + dims_.high) / 2.0f;
    g.half = (dims_.high - dims_.low) / 2.0f;
    for (int k = 0; k < kSets; ++k) {
      g.act = act_[k].p;
      auto fin = gauss_finish_step(head_split_, g, N, A);
      head_steps_[k] = [gemm, fin](cudaStream_t st) {
        gemm(st);
        fin(st);
      };
    }
    return;
  }
  // DeterministicPolicy::act + apply_noise (learners.cpp:96-98), fused
  head::RowsArgs ph{};
  ph.bias = pol_.p + pnet_.b_off[nh];
  ph.ld_out = Ap_;
  ph.mid = (dims_.low + dims_.high) / 2.0f;
  ph.half = (dims_.high - dims_.low) / 2.0f;
  ph.noise_state = noise_rng_.p;
  ph.sigma = sigma_.p;
  ph.low = dims_.low;
  ph.high = dims_.high;
  const float* W = pol_.p + pnet_.w_off[nh];
  // the head's W in fragment order, re-packed whenever the policy changes
  wpack_.alloc(static_cast<size_t>(mlp::head_pack_elems(A, H)) * 4);
  ph.wpack = reinterpret_cast<const float4*>(wpack_.p);
  pack_head();
  // the normalizer update's finish (independent of the policy) rides in the
  // head launch as extra blocks
  ph.fin = actor::norm_finish_args(nshift_.p, N, D_, env_->tma_grid(), npart_.p, nticket_.p,
                                   norm_state());
  fused_finish_ = true;
  for (int k = 0; k < kSets; ++k) {
    ph.out = act_[k].p;
    head_steps_[k] = mlp::head_squash_step(ph, in, ld, W, N, A, H);
  }
}

actor::NormState Actor::norm_state() const {
  return actor::NormState{count_.p, mean_.p, m2_.p, mean_f_.p, inv_f_.p, identity_.p,
                          comm_ ? nbatch_.p : nullptr};
}

void Actor::pack_head() {
  if (!wpack_.p) return;
  const int hout = sac_ ? 2 * A_ : A_;  // GaussianPolicy: [mean | log_std]
  mlp::head_pack(pol_.p + pnet_.w_off[nh_], hout, H_, hout, reinterpret_cast<float4*>(wpack_.p),
                 cfg_.precision == PQLG_PREC_3XTF32, stream_);
}

void Actor::enqueue(int cur) {
  cudaStream_t st = stream_;
  const int N = N_, D = D_;
  const float* obs = obs_[cur].p;
  // PQLG_SKIP_STEP=i drops launch i of the step (tools/skip_probe.py: in-situ
  // marginal costs; the results of such a step are meaningless)
  const int skip = skip_step();
  int idx = 0;
  auto keep = [&] { return idx++ != skip; };
  // actions = pi(obs_norm) + mixed noise; Xn_ holds apply(stats_{t-1}, obs_t)
  for (auto& s : policy_steps_)
    if (keep()) s(st);
  if (keep()) head_steps_[cur](st);
  // normalizer_.update(obs_) (learners.cpp:113): it only reads this step's
  // observations, so it runs before the env step and the env kernel can emit
  // the next policy input apply(stats_t, obs_{t+1}) directly.
  actor::NormState ns = norm_state();
  // the partial sums of obs were written by the env step that produced them
  // (the finish runs inside the head launch unless the head is pql_sac's)
  if (!fused_finish_ && keep())
    actor::norm_finish(nshift_.p, N, D, env_->tma_grid(), npart_.p, nticket_.p, ns, st);
  if (comm_) {
    // sharded: every shard's batch statistics, merged in rank
    // order into identical running stats on all shards (5 KB at config 3)
    allgather_f64(comm_, nbatch_.p, ngather_.p, 2 * static_cast<size_t>(D) + 1, st);
    ns.batch = nullptr;
    launch(actor::norm_merge_kernel, dim3(1), dim3((D + 31) / 32 * 32), 0, st, ngather_.p,
           comm_->world, D, ns);
  }
  // env_->step(actions) + next-obs normalisation
  const int nxt = (cur + 1) % kSets;
  actor::StepOut o{obs_[nxt].p, boot_[cur].p, rew_[cur].p, term_[cur].p, trunc_[cur].p, nullptr,
                   Dp_, status_.p};
  actor::NextNorm nn{Xn_.p, Dp_, mean_f_.p, inv_f_.p, identity_.p};
  // ... and the partials of the next observations for the next step's update
  actor::NormPartialOut np{reinterpret_cast<double2*>(npart_.p), nshift_.p, mean_.p};
  if (keep()) env_->step(act_[cur].p, Ap_, o, st, nn, obs, Dp_, np);
}

int Actor::kernels_per_step() {
  if (kps_ == 0) {
    const uint64_t before = g_launches.load();
    cudaGraph_t g;
    PQLG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    enqueue(0);
    PQLG_CUDA(cudaStreamEndCapture(stream_, &g));
    cudaGraphDestroy(g);
    kps_ = static_cast<int>(g_launches.load() - before);
    g_launches.fetch_sub(kps_);
  }
  return kps_;
}

void Actor::rollout_step(pqlg_step_slice* out) {
  const int cur = cur_;
  // one replay of the step's captured graph (the same launches as enqueue;
  // one host call instead of one per kernel); PQLG_EAGER=1 launches eagerly
  if (eager_updates()) {
    enqueue(cur);
  } else {
    ensure_graphs();
    PQLG_CUDA(cudaGraphLaunch(graph_[cur], stream_));
    count_launch(static_cast<uint64_t>(kps_));
  }
  stepped_ = true;
  if (!step_done_) PQLG_CUDA(cudaEventCreateWithFlags(&step_done_, cudaEventDisableTiming));
  PQLG_CUDA(cudaEventRecord(step_done_, stream_));  // consumers on other streams wait on it
  if (out) {
    out->obs = obs_[cur].p;
    out->act = act_[cur].p;
    out->boot_obs = boot_[cur].p;
    out->rew = rew_[cur].p;
    out->term = term_[cur].p;
    out->trunc = trunc_[cur].p;
    out->ld_obs = Dp_;
    out->ld_act = Ap_;
  }
  cur_ = (cur + 1) % kSets;
}

std::string Actor::time_steps(int reps) {
  return time_in_graph(
      [&] {
        for (int k = 0; k < kSets; ++k) enqueue((cur_ + k) % kSets);
      },
      stream_, reps);
}

void Actor::ensure_graphs() {
  for (int c = 0; c < kSets; ++c) {
    if (graph_[c]) continue;
    kernels_per_step();
    cudaGraph_t g;
    PQLG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    enqueue(c);
    PQLG_CUDA(cudaStreamEndCapture(stream_, &g));
    g_launches.fetch_sub(kps_);
    PQLG_CUDA(cudaGraphInstantiate(&graph_[c], g, 0));
    cudaGraphDestroy(g);
  }
}

void Actor::rollout_n(int n) {
  ensure_graphs();
  for (int i = 0; i < n; ++i) {
    PQLG_CUDA(cudaGraphLaunch(graph_[cur_], stream_));
    cur_ = (cur_ + 1) % kSets;
  }
  count_launch(static_cast<uint64_t>(n) * kps_);
}

void Actor::adopt_policy(const float* flat, int64_t version, bool device) {
  if (version < version_) return;  // PolicyHandle::adopt (learners.cpp:37-42)
  // device snapshots carry [net | log_alpha]; the host ABI passes the net
  PQLG_CUDA(cudaMemcpyAsync(pol_.p, flat, (device ? snapshot_len() : pnet_.params) * 4,
                            device ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, stream_));
  pack_head();
  if (!device) PQLG_CUDA(cudaStreamSynchronize(stream_));
  version_ = version;
}

void Actor::set_norm(int64_t count, const double* mean, const double* m2) {
  PQLG_CUDA(cudaMemcpyAsync(count_.p, &count, 8, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(mean_.p, mean, D_ * 8, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(m2_.p, m2, D_ * 8, cudaMemcpyHostToDevice, stream_));
  launch_norm_consts(count_.p, mean_.p, m2_.p, D_, mean_f_.p, inv_f_.p, identity_.p, stream_);
  launch(actor::normalize_kernel, dim3(4 * mlp::kSMs), dim3(256), 0, stream_, obs_[cur_].p, Dp_,
         Xn_.p, Dp_, mean_f_.p, inv_f_.p, identity_.p, N_, D_);
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

void Actor::norm(int64_t* count, double* mean, double* m2) {
  PQLG_CUDA(cudaMemcpyAsync(count, count_.p, 8, cudaMemcpyDeviceToHost, stream_));
  if (mean) PQLG_CUDA(cudaMemcpyAsync(mean, mean_.p, D_ * 8, cudaMemcpyDeviceToHost, stream_));
  if (m2) PQLG_CUDA(cudaMemcpyAsync(m2, m2_.p, D_ * 8, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

// what: 0 current obs [N x D] f32, 1 last actions [N x A] f32, 2 noise stream
// states [N] u64, 3 env episode steps [N] i64, 4 env stream states [N] u64,
// 5 policy params, 6 status word (u32)
void Actor::read_state(int what, void* out) {
  auto st = stream_;
  switch (what) {
    case 0:
      PQLG_CUDA(cudaMemcpy2DAsync(out, D_ * 4, obs_[cur_].p, Dp_ * 4, D_ * 4, N_,
                                  cudaMemcpyDeviceToHost, st));
      break;
    case 1:
      PQLG_CUDA(cudaMemcpy2DAsync(out, A_ * 4, act_[(cur_ + kSets - 1) % kSets].p, Ap_ * 4,
                                  A_ * 4, N_, cudaMemcpyDeviceToHost, st));
      break;
    case 2: PQLG_CUDA(cudaMemcpyAsync(out, noise_rng_.p, N_ * 8, cudaMemcpyDeviceToHost, st)); break;
    case 3: PQLG_CUDA(cudaMemcpyAsync(out, env_->ep.p, N_ * 8, cudaMemcpyDeviceToHost, st)); break;
    case 4: PQLG_CUDA(cudaMemcpyAsync(out, env_->rng.p, N_ * 8, cudaMemcpyDeviceToHost, st)); break;
    case 5:
      PQLG_CUDA(cudaMemcpyAsync(out, pol_.p, pnet_.params * 4, cudaMemcpyDeviceToHost, st));
      break;
    case 6: PQLG_CUDA(cudaMemcpyAsync(out, status_.p, 4, cudaMemcpyDeviceToHost, st)); break;
    default: throw Error(PQLG_EINVAL, "actor_read: what must be 0..6");
  }
  PQLG_CUDA(cudaStreamSynchronize(st));
}

void Actor::read_last_slice(float* obs, float* act, float* boot, float* rew, uint8_t* term,
                            uint8_t* trunc) {
  require(stepped_, "actor_read_slice: no rollout_step yet");
  const int k = (cur_ + kSets - 1) % kSets;
  auto st = stream_;
  if (obs)
    PQLG_CUDA(cudaMemcpy2DAsync(obs, D_ * 4, obs_[k].p, Dp_ * 4, D_ * 4, N_,
                                cudaMemcpyDeviceToHost, st));
  if (act)
    PQLG_CUDA(cudaMemcpy2DAsync(act, A_ * 4, act_[k].p, Ap_ * 4, A_ * 4, N_,
                                cudaMemcpyDeviceToHost, st));
  if (boot)
    PQLG_CUDA(cudaMemcpy2DAsync(boot, D_ * 4, boot_[k].p, Dp_ * 4, D_ * 4, N_,
                                cudaMemcpyDeviceToHost, st));
  if (rew) PQLG_CUDA(cudaMemcpyAsync(rew, rew_[k].p, N_ * 4, cudaMemcpyDeviceToHost, st));
  if (term) PQLG_CUDA(cudaMemcpyAsync(term, term_[k].p, N_, cudaMemcpyDeviceToHost, st));
  if (trunc) PQLG_CUDA(cudaMemcpyAsync(trunc, trunc_[k].p, N_, cudaMemcpyDeviceToHost, st));
  PQLG_CUDA(cudaStreamSynchronize(st));
}

// ------------------------------------------------------------ evaluation
// evaluate_policy (learners.cpp:280-325) on the synthetic task: a fresh env
// of `episodes` rows (seed eval_seed, every row starting a full episode),
// the deterministic policy on apply_stats(snapshot norm, obs), one episode
// per row, returns accumulated in double until each row's first done.
namespace {
__global__ void eval_accumulate_kernel(const float* rew, const uint8_t* term,
                                       const uint8_t* trunc, int N, double* ret,
                                       uint8_t* finished, unsigned int* n_finished) {
  pdl::entry();
  for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < N; i += gridDim.x * blockDim.x) {
    if (finished[i]) continue;
    ret[i] += static_cast<double>(rew[i]);
    if (term[i] || trunc[i]) {
      finished[i] = 1;
      atomicAdd(n_finished, 1u);
    }
  }
}
}  // namespace

struct Evaluator::Impl {
  pqlg_config cfg;
  int N, D, A;
  int64_t Dp, Ap;
  cudaStream_t st = nullptr;
  NetShape pnet;
  DevBuf<float> pol;
  std::unique_ptr<DeviceEnv> env;
  DevBuf<uint64_t> rng0;  // the env's per-row streams as make_env seeds them
  DevBuf<float> obs[2], boot, rew, act, Xn;
  DevBuf<uint8_t> flags;  // term | trunc | finished
  DevBuf<double> ret;
  DevBuf<unsigned int> n_fin;
  DevBuf<uint32_t> status;
  DeviceNorm norm;
  std::vector<DevBuf<float>> pact;
  std::vector<mlp::Step> steps;
  std::vector<double> r;
  ~Impl() {
    if (st) {
      cudaStreamSynchronize(st);
      cudaStreamDestroy(st);
    }
  }
};

Evaluator::Evaluator(const pqlg_config& cfg, const pqlg_task_dims& dims, int episodes,
                     uint64_t eval_seed)
    : p_(std::make_unique<Impl>()) {
  require(episodes >= 1, "evaluate: episodes must be >= 1");  // learners.cpp:282
  Impl& e = *p_;
  e.cfg = cfg;
  const int N = e.N = episodes, D = e.D = dims.obs_dim, A = e.A = dims.act_dim;
  const int H = cfg.hidden, nh = cfg.hidden_layers;
  require(A <= 32, "evaluate: act_dim > 32 not supported");
  require(cfg.precision == PQLG_PREC_TF32 || cfg.precision == PQLG_PREC_3XTF32,
          "evaluate: unknown precision");
  gemm::PrecisionScope prec(cfg.precision == PQLG_PREC_3XTF32);
  PQLG_CUDA(cudaStreamCreateWithFlags(&e.st, cudaStreamNonBlocking));
  // pql_sac evaluates the squashed mean (GaussianPolicy::mean_act,
  // policy.hpp:110-118): the first A of the 2A head outputs
  const bool sac = cfg.algo == PQLG_ALGO_SAC;
  const int hout = sac ? 2 * A : A;
  std::vector<int> ps{D};
  for (int l = 0; l < nh; ++l) ps.push_back(H);
  ps.push_back(hout);
  e.pnet = NetShape::make(ps);
  e.pol.alloc(e.pnet.params);
  e.env = std::make_unique<DeviceEnv>(N, D, A, eval_seed, cfg.max_episode_len, 0, dims.low,
                                      dims.high);
  e.rng0.alloc(N);
  copy_sync(e.rng0.p, e.env->rng.p, N * 8, cudaMemcpyDeviceToDevice);
  e.Dp = round_up(D, 4);
  e.Ap = round_up(A, 4);
  for (auto& o : e.obs) o.alloc(static_cast<size_t>(N) * e.Dp);
  e.boot.alloc(static_cast<size_t>(N) * e.Dp);
  e.rew.alloc(N);
  e.act.alloc(static_cast<size_t>(N) * e.Ap);
  e.Xn.alloc(static_cast<size_t>(N) * e.Dp);
  e.flags.alloc(3ull * N);
  e.ret.alloc(N);
  e.n_fin.alloc(1);
  e.status.alloc(1);
  e.norm.init(D);
  e.r.resize(N);
  // policy forward (hidden layers, squashing head without noise)
  e.pact.resize(nh);
  const float* in = e.Xn.p;
  int64_t ld = e.Dp;
  int K = D;
  for (int l = 0; l < nh; ++l) {
    e.pact[l].alloc(static_cast<size_t>(N) * H);
    epi::Hidden h{};
    h.bias[0] = e.pol.p + e.pnet.b_off[l];
    h.bn = mlp::bn_for(H);
    h.M = N;
    h.N = H;
    h.store = 1;
    const float* W = e.pol.p + e.pnet.w_off[l];
    e.steps.push_back(mlp::fwd(in, in, ld, W, W, N, H, K, 1, h, 0, e.pact[l].p, e.pact[l].p, H));
    in = e.pact[l].p;
    ld = H;
    K = H;
  }
  head::RowsArgs ph{};
  ph.bias = e.pol.p + e.pnet.b_off[nh];
  ph.out = e.act.p;
  ph.ld_out = e.Ap;
  ph.ldw = hout;  // pql_sac: the mean columns of [mean | log_std]
  ph.mid = (dims.low + dims.high) / 2.0f;
  ph.half = (dims.high - dims.low) / 2.0f;
  e.steps.push_back(mlp::head_squash_step(ph, in, ld, e.pol.p + e.pnet.w_off[nh], N, A, H));
}

Evaluator::~Evaluator() = default;

// Every call starts from make_env's state (the row streams restored from
// rng0, fresh episodes), so repeated calls equal fresh evaluate_policy calls.
void Evaluator::run(const float* policy, int64_t count, const double* mean, const double* m2,
                    double* returns, double* mean_out, double* stderr_out) {
  Impl& e = *p_;
  const int N = e.N, D = e.D;
  cudaStream_t st = e.st;
  DeviceEnv& env = *e.env;
  PQLG_CUDA(cudaMemcpyAsync(e.pol.p, policy, e.pnet.params * 4, cudaMemcpyHostToDevice, st));
  PQLG_CUDA(cudaMemcpyAsync(env.rng.p, e.rng0.p, N * 8, cudaMemcpyDeviceToDevice, st));
  PQLG_CUDA(cudaMemsetAsync(e.flags.p, 0, 3ull * N, st));
  PQLG_CUDA(cudaMemsetAsync(e.ret.p, 0, N * 8, st));
  PQLG_CUDA(cudaMemsetAsync(e.n_fin.p, 0, 4, st));
  PQLG_CUDA(cudaMemsetAsync(e.status.p, 0, 4, st));
  e.norm.set(count, mean, m2, st);
  env.reset(e.obs[0].p, e.Dp, st);
  PQLG_CUDA(cudaMemsetAsync(env.ep.p, 0, N * 8, st));  // make_env: fresh episodes
  launch(actor::normalize_kernel, dim3(4 * mlp::kSMs), dim3(256), 0, st, e.obs[0].p, e.Dp, e.Xn.p,
         e.Dp, e.norm.mean.p, e.norm.inv.p, e.norm.ident.p, N, D);
  const int blocks = std::min((N + 255) / 256, 4 * mlp::kSMs);
  int cur = 0;
  for (int step = 0; step < e.cfg.max_episode_len; ++step) {
    for (auto& s : e.steps) s(st);
    actor::StepOut o{e.obs[1 - cur].p, e.boot.p, e.rew.p, e.flags.p, e.flags.p + N, nullptr, e.Dp,
                     e.status.p};
    actor::NextNorm nn{e.Xn.p, e.Dp, e.norm.mean.p, e.norm.inv.p, e.norm.ident.p};
    env.step(e.act.p, e.Ap, o, st, nn, e.obs[cur].p, e.Dp);
    launch(eval_accumulate_kernel, dim3(blocks), dim3(256), 0, st, e.rew.p, e.flags.p,
           e.flags.p + N, N, e.ret.p, e.flags.p + 2 * N, e.n_fin.p);
    cur = 1 - cur;
    if ((step & 15) == 15 || step + 1 == e.cfg.max_episode_len) {  // every row finished?
      unsigned int fin = 0;
      PQLG_CUDA(cudaMemcpyAsync(&fin, e.n_fin.p, 4, cudaMemcpyDeviceToHost, st));
      PQLG_CUDA(cudaStreamSynchronize(st));
      if (fin == static_cast<unsigned int>(N)) break;
    }
  }
  std::vector<double>& r = e.r;
  PQLG_CUDA(cudaMemcpyAsync(r.data(), e.ret.p, N * 8, cudaMemcpyDeviceToHost, st));
  uint32_t stv = 0;
  PQLG_CUDA(cudaMemcpyAsync(&stv, e.status.p, 4, cudaMemcpyDeviceToHost, st));
  PQLG_CUDA(cudaStreamSynchronize(st));
  if (stv) throw Error(PQLG_ENONFINITE, "evaluate: non-finite action");
  double mu = 0.0;
  for (double x : r) mu += x;
  mu /= static_cast<double>(N);
  double var = 0.0;
  for (double x : r) var += (x - mu) * (x - mu);
  var = N > 1 ? var / static_cast<double>(N - 1) : 0.0;
  if (returns) std::copy(r.begin(), r.end(), returns);
  *mean_out = mu;
  *stderr_out = std::sqrt(var / static_cast<double>(N));
}

void evaluate_policy(const pqlg_config& cfg, const pqlg_task_dims& dims, const float* policy,
                     int64_t count, const double* mean, const double* m2, int episodes,
                     uint64_t eval_seed, double* returns, double* mean_out, double* stderr_out) {
  Evaluator(cfg, dims, episodes, eval_seed)
      .run(policy, count, mean, m2, returns, mean_out, stderr_out);
}

}  // namespace pqlg

// ------------------------------------------------------------------ C ABI
struct pqlg_actor_s {
  std::unique_ptr<pqlg::Actor> a;
};

namespace pqlg {
Actor* actor_of(pqlg_actor h) {
  require(h != nullptr, "null actor handle");
  return h->a.get();
}
}  // namespace pqlg
struct pqlg_env_s {
  std::unique_ptr<pqlg::DeviceEnv> e;
  pqlg::DevBuf<uint32_t> status;
  cudaStream_t stream;
};

using namespace pqlg;

extern "C" {

int pqlg_actor_create(const pqlg_config* cfg, const pqlg_task_dims* dims, void* stream,
                      pqlg_actor* out) {
  return guarded([&] {
    require(cfg && dims && out, "actor_create: null argument");
    auto h = std::make_unique<pqlg_actor_s>();
    h->a = std::make_unique<Actor>(*cfg, *dims, static_cast<cudaStream_t>(stream));
    *out = h.release();
  });
}

int pqlg_actor_create_sharded(const pqlg_config* cfg, const pqlg_task_dims* dims, pqlg_comm comm,
                              void* stream, pqlg_actor* out) {
  return guarded([&] {
    require(cfg && dims && out && comm, "actor_create_sharded: null argument");
    auto h = std::make_unique<pqlg_actor_s>();
    h->a = std::make_unique<Actor>(*cfg, *dims, static_cast<cudaStream_t>(stream), comm);
    *out = h.release();
  });
}

int pqlg_actor_step_event(pqlg_actor h, void** event_out) {
  return guarded([&] {
    require(h && event_out, "actor_step_event: null argument");
    *event_out = h->a->step_event();
  });
}

int pqlg_actor_wait_event(pqlg_actor h, void* event) {
  return guarded([&] {
    require(h && event, "actor_wait_event: null argument");
    PQLG_CUDA(cudaStreamWaitEvent(h->a->stream(), static_cast<cudaEvent_t>(event), 0));
  });
}

int pqlg_actor_destroy(pqlg_actor h) {
  return guarded([&] { delete h; });
}

int pqlg_evaluate(const pqlg_config* cfg, const pqlg_task_dims* dims, const float* policy_host,
                  const pqlg_norm_stats* norm, int episodes, uint64_t eval_seed,
                  double* returns_host, double* mean, double* stderr_out) {
  return guarded([&] {
    require(cfg && dims && policy_host && norm && mean && stderr_out, "evaluate: null argument");
    evaluate_policy(*cfg, *dims, policy_host, norm->count, norm->mean, norm->m2, episodes,
                    eval_seed, returns_host, mean, stderr_out);
  });
}

int pqlg_k_evaluate_seq(const pqlg_config* cfg, const pqlg_task_dims* dims,
                        const float* policies_host, int n_policies, const pqlg_norm_stats* norm,
                        int episodes, uint64_t eval_seed, double* returns_host, double* mean,
                        double* stderr_out) {
  return guarded([&] {
    require(cfg && dims && policies_host && norm && returns_host && mean && stderr_out,
            "evaluate_seq: null argument");
    require(n_policies >= 1, "evaluate_seq: n_policies must be >= 1");
    std::vector<int> ps{dims->obs_dim};
    for (int l = 0; l < cfg->hidden_layers; ++l) ps.push_back(cfg->hidden);
    ps.push_back(cfg->algo == PQLG_ALGO_SAC ? 2 * dims->act_dim : dims->act_dim);
    const int64_t P = NetShape::make(ps).params;
    Evaluator ev(*cfg, *dims, episodes, eval_seed);
    for (int k = 0; k < n_policies; ++k)
      ev.run(policies_host + k * P, norm->count, norm->mean, norm->m2,
             returns_host + static_cast<int64_t>(k) * episodes, mean + k, stderr_out + k);
  });
}

int pqlg_actor_adopt_policy(pqlg_actor h, const float* flat, int64_t version) {
  return guarded([&] { h->a->adopt_policy(flat, version, false); });
}

int pqlg_actor_rollout_step(pqlg_actor h, pqlg_step_slice* out) {
  return guarded([&] { h->a->rollout_step(out); });
}

int pqlg_actor_rollout_n(pqlg_actor h, int n) {
  return guarded([&] { h->a->rollout_n(n); });
}

int pqlg_actor_norm(pqlg_actor h, int64_t* count, double* mean, double* m2) {
  return guarded([&] { h->a->norm(count, mean, m2); });
}

int pqlg_actor_policy_version(pqlg_actor h, int64_t* out) {
  return guarded([&] { *out = h->a->policy_version(); });
}

int pqlg_actor_read(pqlg_actor h, int what, void* out) {
  return guarded([&] { h->a->read_state(what, out); });
}

int pqlg_actor_read_slice(pqlg_actor h, float* obs, float* act, float* boot_obs, float* rew,
                          uint8_t* term, uint8_t* trunc) {
  return guarded([&] {
    require(h, "actor_read_slice: null handle");
    h->a->read_last_slice(obs, act, boot_obs, rew, term, trunc);
  });
}

int pqlg_actor_kernels_per_step(pqlg_actor h, int* out) {
  return guarded([&] { *out = h->a->kernels_per_step(); });
}

int pqlg_actor_time_steps(pqlg_actor h, int reps, char* out, int cap) {
  return guarded([&] {
    require(h && out && cap > 0, "actor_time_steps: null argument");
    copy_cstr(h->a->time_steps(reps), out, cap);
  });
}

int pqlg_env_create(int n_envs, int obs_dim, int act_dim, uint64_t seed, int max_episode_len,
                    int env_offset, float low, float high, void* stream, pqlg_env* out) {
  return guarded([&] {
    auto h = std::make_unique<pqlg_env_s>();
    h->e = std::make_unique<DeviceEnv>(n_envs, obs_dim, act_dim, seed, max_episode_len,
                                       env_offset, low, high);
    h->status.alloc(1);
    h->stream = static_cast<cudaStream_t>(stream);
    *out = h.release();
  });
}

int pqlg_env_destroy(pqlg_env h) {
  return guarded([&] { delete h; });
}

int pqlg_env_reset_all(pqlg_env h, float* obs_dev, int64_t ld) {
  return guarded([&] { h->e->reset(obs_dev, ld > 0 ? ld : h->e->D, h->stream); });
}

int pqlg_env_step(pqlg_env h, const float* act_dev, int64_t ld_act, float* next_obs_dev,
                  float* terminal_obs_dev, float* rew_dev, uint8_t* done_dev, uint8_t* trunc_dev,
                  int64_t ld_obs) {
  return guarded([&] {
    auto& e = *h->e;
    // term is (done && !trunc); the EnvBatch contract reports dones (vecenv.hpp:23-29)
    DevBuf<uint8_t> term(e.N);
    actor::StepOut o{next_obs_dev, terminal_obs_dev, rew_dev, term.p, trunc_dev, done_dev,
                     ld_obs > 0 ? ld_obs : e.D, h->status.p};
    e.step(act_dev, ld_act > 0 ? ld_act : e.A, o, h->stream);
    uint32_t st = 0;
    PQLG_CUDA(cudaMemcpyAsync(&st, h->status.p, 4, cudaMemcpyDeviceToHost, h->stream));
    PQLG_CUDA(cudaStreamSynchronize(h->stream));
    if (st) {
      PQLG_CUDA(cudaMemsetAsync(h->status.p, 0, 4, h->stream));
      PQLG_CUDA(cudaStreamSynchronize(h->stream));
      throw Error(PQLG_ENONFINITE, "step: non-finite action (upstream divergence)");
    }
  });
}

int pqlg_k_apply_noise(float* act_dev, int64_t ld, int n, int act_dim, const float* sigma_dev,
                       float low, float high, uint64_t* states_dev, void* stream) {
  return guarded([&] {
    launch(actor::noise_kernel, dim3((n + 127) / 128), dim3(128), 0, static_cast<cudaStream_t>(stream), act_dev, ld > 0 ? ld : act_dim, n, act_dim, sigma_dev, low, high, states_dev);
  });
}

int pqlg_k_normalizer_update(int64_t* count_dev, double* mean_dev, double* m2_dev,
                             const float* batch_dev, int64_t ld, int rows, int dim,
                             float* mean_f_dev, float* inv_f_dev, void* stream) {
  return guarded([&] {
    auto st = static_cast<cudaStream_t>(stream);
    if (rows == 0) return;  // normalizer.hpp:34
    DevBuf<double> part(static_cast<size_t>(actor::kNormBlocks) * dim * 2);
    DevBuf<int> ident(1);
    DevBuf<unsigned int> ticket(actor::norm_tickets(dim));
    DevBuf<double> shift(dim);
    const int64_t ldx = ld > 0 ? ld : dim;
    actor::NormState ns{count_dev, mean_dev, m2_dev, mean_f_dev, inv_f_dev, ident.p};
    actor::norm_update(batch_dev, ldx, rows, dim, part.p, shift.p, ticket.p, ns, st);
    PQLG_CUDA(cudaStreamSynchronize(st));
  });
}

}  // extern "C"

#ifdef PQLG_ENV_TRACE
extern "C" __attribute__((visibility("default"))) int pqlg_env_trace_set(unsigned long long* buf) {
  return pqlg::guarded([&] { PQLG_CUDA(cudaMemcpyToSymbol(pqlg::actor::g_env_trace, &buf, sizeof(buf))); });
}
#endif
