// P-learner: PolicyLearnerCore (proj/include/pql/runtime/learners.hpp:110-139,
// proj/src/runtime/learners.cpp:202-274) on one B200.
//
// One update = state sample (+ normalize) -> policy forward (masks + tanh kept)
// -> twin online critic replicas forward (masks only) -> pick min critic ->
// input gradient back through the picked critic (dgrad chain; the layer-0
// dgrad only for the action columns) -> policy head backward -> policy
// wgrad/dgrad chain -> fixed-order gradient reduction + fp64 norm -> clip +
// Adam (no Polyak for the policy).
#include "pdl.cuh"
#include <cstring>
#include <memory>
#include <random>
#include <vector>

#include "c51_kernels.cuh"
#include "comm.h"
#include "critic_kernels.cuh"
#include "dp_buckets.h"
#include "learner.h"
#include "optim.cuh"
#include "sac_host.h"

namespace pqlg {

PLearner::PLearner(const pqlg_config& cfg, const pqlg_task_dims& dims, uint64_t init_seed,
                   cudaStream_t st, pqlg_comm_s* comm)
    : cfg_(cfg), dims_(dims), stream_(st), comm_(comm) {
  if (comm_) {
    rank_ = comm_->rank;
    world_ = comm_->world;
  }
  if (!stream_) {
    PQLG_CUDA(cudaStreamCreateWithFlags(&owned_stream_, cudaStreamNonBlocking));
    stream_ = owned_stream_;
  }
  require(cfg.precision == PQLG_PREC_TF32 || cfg.precision == PQLG_PREC_3XTF32,
          "plearner: unknown precision");
  require(cfg.algo == PQLG_ALGO_DDPG || cfg.algo == PQLG_ALGO_C51 || cfg.algo == PQLG_ALGO_SAC,
          "plearner: unknown algo");
  dist_ = cfg.algo == PQLG_ALGO_C51;
  sac_ = cfg.algo == PQLG_ALGO_SAC;
  if (dist_) {
    require(cfg.n_atoms >= 2 && cfg.n_atoms <= c51::kMaxAtoms,
            "plearner: n_atoms must be in [2, 64]");
    require(cfg.vmin < cfg.vmax, "categorical head: bad support");
    L_ = cfg.n_atoms;
    Lp_ = static_cast<int>(round_up(L_, 4));
  }
  require(cfg.hidden_layers >= 1 && cfg.hidden >= 32 && cfg.hidden % 32 == 0,
          "plearner: hidden width must be a multiple of 32");
  D_ = dims.obs_dim;
  A_ = dims.act_dim;
  Ap_ = static_cast<int>(round_up(A_, 4));
  H_ = cfg.hidden;
  nh_ = cfg.hidden_layers;
  B_ = cfg.batch_size;
  Kp_ = static_cast<int>(round_up(D_ + A_, 4));
  require(A_ <= 32, "plearner: act_dim > 32 not supported by the policy head kernels");

  std::vector<int> qs{D_ + A_}, ps{D_};
  for (int i = 0; i < nh_; ++i) {
    qs.push_back(H_);
    ps.push_back(H_);
  }
  qs.push_back(L_);  // learners.cpp:206-209
  Ah_ = sac_ ? 2 * A_ : A_;  // GaussianPolicy head: [mean | log_std] (learners.cpp:20-22)
  Ahp_ = static_cast<int>(round_up(Ah_, 4));
  ps.push_back(Ah_);
  qnet_ = NetShape::make(qs);
  pnet_ = NetShape::make(ps);
  Ps_ = round_up(qnet_.params, 64);

  // critics_ (learners.cpp:202-205): CriticPair::create with the caller's
  // init_rng; the policy from make_rng(seed, init, 0) (learners.cpp:214).
  std::mt19937_64 init_rng(init_seed);
  std::vector<float> q1, q2, pol;
  init_orthogonal(qnet_, q1, init_rng, static_cast<float>(std::sqrt(2.0)), 1.0f);
  init_orthogonal(qnet_, q2, init_rng, static_cast<float>(std::sqrt(2.0)), 1.0f);
  std::mt19937_64 prng(rng::derive_seed(cfg.seed, rng::kInit, 0));
  init_orthogonal(pnet_, pol, prng, static_cast<float>(std::sqrt(2.0)), 1e-2f);
  q_.alloc(2 * Ps_);
  // [net | log_alpha] (log alpha starts at 0, learners.cpp:218); its Adam
  // moments sit at the same index of m_ / v_
  pol_.alloc(snapshot_len());
  m_.alloc(snapshot_len());
  v_.alloc(snapshot_len());
  grads_.alloc(pnet_.params);
  copy_sync(q_.p, q1.data(), q1.size() * 4, cudaMemcpyHostToDevice);
  copy_sync(q_.p + Ps_, q2.data(), q2.size() * 4, cudaMemcpyHostToDevice);
  copy_sync(pol_.p, pol.data(), pol.size() * 4, cudaMemcpyHostToDevice);

  states_ = std::make_unique<DeviceStates>(cfg.buffer_capacity, D_, stream_);
  norm_.init(D_);
  sampler_.alloc(1);
  // make_rng(seed, sample, 2) (learners.cpp:212); data-parallel rank r: 2 + 2r
  const uint64_t skey = rng::derive_seed(cfg.seed, rng::kSample, 2 + 2 * static_cast<uint64_t>(rank_));
  replay::SamplerState s0{skey, 0, 0, 0};
  copy_sync(sampler_.p, &s0, sizeof(s0), cudaMemcpyHostToDevice);
  mt_.seed(skey);
  idx_.alloc(B_);
  idx_host_.resize(B_);
  // eps stream make_rng(seed, sac, 2) (learners.cpp:213); rank r: 2 + 2r
  if (sac_)
    eps_.init(rng::derive_seed(cfg.seed, rng::kSac, 2 + 2 * static_cast<uint64_t>(rank_)),
              static_cast<int64_t>(B_) * A_);
  step_.alloc(1);
  auto tab = mlp::adam_bias_table(0.9, 0.999);
  bc_.alloc(tab.size());
  copy_sync(bc_.p, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
  status_.alloc(1);
  hbuf_.alloc(2);
  loss_.alloc(2);  // actor loss (+ pql_sac: mean log-prob for the alpha update)
  {
    gemm::PrecisionScope prec(cfg.precision == PQLG_PREC_3XTF32);
    build_update();
  }
  PQLG_CUDA(cudaDeviceSynchronize());
}

PLearner::~PLearner() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph2_exec_) cudaGraphExecDestroy(graph2_exec_);
  if (owned_stream_) {
    cudaStreamSynchronize(owned_stream_);
    cudaStreamDestroy(owned_stream_);
  }
}

namespace {
// Small row-wise kernels of the update (launched through closures).
}  // namespace

void PLearner::build_update() {
  const int B = B_, D = D_, A = A_, H = H_, nh = nh_, K0 = D + A;
  const int nt = mlp::hidden_slots(H);  // head-dot partial slots
  const int bnH = mlp::bn_for(H);
  const int mt = (B + 127) / 128;
  const int wpr = H / 32;
  const float* q[2] = {q_.p, q_.p + Ps_};

  X_.alloc(static_cast<size_t>(B) * Kp_);
  T_.alloc(static_cast<size_t>(B) * Ap_);
  dy_.alloc(static_cast<size_t>(B) * Ahp_);
  if (sac_) {
    sd_.alloc(static_cast<size_t>(B) * Ap_);
    logp_.alloc(B);
  }
  up_.alloc(2ull * B);
  part_.alloc(2ull * nt * B);
  pact_.resize(nh);
  pmask_.resize(nh);
  Gp_.resize(nh);
  for (int l = 0; l < nh; ++l) {
    pact_[l].alloc(static_cast<size_t>(B) * H);
    pmask_[l].alloc(static_cast<size_t>(B) * wpr);
    Gp_[l].alloc(static_cast<size_t>(B) * H);
  }
  for (int k = 0; k < 2; ++k) {
    cact_[k].resize(nh);
    cmask_[k].resize(nh);
    Gc_[k].resize(nh);
    for (int l = 0; l < nh; ++l) {
      cact_[k][l].alloc((l + 1 < nh || dist_) ? static_cast<size_t>(B) * H : 0);
      cmask_[k][l].alloc(static_cast<size_t>(B) * wpr);
      Gc_[k][l].alloc(static_cast<size_t>(B) * H);
    }
    dact_[k].alloc(static_cast<size_t>(B) * Ap_);
  }
  const int loss_blocks = (B + critic::kRowThreads - 1) / critic::kRowThreads;
  block_loss_.alloc(std::max((B + c51::kThreads - 1) / c51::kThreads,
                             2 * ((B + sac::kRowThreads - 1) / sac::kRowThreads)));
  if (dist_) {
    const auto z = c51_atoms(L_, static_cast<float>(cfg_.vmin), static_cast<float>(cfg_.vmax));
    atoms_.alloc(L_);
    copy_sync(atoms_.p, z.data(), L_ * 4, cudaMemcpyHostToDevice);
    probs_.alloc(2ull * B * Lp_);
    ev_.alloc(2ull * B);
    up51_.alloc(2ull * B * Lp_);
    for (int k = 0; k < 2; ++k) heads_[k].init(q[k] + qnet_.w_off[nh], H, L_);
    // critic snapshots are adopted between updates: refresh the padded heads first
    const WeightMirror* hm = heads_.data();
    steps_.push_back([hm](cudaStream_t st) { refresh_mirrors(hm, 2, st); });
  }
  loss_counter_.alloc(1);

  // the policy head's W in the head kernel's fragment order, packed from the
  // previous update's Adam result (a tiny launch the early-starting sample
  // overlaps)
  {
    const int Ah = Ah_;  // A, or 2A ([mean | log_std]) for pql_sac
    wpack_.alloc(static_cast<size_t>(mlp::head_pack_elems(Ah, H)) * 4);
    const bool x3 = gemm::build_x3();
    steps_.push_back([this, Ah, H, nh, x3](cudaStream_t st) {
      mlp::head_pack(pol_.p + pnet_.w_off[nh], Ah, H, Ah, reinterpret_cast<float4*>(wpack_.p), x3,
                     st);
    });
  }
  // ------------------------------------------------- sample + normalize
  steps_.push_back([this, B](cudaStream_t st) {
    const uint64_t* idx = mt_mode_ ? idx_.p : nullptr;
    launch_state_sample(*states_, norm_.view(), X_.p, Kp_, sampler_.p, idx, B, st, capture_);
  });
  if (sac_) {  // eps of the reparameterised actions (learners.cpp:247-249)
    steps_.push_back([this](cudaStream_t st) {
      if (mt_mode_) eps_.fill_mt(st);
      else eps_.fork(st);  // parallel branch, joined before the sampling finish
    });
  }

  // -------------------------------------------------------- policy forward
  {
    const float* in = X_.p;
    int64_t ld = Kp_;
    int K = D;
    for (int l = 0; l < nh; ++l) {
      epi::Hidden e{};
      e.bias[0] = e.bias[1] = pol_.p + pnet_.b_off[l];
      e.mask[0] = e.mask[1] = pmask_[l].p;
      e.ld_mask = B;  // word-major masks
      e.bn = bnH;
      e.M = B;
      e.N = H;
      e.store = 1;
      const float* W = pol_.p + pnet_.w_off[l];
      steps_.push_back(mlp::fwd(in, in, ld, W, W, B, H, K, 1, e, 0, pact_[l].p, pact_[l].p, H));
      in = pact_[l].p;
      ld = H;
      K = H;
    }
    head_.init(pol_.p + pnet_.w_off[nh], H, Ah_);
    head_.refresh(stream_);
    const float* Wh = pol_.p + pnet_.w_off[nh];
    if (sac_) {
      // s = policy.sample(states, eps) (sac.hpp:77): actions, log-probs, and
      // tanh(pre) / std kept for the backward
      head::RowsArgs base{};
      base.wpack = reinterpret_cast<const float4*>(wpack_.p);
      steps_.push_back(mlp::head_raw_step(head_split_, in, ld, Wh, B, Ah_, H, base));
      sac::GaussArgs g{};
      g.bias = pol_.p + pnet_.b_off[nh];
      g.eps = eps_.out.p;
      g.act = X_.p + D;
      g.ld_act = Kp_;
      g.logp = logp_.p;
      g.tanh_out = T_.p;
      g.sd_out = sd_.p;
      g.ld_aux = Ap_;
      g.mid = (dims_.low + dims_.high) / 2.0f;
      g.half = (dims_.high - dims_.low) / 2.0f;
      steps_.push_back([this](cudaStream_t st) { eps_.join(st); });
      steps_.push_back(gauss_finish_step(head_split_, g, B, A));
    } else {
      head::RowsArgs ph{};
      ph.bias = pol_.p + pnet_.b_off[nh];
      ph.out = X_.p + D;  // critic input [norm(s) | pi(s)]
      ph.ld_out = Kp_;
      ph.tanh_out = T_.p;
      ph.ld_tanh = Ap_;
      ph.mid = (dims_.low + dims_.high) / 2.0f;
      ph.half = (dims_.high - dims_.low) / 2.0f;
      ph.wpack = reinterpret_cast<const float4*>(wpack_.p);
      steps_.push_back(mlp::head_squash_step(ph, in, ld, Wh, B, A, H));
    }
  }

  // ------------------------------------------ twin critic replicas forward
  for (int l = 0; l < nh; ++l) {
    epi::Hidden e{};
    for (int k = 0; k < 2; ++k) {
      e.bias[k] = q[k] + qnet_.b_off[l];
      e.mask[k] = cmask_[k][l].p;
    }
    e.ld_mask = B;  // word-major masks
    e.bn = bnH;
    e.M = B;
    e.N = H;
    const bool last = l + 1 == nh;
    e.store = (last && !dist_) ? 0 : 3;
    if (last && !dist_) {
      for (int k = 0; k < 2; ++k) {
        e.w_head[k] = q[k] + qnet_.w_off[nh];
        e.partial[k] = part_.p + static_cast<size_t>(k) * nt * B;
      }
      e.ld_part = B;
      e.n_slots = nt;
    }
    const float* a0 = l == 0 ? X_.p : cact_[0][l - 1].p;
    const float* a1 = l == 0 ? X_.p : cact_[1][l - 1].p;
    const int64_t lda = l == 0 ? Kp_ : H;
    const int K = l == 0 ? K0 : H;
    const bool st = !last || dist_;
    steps_.push_back(mlp::fwd(a0, a1, lda, q[0] + qnet_.w_off[l], q[1] + qnet_.w_off[l], B, H, K,
                              2, e, 0, st ? cact_[0][l].p : nullptr,
                              st ? cact_[1][l].p : nullptr, H));
  }
  if (dist_) {
    // categorical heads at (s, pi(s)): softmax + expected value (c51.hpp:175-187)
    epi::C51Head ch{};
    for (int k = 0; k < 2; ++k) {
      ch.bias[k] = q[k] + qnet_.b_off[nh];
      ch.probs[k] = probs_.p + static_cast<size_t>(k) * B * Lp_;
      ch.ev[k] = ev_.p + static_cast<size_t>(k) * B;
    }
    ch.ld = Lp_;
    ch.atoms = atoms_.p;
    ch.M = B;
    ch.L = L_;
    steps_.push_back(mlp::fwd(cact_[0][nh - 1].p, cact_[1][nh - 1].p, H, heads_[0].ptr(),
                              heads_[1].ptr(), B, L_, H, 2, ch, heads_[0].stride()));
  }
  // ------------------------------------------------ min critic + upstream
  if (dist_) {
    c51::ActorPickArgs a{};
    for (int k = 0; k < 2; ++k) {
      a.po[k] = probs_.p + static_cast<size_t>(k) * B * Lp_;
      a.ev[k] = ev_.p + static_cast<size_t>(k) * B;
    }
    a.ld = Lp_;
    a.atoms = atoms_.p;
    a.L = L_;
    a.up = up51_.p;
    a.step = step_.p;
    a.block_loss = block_loss_.p;
    a.counter = loss_counter_.p;
    a.loss_out = loss_.p;
    a.status = status_.p;
    a.B = B;
    a.Bg = B * world_;
    const int blocks = (B + c51::kThreads - 1) / c51::kThreads;
    steps_.push_back([a, blocks](cudaStream_t st) {
      launch(c51::c51_actor_pick_kernel, dim3(blocks), dim3(c51::kThreads), 0, st, a);
    });
  } else if (sac_) {
    // sac_actor_loss rows (sac.hpp:86-96): loss, mean log-prob, upstream
    sac::PickArgs a{};
    a.partial = part_.p;
    a.ld = B;
    a.n_tiles = nt;
    a.q1 = q[0];
    a.q2 = q[1];
    a.head_b_off = qnet_.b_off[nh];
    a.logp = logp_.p;
    a.log_alpha = pol_.p + pnet_.params;
    a.up = up_.p;
    a.step = step_.p;
    a.block_part = block_loss_.p;
    a.counter = loss_counter_.p;
    a.out = loss_.p;
    a.status = status_.p;
    a.B = B;
    a.Bg = B * world_;
    const int blocks = (B + sac::kRowThreads - 1) / sac::kRowThreads;
    steps_.push_back([a, blocks](cudaStream_t st) {
      launch(sac::sac_pick_kernel, dim3(blocks), dim3(sac::kRowThreads), 0, st, a);
    });
  } else {
    critic::LossArgs a{};
    a.partial = part_.p;
    a.ld = B;
    a.n_tiles = nt;
    a.q1 = q[0];
    a.q2 = q[1];
    a.head_b_off = qnet_.b_off[nh];
    a.up = up_.p;
    a.block_loss = block_loss_.p;
    a.counter = loss_counter_.p;
    a.loss_out = loss_.p;
    a.status = status_.p;
    a.step = step_.p;  // Adam step of the policy, advanced once per update
    a.B = B;
    a.Bg = B * world_;
    steps_.push_back([a, loss_blocks](cudaStream_t st) {
      launch(critic::actor_pick_kernel, dim3(loss_blocks), dim3(critic::kRowThreads), 0, st, a);
    });
  }
  // --------------------------------- input gradient through the critics
  if (dist_) {
    // backward_input_only through the categorical heads: G = (up W^T) * mask
    epi::DgradMask dm{};
    for (int k = 0; k < 2; ++k) dm.mask[k] = cmask_[k][nh - 1].p;
    dm.ld_mask = B;  // word-major masks
    dm.bn = bnH;
    dm.M = B;
    dm.N = H;
    steps_.push_back(mlp::dgrad(up51_.p, up51_.p + static_cast<size_t>(B) * Lp_, Lp_,
                                heads_[0].ptr(), heads_[1].ptr(), heads_[0].stride(), B, H, L_, 2,
                                dm, Gc_[0][nh - 1].p, Gc_[1][nh - 1].p, H));
  } else {
    critic::HeadInputGradArgs a{};
    a.up = up_.p;
    for (int k = 0; k < 2; ++k) {
      a.mask[k] = cmask_[k][nh - 1].p;
      a.w[k] = q[k] + qnet_.w_off[nh];
      a.G[k] = Gc_[k][nh - 1].p;
    }
    a.B = B;
    a.H = H;
    const int blocks = 4 * mlp::kSMs;
    steps_.push_back([a, blocks](cudaStream_t st) {
      launch(critic::head_input_grad_kernel, dim3(dim3(blocks, 2)), dim3(256), 0, st, a);
    });
  }
  for (int l = nh - 1; l >= 1; --l) {
    epi::DgradMask dm{};
    for (int k = 0; k < 2; ++k) dm.mask[k] = cmask_[k][l - 1].p;
    dm.ld_mask = B;  // word-major masks
    dm.bn = bnH;
    dm.M = B;
    dm.N = H;
    steps_.push_back(mlp::dgrad(Gc_[0][l].p, Gc_[1][l].p, H, q[0] + qnet_.w_off[l],
                                q[1] + qnet_.w_off[l], H, B, H, H, 2, dm, Gc_[0][l - 1].p,
                                Gc_[1][l - 1].p, H));
  }
  {
    // layer-0 dgrad restricted to the action columns: rows D..D+A-1 of W0
    epi::Store s{};
    s.out[0] = dact_[0].p;
    s.out[1] = dact_[1].p;
    s.ld_out = Ap_;
    s.M = B;
    s.N = A;
    steps_.push_back(mlp::dgrad(Gc_[0][0].p, Gc_[1][0].p, H, q[0] + qnet_.w_off[0] + D * H,
                                q[1] + qnet_.w_off[0] + D * H, H, B, A, H, 2, s));
  }
  // ------------------------------------------------- policy head backward
  const int ptiles = (B + 7) / 8;  // policy-head backward tiles (8 rows, one warp each)
  head_db_.alloc(static_cast<size_t>(ptiles) * Ah_);
  if (sac_) {
    // GaussianPolicy::backward's dy (policy.hpp:127-150), dlogp = alpha / B
    sac::HeadBwdArgs a{};
    a.dact1 = dact_[0].p;
    a.dact2 = dact_[1].p;
    a.ld_dact = Ap_;
    a.tanh_in = T_.p;
    a.sd_in = sd_.p;
    a.ld_aux = Ap_;
    a.eps = eps_.out.p;
    a.log_alpha = pol_.p + pnet_.params;
    a.dy = dy_.p;
    a.ld_dy = Ahp_;
    a.db_part = head_db_.p;
    a.half = (dims_.high - dims_.low) / 2.0f;
    a.B = B;
    a.A = A;
    a.Bg = B * world_;
    a.rows_per_tile = 8;
    steps_.push_back([a, ptiles](cudaStream_t st) {
      launch(sac::sac_head_backward_kernel, dim3(ptiles), dim3(32), 0, st, a);
    });
  } else {
    critic::PolicyHeadBwdArgs a{};
    a.dact1 = dact_[0].p;
    a.dact2 = dact_[1].p;
    a.ld_dact = Ap_;
    a.t = T_.p;
    a.ld_t = Ap_;
    a.dy = dy_.p;
    a.ld_dy = Ap_;
    a.db_part = head_db_.p;
    a.half = (dims_.high - dims_.low) / 2.0f;
    a.B = B;
    a.A = A;
    a.rows_per_tile = 8;
    steps_.push_back([a, ptiles](cudaStream_t st) {
      launch(critic::policy_head_backward_kernel, dim3(ptiles), dim3(32), 0, st, a);
    });
  }
  // ----------------------------------------------------- policy backward
  wpart_.resize(nh + 1);
  colsum_.resize(nh);
  wsplits_.resize(nh + 1);
  for (int l = 0; l <= nh; ++l) {
    const int in = l == 0 ? D : H;
    const int out = l == nh ? Ah_ : H;
    const int ldo = l == nh ? Ahp_ : H;
    wsplits_[l] = mlp::wgrad_splits(in, out, B, 1);
    wpart_[l].alloc(static_cast<size_t>(wsplits_[l]) * in * ldo);
    if (l < nh) colsum_[l].alloc(static_cast<size_t>(mt) * H);
  }
  // gradient segments of policy layer l (l == nh: the head), see VLearner
  auto layer_segs = [&](int l) {
    std::vector<optim::Segment> v;
    if (l == nh) {
      optim::Segment wh{pnet_.w_off[nh], static_cast<int64_t>(H) * Ah_, wpart_[nh].p, 0,
                        wsplits_[nh], static_cast<int64_t>(H) * Ahp_};
      wh.cols = Ah_;
      wh.ld_src = Ahp_;
      v.push_back(wh);
      v.push_back(optim::Segment{pnet_.b_off[nh], Ah_, head_db_.p, 0, ptiles, Ah_});
    } else {
      const int in = l == 0 ? D : H;
      v.push_back(optim::Segment{pnet_.w_off[l], static_cast<int64_t>(in) * H, wpart_[l].p, 0,
                                 wsplits_[l], static_cast<int64_t>(in) * H});
      v.push_back(optim::Segment{pnet_.b_off[l], H, colsum_[l].p, 0, mt, H});
    }
    return v;
  };
  // data parallel: bucketed reduce + all-reduce per layer (dp_buckets.h); the
  // head bucket carries the loss (and pql_sac's mean log-prob, loss_[1])
  if (comm_) dp_ = std::make_unique<DpBuckets>(comm_, grads_.p, 1, pnet_.params);
  auto dp_bucket = [&](int l) {
    const int64_t lo = pnet_.w_off[l], hi = pnet_.b_off[l] + pnet_.sizes[l + 1];
    const bool head = l == nh;
    steps_.push_back(dp_->bucket(layer_segs(l), lo, hi, head ? loss_.p : nullptr,
                                 head ? (sac_ ? 2 : 1) : 0));
  };
  // head layer: dW_nh = act_{nh-1}^T dy ; G_{nh-1} = (dy W_nh^T) * mask
  steps_.push_back(mlp::wgrad(pact_[nh - 1].p, pact_[nh - 1].p, H, dy_.p, dy_.p, Ahp_, H, Ah_, B,
                              1, wsplits_[nh], epi::Partial{}, wpart_[nh].p, Ahp_));
  if (dp_) dp_bucket(nh);
  {
    epi::DgradMask dm{};
    dm.mask[0] = dm.mask[1] = pmask_[nh - 1].p;
    dm.ld_mask = B;  // word-major masks
    dm.colsum = colsum_[nh - 1].p;
    dm.ld_cs = H;
    dm.m_tiles = mt;
    dm.bn = bnH;
    dm.M = B;
    dm.N = H;
    steps_.push_back(mlp::dgrad(dy_.p, dy_.p, Ahp_, head_.ptr(), head_.ptr(), head_.stride(), B,
                                H, Ah_, 1, dm, Gp_[nh - 1].p, Gp_[nh - 1].p, H));
  }
  for (int l = nh - 1; l >= 0; --l) {
    const int in = l == 0 ? D : H;
    const float* h = l == 0 ? X_.p : pact_[l - 1].p;
    const int64_t ldh = l == 0 ? Kp_ : H;
    steps_.push_back(mlp::wgrad(h, h, ldh, Gp_[l].p, Gp_[l].p, H, in, H, B, 1, wsplits_[l],
                                epi::Partial{}, wpart_[l].p));
    if (dp_) dp_bucket(l);
    if (l > 0) {
      epi::DgradMask dm{};
      dm.mask[0] = dm.mask[1] = pmask_[l - 1].p;
      dm.ld_mask = B;  // word-major masks
      dm.colsum = colsum_[l - 1].p;
      dm.ld_cs = H;
      dm.m_tiles = mt;
      dm.bn = bnH;
      dm.M = B;
      dm.N = H;
      const float* W = pol_.p + pnet_.w_off[l];
      steps_.push_back(mlp::dgrad(Gp_[l].p, Gp_[l].p, H, W, W, H, B, H, H, 1, dm,
                                  Gp_[l - 1].p, Gp_[l - 1].p, H));
    }
  }
  // ------------------------------------- reduction + clip + Adam (policy)
  {
    optim::FinalizeArgs f{};
    int s = 0;
    if (comm_) {  // the buckets hold the all-reduced gradient: norm + clip pass
      steps_.push_back(dp_->join());
      f.seg[s++] = optim::Segment{0, pnet_.params, grads_.p, 0, 1, 0};
      f.check = loss_.p;
    } else {
      for (int l = 0; l <= nh; ++l)
        for (const auto& sg : layer_segs(l)) f.seg[s++] = sg;
    }
    require(s <= optim::kMaxSegments, "plearner: too many layers");
    f.n_seg = s;
    f.total = pnet_.params;
    f.gstride = pnet_.params;
    f.grads = grads_.p;
    const int fb = optim::plan_finalize(f);
    block_sq_.alloc(fb);
    fin_counter_.alloc(1);
    scale_.alloc(1);
    f.block_sq = block_sq_.p;
    f.counter = fin_counter_.p;
    f.scale = scale_.p;
    f.status = status_.p;
    f.max_norm = 0.5f;
    steps_.push_back([f, fb](cudaStream_t st) {
      launch(optim::finalize_kernel, dim3(dim3(fb, 1)), dim3(optim::kFinalizeThreads), 0, st, f);
    });
    optim::AdamArgs a{};
    a.p = pol_.p;
    a.g = grads_.p;
    a.m = m_.p;
    a.v = v_.p;
    a.target = nullptr;
    a.n = pnet_.params;
    a.gstride = pnet_.params;
    a.scale = scale_.p;
    a.status = status_.p;
    a.step = step_.p;
    a.bc = bc_.p;
    a.bc_len = static_cast<int64_t>(bc_.n);
    a.lr = static_cast<float>(cfg_.lr_actor);
    a.beta1 = 0.9f;
    a.beta2 = 0.999f;
    a.eps = 1e-8f;
    a.tau = 0.0f;
    if (sac_) {  // alpha step (learners.cpp:254-256), Adam state at index params
      a.alpha.log_alpha = pol_.p + pnet_.params;
      a.alpha.m = m_.p + pnet_.params;
      a.alpha.v = v_.p + pnet_.params;
      a.alpha.mean_logp = loss_.p + 1;
      a.alpha.target_entropy = -static_cast<float>(A);
      a.alpha.lr = static_cast<float>(cfg_.lr_actor);
    }
    const int blocks = static_cast<int>(std::min<int64_t>(4 * mlp::kSMs, (pnet_.params + 255) / 256));
    steps_.push_back([a, blocks](cudaStream_t st) {
      launch(optim::adam_polyak_kernel, dim3(dim3(blocks, 1)), dim3(256), 0, st, a);
    });
  }
  // the padded head mirror follows the updated policy
  steps_.push_back([this](cudaStream_t st) { head_.refresh(st); });
}

void PLearner::adopt_critics(const float* q1, const float* q2, int64_t version) {
  if (version < critic_version_) return;  // learners.cpp:222-227
  const int64_t P = qnet_.params;
  PQLG_CUDA(cudaMemcpyAsync(q_.p, q1, P * 4, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(q_.p + Ps_, q2, P * 4, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
  critic_version_ = version;
}

void PLearner::adopt_critics_device(const float* q1, const float* q2, int64_t version) {
  if (version < critic_version_) return;
  const int64_t P = qnet_.params;
  PQLG_CUDA(cudaMemcpyAsync(q_.p, q1, P * 4, cudaMemcpyDeviceToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(q_.p + Ps_, q2, P * 4, cudaMemcpyDeviceToDevice, stream_));
  critic_version_ = version;
}

void PLearner::adopt_norm(int64_t count, const double* mean, const double* m2) {
  // an empty NormStats (count <= 1: identity, normalizer.hpp:18-19) may come
  // without vectors, as a default-constructed fa::NormStats does
  require(count <= 1 || (mean && m2), "adopt_norm: mean / m2 required when count > 1");
  norm_count_ = count;
  if (mean && m2) {
    norm_mean_.assign(mean, mean + D_);
    norm_m2_.assign(m2, m2 + D_);
  } else {
    norm_mean_.assign(D_, 0.0);
    norm_m2_.assign(D_, 0.0);
  }
  norm_.set(count, norm_mean_.data(), norm_m2_.data(), stream_);
}

void PLearner::ingest(const float* states, int64_t ld, uint64_t n) {
  states_->insert(states, ld, n, stream_);
}

// PolicyLearnerCore::ingest(const MatF&) (learners.hpp:121) from host rows.
void PLearner::ingest_host(const float* states, int64_t ld, uint64_t n) {
  if (n == 0) return;
  require(states != nullptr, "ingest: null states");
  const int64_t Dp = round_up(D_, 4);
  if (in_f_.n < n * Dp) in_f_.alloc(n * Dp);
  PQLG_CUDA(cudaMemcpy2DAsync(in_f_.p, Dp * 4, states, ld * 4, D_ * 4, n, cudaMemcpyHostToDevice,
                              stream_));
  ingest(in_f_.p, Dp, n);
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

bool PLearner::ready(int64_t c_a) {
  return c_a >= cfg_.warm_up && states_->size() >= static_cast<uint64_t>(B_);
}

void PLearner::enqueue() {
  const int skip = skip_step();
  for (size_t i = 0; i < steps_.size(); ++i)
    if (static_cast<int>(i) != skip) steps_[i](stream_);
}

std::string PLearner::time_update(int reps) {
  require(!mt_mode_, "time_update: graph replay needs the Philox sampler");
  if (states_->size() < static_cast<uint64_t>(B_))
    throw Error(PQLG_NOT_READY, "policy update before state warm-up");
  return time_in_graph([&] { enqueue(); }, stream_, reps);
}

int PLearner::check_status() {
  uint32_t st = 0;
  PQLG_CUDA(cudaMemcpyAsync(&st, status_.p, 4, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
  if (st) {
    PQLG_CUDA(cudaMemsetAsync(status_.p, 0, 4, stream_));
    return PQLG_ENONFINITE;
  }
  return PQLG_OK;
}

float PLearner::update() {
  if (states_->size() < static_cast<uint64_t>(B_))
    throw Error(PQLG_NOT_READY, "policy update before state warm-up");
  if (mt_mode_ || eager_updates()) {
    const uint64_t count = states_->size();
    std::uniform_int_distribution<std::size_t> pick(0, count - 1);
    if (mt_mode_) {
      for (int r = 0; r < B_; ++r) idx_host_[r] = pick(mt_);
      PQLG_CUDA(cudaMemcpyAsync(idx_.p, idx_host_.data(), B_ * sizeof(uint64_t),
                                cudaMemcpyHostToDevice, stream_));
    }
    enqueue();
  } else {
    update_n(1);  // one replay of the captured update graph
  }
  // loss + status into pinned memory, one synchronisation
  PQLG_CUDA(cudaMemcpyAsync(&hbuf_.p[0], loss_.p, 4, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaMemcpyAsync(&hbuf_.p[1], status_.p, 4, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
  if (hbuf_.p[1] != 0u) {
    PQLG_CUDA(cudaMemsetAsync(status_.p, 0, 4, stream_));
    throw Error(PQLG_ENONFINITE, "ddpg actor update: non-finite");
  }
  float loss;
  std::memcpy(&loss, &hbuf_.p[0], 4);
  return loss;
}

int PLearner::kernels_per_update() {
  if (kpu_ == 0) {
    const uint64_t before = g_launches.load();
    cudaGraph_t g;
    PQLG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
    enqueue();
    PQLG_CUDA(cudaStreamEndCapture(stream_, &g));
    cudaGraphDestroy(g);
    kpu_ = static_cast<int>(g_launches.load() - before);
    g_launches.fetch_sub(kpu_);
  }
  return kpu_;
}

void PLearner::update_n(int n) {
  require(!mt_mode_, "update_n: graph replay needs the Philox sampler");
  if (states_->size() < static_cast<uint64_t>(B_))
    throw Error(PQLG_NOT_READY, "policy update before state warm-up");
  if (!graph_exec_) {
    kernels_per_update();
    capture_ = true;
    for (int reps = 1; reps <= 2; ++reps) {
      cudaGraph_t g;
      PQLG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
      for (int r = 0; r < reps; ++r) enqueue();
      PQLG_CUDA(cudaStreamEndCapture(stream_, &g));
      g_launches.fetch_sub(static_cast<uint64_t>(reps) * kpu_);
      PQLG_CUDA(cudaGraphInstantiate(reps == 1 ? &graph_exec_ : &graph2_exec_, g, 0));
      cudaGraphDestroy(g);
    }
    capture_ = false;
  }
  for (int i = 0; i + 1 < n; i += 2) PQLG_CUDA(cudaGraphLaunch(graph2_exec_, stream_));
  if (n % 2) PQLG_CUDA(cudaGraphLaunch(graph_exec_, stream_));
  count_launch(static_cast<uint64_t>(n) * kpu_);
}

float PLearner::last_loss() {
  float loss = 0.0f;
  PQLG_CUDA(cudaMemcpyAsync(&loss, loss_.p, 4, cudaMemcpyDeviceToHost, stream_));
  if (check_status() != PQLG_OK) throw Error(PQLG_ENONFINITE, "ddpg actor update: non-finite");
  return loss;
}

// which: 0 policy, 1 critic replica q1, 2 critic replica q2
void PLearner::get_params(int which, float* out) {
  const float* src = which == 0 ? pol_.p : (which == 1 ? q_.p : q_.p + Ps_);
  const int64_t n = param_count(which);
  require(which >= 0 && which <= 2, "get_params: which must be 0..2");
  PQLG_CUDA(cudaMemcpyAsync(out, src, n * 4, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

void PLearner::set_params(int which, const float* flat) {
  require(which >= 0 && which <= 2, "set_params: which must be 0..2");
  float* dst = which == 0 ? pol_.p : (which == 1 ? q_.p : q_.p + Ps_);
  PQLG_CUDA(cudaMemcpyAsync(dst, flat, param_count(which) * 4, cudaMemcpyHostToDevice, stream_));
  if (which == 0) head_.refresh(stream_);
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

int64_t PLearner::param_count(int which) const {
  return which == 0 ? pnet_.params : qnet_.params;
}

float PLearner::log_alpha() {
  float v = 0.0f;
  if (sac_) {
    PQLG_CUDA(cudaMemcpyAsync(&v, pol_.p + pnet_.params, 4, cudaMemcpyDeviceToHost, stream_));
    PQLG_CUDA(cudaStreamSynchronize(stream_));
  }
  return v;
}

}  // namespace pqlg

// ------------------------------------------------------------------ C ABI
struct pqlg_plearner_s {
  std::unique_ptr<pqlg::PLearner> p;
  cudaEvent_t ev = nullptr;  // record_event
  ~pqlg_plearner_s() {
    if (ev) cudaEventDestroy(ev);
  }
};

namespace pqlg {
PLearner* plearner_of(pqlg_plearner h) {
  require(h != nullptr, "null plearner handle");
  return h->p.get();
}
}  // namespace pqlg

using namespace pqlg;

extern "C" {

int pqlg_plearner_create(const pqlg_config* cfg, const pqlg_task_dims* dims,
                         uint64_t init_rng_seed, void* stream, pqlg_plearner* out) {
  return guarded([&] {
    require(cfg && dims && out, "plearner_create: null argument");
    auto h = std::make_unique<pqlg_plearner_s>();
    h->p = std::make_unique<PLearner>(*cfg, *dims, init_rng_seed,
                                      static_cast<cudaStream_t>(stream));
    *out = h.release();
  });
}

int pqlg_plearner_create_dp(const pqlg_config* cfg, const pqlg_task_dims* dims,
                            uint64_t init_rng_seed, pqlg_comm comm, void* stream,
                            pqlg_plearner* out) {
  return guarded([&] {
    require(cfg && dims && out && comm, "plearner_create_dp: null argument");
    auto h = std::make_unique<pqlg_plearner_s>();
    h->p = std::make_unique<PLearner>(*cfg, *dims, init_rng_seed,
                                      static_cast<cudaStream_t>(stream), comm);
    *out = h.release();
  });
}

int pqlg_plearner_wait_event(pqlg_plearner h, void* event) {
  return guarded([&] {
    require(h && event, "plearner_wait_event: null argument");
    PQLG_CUDA(cudaStreamWaitEvent(h->p->stream(), static_cast<cudaEvent_t>(event), 0));
  });
}

int pqlg_plearner_record_event(pqlg_plearner h, void** event_out) {
  return guarded([&] {
    require(h && event_out, "plearner_record_event: null argument");
    if (!h->ev) PQLG_CUDA(cudaEventCreateWithFlags(&h->ev, cudaEventDisableTiming));
    PQLG_CUDA(cudaEventRecord(h->ev, h->p->stream()));
    *event_out = h->ev;
  });
}

int pqlg_plearner_destroy(pqlg_plearner h) {
  return guarded([&] { delete h; });
}

int pqlg_plearner_adopt_critics(pqlg_plearner h, const float* q1, const float* q2,
                                int64_t version) {
  return guarded([&] { h->p->adopt_critics(q1, q2, version); });
}

int pqlg_plearner_adopt_norm(pqlg_plearner h, const pqlg_norm_stats* n) {
  return guarded([&] { h->p->adopt_norm(n->count, n->mean, n->m2); });
}

int pqlg_plearner_ingest(pqlg_plearner h, const float* states_dev, int64_t ld, uint64_t n) {
  return guarded([&] { h->p->ingest(states_dev, ld > 0 ? ld : h->p->obs_dim(), n); });
}

int pqlg_plearner_ingest_host(pqlg_plearner h, const float* states_host, int64_t ld, uint64_t n) {
  return guarded([&] { h->p->ingest_host(states_host, ld > 0 ? ld : h->p->obs_dim(), n); });
}

int pqlg_plearner_ready(pqlg_plearner h, int64_t c_a, int* ready) {
  return guarded([&] { *ready = h->p->ready(c_a) ? 1 : 0; });
}

int pqlg_plearner_update(pqlg_plearner h, float* loss) {
  return guarded([&] {
    const float l = h->p->update();
    if (loss) *loss = l;
  });
}

int pqlg_plearner_update_n(pqlg_plearner h, int n) {
  return guarded([&] { h->p->update_n(n); });
}

int pqlg_plearner_last_loss(pqlg_plearner h, float* loss) {
  return guarded([&] { *loss = h->p->last_loss(); });
}

int pqlg_plearner_snapshot(pqlg_plearner h, float* flat) {
  return guarded([&] { h->p->get_params(0, flat); });
}

int pqlg_plearner_get_params(pqlg_plearner h, int which, float* flat) {
  return guarded([&] { h->p->get_params(which, flat); });
}

int pqlg_plearner_set_params(pqlg_plearner h, int which, const float* flat) {
  return guarded([&] { h->p->set_params(which, flat); });
}

int pqlg_plearner_param_count(pqlg_plearner h, int which, int64_t* out) {
  return guarded([&] { *out = h->p->param_count(which); });
}

int pqlg_plearner_log_alpha(pqlg_plearner h, float* out) {
  return guarded([&] { *out = h->p->log_alpha(); });
}

int pqlg_plearner_buffer_size(pqlg_plearner h, uint64_t* out) {
  return guarded([&] { *out = h->p->buffer_size(); });
}

int pqlg_plearner_set_sampler(pqlg_plearner h, int mode) {
  return guarded([&] {
    require(mode == PQLG_RNG_PHILOX || mode == PQLG_RNG_INDICES, "set_sampler: bad mode");
    h->p->set_mt_mode(mode == PQLG_RNG_INDICES);
  });
}

int pqlg_plearner_kernels_per_update(pqlg_plearner h, int* out) {
  return guarded([&] { *out = h->p->kernels_per_update(); });
}

int pqlg_plearner_time_update(pqlg_plearner h, int reps, char* out, int cap) {
  return guarded([&] {
    require(h && out && cap > 0, "plearner_time_update: null argument");
    copy_cstr(h->p->time_update(reps), out, cap);
  });
}

}  // extern "C"
