// V-learner: CriticLearnerCore (proj/include/pql/runtime/learners.hpp:77-106,
// proj/src/runtime/learners.cpp:122-196) on one B200.
//
// One update = sample -> target policy -> twin target critics -> TD target ->
// twin online critics -> loss -> backward (head, then wgrad/dgrad per layer)
// -> fixed-order gradient reduction + fp64 norm -> fused clip/Adam/Polyak.
// Every step is a pre-built launch; update_n() replays them from a CUDA graph.
#include <algorithm>
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

using mlp::Step;

VLearner::VLearner(const pqlg_config& cfg, const pqlg_task_dims& dims, uint64_t init_seed,
                   cudaStream_t st, pqlg_comm_s* comm)
    : cfg_(cfg), dims_(dims), stream_(st), comm_(comm) {
  if (comm_) {
    rank_ = comm_->rank;
    world_ = comm_->world;
  }
  if (!stream_) {  // the legacy default stream cannot be graph-captured
    PQLG_CUDA(cudaStreamCreateWithFlags(&owned_stream_, cudaStreamNonBlocking));
    stream_ = owned_stream_;
  }
  st = stream_;
  require(cfg.precision == PQLG_PREC_TF32 || cfg.precision == PQLG_PREC_3XTF32,
          "vlearner: unknown precision");
  require(cfg.algo == PQLG_ALGO_DDPG || cfg.algo == PQLG_ALGO_C51 || cfg.algo == PQLG_ALGO_SAC,
          "vlearner: unknown algo");
  dist_ = cfg.algo == PQLG_ALGO_C51;
  sac_ = cfg.algo == PQLG_ALGO_SAC;
  require(!sac_ || dims.act_dim <= 32, "vlearner: pql_sac needs act_dim <= 32");
  if (dist_) {
    // CategoricalHead::create (c51.hpp:21-27) validation
    require(cfg.n_atoms >= 2 && cfg.n_atoms <= c51::kMaxAtoms,
            "vlearner: n_atoms must be in [2, 64]");
    require(cfg.vmin < cfg.vmax, "categorical head: bad support");
    L_ = cfg.n_atoms;
    Lp_ = static_cast<int>(round_up(L_, 4));
  }
  require(cfg.hidden_layers >= 1 && cfg.hidden >= 32 && cfg.hidden % 32 == 0,
          "vlearner: hidden width must be a multiple of 32");
  require(cfg.batch_size >= 1, "vlearner: batch_size must be >= 1");
  D_ = dims.obs_dim;
  A_ = dims.act_dim;
  H_ = cfg.hidden;
  nh_ = cfg.hidden_layers;
  B_ = cfg.batch_size;
  Kp_ = static_cast<int>(round_up(D_ + A_, 4));
  reward_scale_ = static_cast<float>(cfg.reward_scale);
  gamma_ = static_cast<float>(cfg.gamma);

  std::vector<int> qs{D_ + A_}, ps{D_};
  for (int i = 0; i < nh_; ++i) {
    qs.push_back(H_);
    ps.push_back(H_);
  }
  qs.push_back(L_);  // learners.cpp:127-130: n_atoms outputs for pql_d, else 1
  ps.push_back(sac_ ? 2 * A_ : A_);  // GaussianPolicy: [mean | log_std] (learners.cpp:20-22)
  qnet_ = NetShape::make(qs);
  pnet_ = NetShape::make(ps);
  const int64_t P = qnet_.params;
  Ps_ = round_up(P, 64);  // group stride: 16-byte aligned second critic for TMA
  const int64_t Ps = Ps_;

  // --- parameters: CriticPair::create (critic.hpp:16-26) and the lagged policy
  std::mt19937_64 init_rng(init_seed);
  std::vector<float> q1, q2, pol;
  init_orthogonal(qnet_, q1, init_rng, static_cast<float>(std::sqrt(2.0)), 1.0f);
  init_orthogonal(qnet_, q2, init_rng, static_cast<float>(std::sqrt(2.0)), 1.0f);
  std::mt19937_64 prng(rng::derive_seed(cfg.seed, rng::kInit, 0));
  init_orthogonal(pnet_, pol, prng, static_cast<float>(std::sqrt(2.0)), 1e-2f);
  q_.alloc(2 * Ps);
  qt_.alloc(2 * Ps);
  m_.alloc(2 * Ps);
  v_.alloc(2 * Ps);
  grads_.alloc(2 * Ps);
  lagged_.alloc(snapshot_len());  // [net | log_alpha] for pql_sac
  copy_sync(q_.p, q1.data(), P * 4, cudaMemcpyHostToDevice);
  copy_sync(q_.p + Ps, q2.data(), P * 4, cudaMemcpyHostToDevice);
  copy_sync(qt_.p, q_.p, 2 * Ps * 4, cudaMemcpyDeviceToDevice);
  copy_sync(lagged_.p, pol.data(), pnet_.params * 4, cudaMemcpyHostToDevice);

  // --- replay + n-step (learners.cpp:131-136)
  replay_ = std::make_unique<DeviceReplay>(cfg.buffer_capacity, D_, A_, st);
  nstep_ = std::make_unique<DeviceNStep>(cfg.n_envs, D_, A_, gamma_, cfg.n_step);
  norm_.init(D_);
  sampler_.alloc(1);
  // sample stream make_rng(seed, sample, 1) (learners.cpp:136); data-parallel
  // rank r draws from its own stream 1 + 2r (rank 0 = the reference's)
  const uint64_t skey = rng::derive_seed(cfg.seed, rng::kSample, 1 + 2 * static_cast<uint64_t>(rank_));
  replay::SamplerState s0{skey, 0, 0, 0};
  copy_sync(sampler_.p, &s0, sizeof(s0), cudaMemcpyHostToDevice);
  mt_.seed(skey);
  idx_.alloc(B_);
  idx_host_.resize(B_);
  // eps stream make_rng(seed, sac, 1) (learners.cpp:137); rank r: 1 + 2r
  if (sac_)
    eps_.init(rng::derive_seed(cfg.seed, rng::kSac, 1 + 2 * static_cast<uint64_t>(rank_)),
              static_cast<int64_t>(B_) * A_);

  // --- optimizer state
  step_.alloc(1);
  auto tab = mlp::adam_bias_table(0.9, 0.999);
  bc_.alloc(tab.size());
  copy_sync(bc_.p, tab.data(), tab.size() * sizeof(float2), cudaMemcpyHostToDevice);
  status_.alloc(1);
  hbuf_.alloc(2);
  loss_.alloc(1);

  {
    gemm::PrecisionScope prec(cfg.precision == PQLG_PREC_3XTF32);
    build_update();
  }
  PQLG_CUDA(cudaDeviceSynchronize());
}

VLearner::~VLearner() {
  if (graph_exec_) cudaGraphExecDestroy(graph_exec_);
  if (graph2_exec_) cudaGraphExecDestroy(graph2_exec_);
  if (owned_stream_) {
    cudaStreamSynchronize(owned_stream_);
    cudaStreamDestroy(owned_stream_);
  }
}

void VLearner::build_update() {
  const int B = B_, D = D_, A = A_, H = H_, nh = nh_, K0 = D + A;
  const int64_t P = qnet_.params;
  const int nt = mlp::hidden_slots(H);  // head-dot partial slots
  const int bnH = mlp::bn_for(H);
  const int mt = (B + 127) / 128;
  const int wpr = H / 32;  // mask words per row
  float* q1 = q_.p;
  float* q2 = q_.p + Ps_;
  float* q1t = qt_.p;
  float* q2t = qt_.p + Ps_;

  Xon_.alloc(static_cast<size_t>(B) * Kp_);
  Xtg_.alloc(static_cast<size_t>(B) * Kp_);
  ret_.alloc(B);
  eff_.alloc(B);
  y_.alloc(B);
  pact_.resize(nh);
  for (auto& b : pact_) b.alloc(static_cast<size_t>(B) * H);
  for (int k = 0; k < 2; ++k) {
    tact_[k].resize(nh);
    oact_[k].resize(nh);
    omask_[k].resize(nh);
    G_[k].resize(nh);
    for (int l = 0; l < nh; ++l) {
      tact_[k][l].alloc((l + 1 < nh || dist_) ? static_cast<size_t>(B) * H : 0);
      oact_[k][l].alloc(static_cast<size_t>(B) * H);
      omask_[k][l].alloc(static_cast<size_t>(B) * wpr);
      G_[k][l].alloc(static_cast<size_t>(B) * H);
    }
  }
  part_t_.alloc(2ull * nt * B);
  part_o_.alloc(2ull * nt * B);
  up_.alloc(2ull * B);
  const int loss_blocks = (B + critic::kRowThreads - 1) / critic::kRowThreads;
  block_loss_.alloc(std::max((B + c51::kThreads - 1) / c51::kThreads, c51::kLossBlocks));
  loss_counter_.alloc(1);

  if (dist_) {
    const auto z = c51_atoms(L_, static_cast<float>(cfg_.vmin), static_cast<float>(cfg_.vmax));
    atoms_.alloc(L_);
    copy_sync(atoms_.p, z.data(), L_ * 4, cudaMemcpyHostToDevice);
    probs_t_.alloc(2ull * B * Lp_);
    probs_o_.alloc(2ull * B * Lp_);
    ev_t_.alloc(2ull * B);
    up51_.alloc(2ull * B * Lp_);
    c51_blocks_ = c51::kLossBlocks * c51::kLossWarps;  // head-bias partial terms (warps)
    db51_.alloc(2ull * c51_blocks_ * L_);
    // the GEMMs read the 51-wide heads from padded mirrors (16-byte rows),
    // refreshed at the start of every update (the previous update's Adam /
    // Polyak, or set_params, changed them)
    const float* src[4] = {q1, q2, q1t, q2t};
    for (int k = 0; k < 4; ++k) heads_[k].init(src[k] + qnet_.w_off[nh], H, L_);
    const WeightMirror* hm = heads_.data();
    steps_.push_back([hm](cudaStream_t st) { refresh_mirrors(hm, 4, st); });
  }

  // ---------------------------------------------------------------- sample
  steps_.push_back([this, B](cudaStream_t st) {
    const uint64_t* idx = mt_mode_ ? idx_.p : nullptr;
    replay::Gather g{Xon_.p, Kp_, Xon_.p + D_, Kp_, Xtg_.p, Kp_, ret_.p, eff_.p};
    launch_replay_sample(*replay_, norm_.view(), g, sampler_.p, idx, B, st, capture_);
  });
  if (sac_) {  // eps for the reparameterised next actions (learners.cpp:171-173)
    logp_.alloc(B);
    steps_.push_back([this](cudaStream_t st) {
      if (mt_mode_) eps_.fill_mt(st);
      else eps_.fork(st);  // parallel branch, joined before the sampling finish
    });
  }

  // ------------------------------------------- target policy (lagged, 1 group)
  {
    const float* in = Xtg_.p;
    int64_t ld = Kp_;
    int K = D;
    for (int l = 0; l < nh; ++l) {
      epi::Hidden e{};
      e.bias[0] = e.bias[1] = lagged_.p + pnet_.b_off[l];
      e.bn = bnH;
      e.M = B;
      e.N = H;
      e.store = 1;
      const float* W = lagged_.p + pnet_.w_off[l];
      steps_.push_back(mlp::fwd(in, in, ld, W, W, B, H, K, 1, e, 0, pact_[l].p, pact_[l].p, H));
      in = pact_[l].p;
      ld = H;
      K = H;
    }
    const int hout = sac_ ? 2 * A : A;
    const float* Wh = lagged_.p + pnet_.w_off[nh];
    if (sac_) {
      // next = lagged.sample(boot, eps) (sac.hpp:31): actions + log-probs;
      // the head's W packed on adopt (lagged_changed)
      wpack_.alloc(static_cast<size_t>(mlp::head_pack_elems(hout, H)) * 4);
      wpack_n_ = hout;
      lagged_changed();
      head::RowsArgs base{};
      base.wpack = reinterpret_cast<const float4*>(wpack_.p);
      steps_.push_back(mlp::head_raw_step(head_split_, in, ld, Wh, B, hout, H, base));
      sac::GaussArgs g{};
      g.bias = lagged_.p + pnet_.b_off[nh];
      g.eps = eps_.out.p;
      g.act = Xtg_.p + D;
      g.ld_act = Kp_;
      g.logp = logp_.p;
      g.mid = (dims_.low + dims_.high) / 2.0f;
      g.half = (dims_.high - dims_.low) / 2.0f;
      steps_.push_back([this](cudaStream_t st) { eps_.join(st); });
      steps_.push_back(gauss_finish_step(head_split_, g, B, A));
    } else {
      head::RowsArgs ph{};
      ph.bias = lagged_.p + pnet_.b_off[nh];
      ph.out = Xtg_.p + D;  // critic target input [norm(boot) | pi(boot)]
      ph.ld_out = Kp_;
      ph.mid = (dims_.low + dims_.high) / 2.0f;
      ph.half = (dims_.high - dims_.low) / 2.0f;
      // W in the head kernel's fragment order, re-packed when the lagged
      // policy changes (lagged_changed)
      wpack_.alloc(static_cast<size_t>(mlp::head_pack_elems(A, H)) * 4);
      wpack_n_ = A;
      ph.wpack = reinterpret_cast<const float4*>(wpack_.p);
      lagged_changed();
      steps_.push_back(mlp::head_squash_step(ph, in, ld, Wh, B, A, H));
    }
  }

  // ---------- twin target + twin online critics: one 4-group launch per layer
  // Groups (q1', q2', q1, q2): the target and online chains are independent
  // given their inputs [norm(boot) | pi(boot)] and [norm(obs) | act], so each
  // layer is one persistent launch of 4 x (M/128) x (H/BN) tiles (measured:
  // splitting them into two 2-group chains on forked graph branches, the
  // online one beside the target-policy chain, costs 291 vs 282 us/update).
  {
    float* nets[4] = {q1t, q2t, q1, q2};
    for (int l = 0; l < nh; ++l) {
      epi::Hidden e{};
      const float* A[4];
      const float* W[4];
      const float* Dst[4];
      const bool last = l + 1 == nh;
      for (int g = 0; g < 4; ++g) {
        const bool tgt = g < 2;
        const int k = g & 1;
        e.bias[g] = nets[g] + qnet_.b_off[l];
        e.mask[g] = tgt ? nullptr : omask_[k][l].p;
        W[g] = nets[g] + qnet_.w_off[l];
        A[g] = l == 0 ? (tgt ? Xtg_.p : Xon_.p) : (tgt ? tact_[k][l - 1].p : oact_[k][l - 1].p);
        const bool store = !tgt || !last || dist_;
        if (store) e.store |= 1 << g;
        Dst[g] = store ? (tgt ? tact_[k][l].p : oact_[k][l].p) : nullptr;
        if (last && !dist_) {  // DDPG value head 512->1 folded in as partial dots
          e.w_head[g] = nets[g] + qnet_.w_off[nh];
          e.partial[g] = (tgt ? part_t_.p : part_o_.p) + static_cast<size_t>(k) * nt * B;
        }
      }
      e.ld_mask = B;  // word-major masks
      e.bn = bnH;
      e.M = B;
      e.N = H;
      e.ld_part = B;
      e.n_slots = nt;
      const int64_t lda = l == 0 ? Kp_ : H;
      const int K = l == 0 ? K0 : H;
      steps_.push_back(mlp::fwd_groups(A, lda, W, B, H, K, 4, e, 0, Dst, H));
    }
    if (dist_) {
      // categorical heads H -> L: logits + softmax (+ expected values of the
      // target heads) in the epilogue (c51.hpp:114-126, :135-138)
      epi::C51Head ch{};
      const float* A[4];
      const float* W[4];
      for (int g = 0; g < 4; ++g) {
        const bool tgt = g < 2;
        const int k = g & 1;
        ch.bias[g] = nets[g] + qnet_.b_off[nh];
        ch.probs[g] = (tgt ? probs_t_.p : probs_o_.p) + static_cast<size_t>(k) * B * Lp_;
        ch.ev[g] = tgt ? ev_t_.p + static_cast<size_t>(k) * B : nullptr;
        A[g] = tgt ? tact_[k][nh - 1].p : oact_[k][nh - 1].p;
        W[g] = heads_[tgt ? 2 + k : k].ptr();
      }
      ch.ld = Lp_;
      ch.atoms = atoms_.p;
      ch.M = B;
      ch.L = L_;
      steps_.push_back(mlp::fwd_groups(A, H, W, B, L_, H, 4, ch, heads_[0].stride(), nullptr, 0));
    }
  }

  // ------------------------------------------- TD target + loss + upstream
  if (dist_) {
    c51::CriticLossArgs a{};
    for (int k = 0; k < 2; ++k) {
      a.pt[k] = probs_t_.p + static_cast<size_t>(k) * B * Lp_;
      a.evt[k] = ev_t_.p + static_cast<size_t>(k) * B;
      a.po[k] = probs_o_.p + static_cast<size_t>(k) * B * Lp_;
    }
    a.ld = Lp_;
    a.ret = ret_.p;
    a.eff = eff_.p;
    a.atoms = atoms_.p;
    const float vmin = static_cast<float>(cfg_.vmin), vmax = static_cast<float>(cfg_.vmax);
    a.vmin = vmin;  // head.vmin / vmax are floats widened to double (c51.hpp:72)
    a.vmax = vmax;
    a.dz = (static_cast<double>(vmax) - vmin) / static_cast<double>(L_ - 1);
    a.L = L_;
    a.up = up51_.p;
    a.db_part = db51_.p;
    a.step = step_.p;
    a.block_loss = block_loss_.p;
    a.counter = loss_counter_.p;
    a.loss_out = loss_.p;
    a.status = status_.p;
    a.B = B;
    a.Bg = B * world_;
    steps_.push_back([a](cudaStream_t st) {
      launch(c51::c51_critic_loss_kernel, dim3(c51::kLossBlocks), dim3(c51::kLossWarps * 32), 0,
             st, a);
    });
  } else {
    critic::LossArgs a{};
    a.partial = part_o_.p;
    a.ld = B;
    a.n_tiles = nt;
    a.q1 = q1;
    a.q2 = q2;
    a.head_b_off = qnet_.b_off[nh];
    a.partial_t = part_t_.p;
    a.q1t = q1t;
    a.q2t = q2t;
    a.ret = ret_.p;
    a.eff = eff_.p;
    a.y = y_.p;
    if (sac_) {  // y = G + eff * (min Q' - alpha log pi) (sac.hpp:36-41)
      a.logp = logp_.p;
      a.log_alpha = lagged_.p + pnet_.params;
    }
    a.step = step_.p;
    a.up = up_.p;
    a.block_loss = block_loss_.p;
    a.counter = loss_counter_.p;
    a.loss_out = loss_.p;
    a.status = status_.p;
    a.B = B;
    a.Bg = B * world_;
    steps_.push_back([a, loss_blocks](cudaStream_t st) {
      launch(critic::critic_loss_kernel, dim3(loss_blocks), dim3(critic::kRowThreads), 0, st, a);
    });
  }

  // -------------------------------------------------------------- backward
  wpart_.resize(nh);
  colsum_.resize(nh);
  wsplits_.resize(nh);
  for (int l = 0; l < nh; ++l) {
    const int in = l == 0 ? K0 : H;
    wsplits_[l] = mlp::wgrad_splits(in, H, B, 2);
    wpart_[l].alloc(2ull * wsplits_[l] * in * H);
    colsum_[l].alloc(2ull * mt * H);
  }
  const int ht = (B + critic::kHeadRows - 1) / critic::kHeadRows;  // head-backward row tiles
  head_dw_.alloc(2ull * ht * H);
  head_db_.alloc(2ull * ht);
  head_cs_.alloc(2ull * ht * H);
  // gradient segments (split-K / row-tile partials -> flat gradient) of
  // hidden layer l and of the head layer, for the finalize pass(es)
  auto layer_segs = [&](int l) {
    const int in = l == 0 ? K0 : H;
    std::vector<optim::Segment> v;
    v.push_back(optim::Segment{qnet_.w_off[l], static_cast<int64_t>(in) * H, wpart_[l].p,
                               static_cast<int64_t>(wsplits_[l]) * in * H, wsplits_[l],
                               static_cast<int64_t>(in) * H});
    if (l + 1 < nh || dist_)
      v.push_back(optim::Segment{qnet_.b_off[l], H, colsum_[l].p, static_cast<int64_t>(mt) * H,
                                 mt, H});
    else  // the last hidden layer's bias gradient comes from the head backward
      v.push_back(optim::Segment{qnet_.b_off[l], H, head_cs_.p, static_cast<int64_t>(ht) * H,
                                 ht, H});
    return v;
  };
  auto head_segs = [&]() {
    std::vector<optim::Segment> v;
    if (dist_) {
      optim::Segment wh{qnet_.w_off[nh], static_cast<int64_t>(H) * L_, head_wpart_.p,
                        static_cast<int64_t>(head_splits_) * H * Lp_, head_splits_,
                        static_cast<int64_t>(H) * Lp_};
      wh.cols = L_;
      wh.ld_src = Lp_;
      v.push_back(wh);
      v.push_back(optim::Segment{qnet_.b_off[nh], L_, db51_.p,
                                 static_cast<int64_t>(c51_blocks_) * L_, c51_blocks_, L_});
    } else {
      v.push_back(optim::Segment{qnet_.w_off[nh], H, head_dw_.p, static_cast<int64_t>(ht) * H,
                                 ht, H});
      v.push_back(optim::Segment{qnet_.b_off[nh], 1, head_db_.p, ht, ht, 1});
    }
    return v;
  };
  // data parallel: bucketed reduce + all-reduce per layer on
  // a communication branch, issued as each layer's gradient completes
  if (comm_) dp_ = std::make_unique<DpBuckets>(comm_, grads_.p, 2, Ps_);
  auto dp_bucket = [&](std::vector<optim::Segment> segs, int layer, bool with_loss) {
    const int64_t lo = qnet_.w_off[layer], hi = qnet_.b_off[layer] + qnet_.sizes[layer + 1];
    steps_.push_back(dp_->bucket(std::move(segs), lo, hi, with_loss ? loss_.p : nullptr,
                                 with_loss ? 1 : 0));
  };
  if (dist_) {
    // categorical head layer H -> L (fa::backward, mlp.hpp:161-184):
    //   dW_head = h^T up   (split-K over the batch, fixed-order reduction)
    //   G_{nh-1} = (up W_head^T) * [h > 0]  + bias column sums of layer nh-1
    head_splits_ = mlp::wgrad_splits(H, L_, B, 2);
    head_wpart_.alloc(2ull * head_splits_ * H * Lp_);
    const float* u0 = up51_.p;
    const float* u1 = up51_.p + static_cast<size_t>(B) * Lp_;
    steps_.push_back(mlp::wgrad(oact_[0][nh - 1].p, oact_[1][nh - 1].p, H, u0, u1, Lp_, H, L_,
                                B, 2, head_splits_, epi::Partial{}, head_wpart_.p, Lp_));
    epi::DgradMask dm{};
    for (int k = 0; k < 2; ++k) dm.mask[k] = omask_[k][nh - 1].p;
    dm.ld_mask = B;  // word-major masks
    dm.colsum = colsum_[nh - 1].p;
    dm.ld_cs = H;
    dm.m_tiles = mt;
    dm.bn = bnH;
    dm.M = B;
    dm.N = H;
    steps_.push_back(mlp::dgrad(u0, u1, Lp_, heads_[0].ptr(), heads_[1].ptr(), heads_[0].stride(),
                                B, H, L_, 2, dm, G_[0][nh - 1].p, G_[1][nh - 1].p, H));
    if (dp_) dp_bucket(head_segs(), nh, true);
  } else {
    critic::HeadBwdArgs a{};
    a.up = up_.p;
    for (int k = 0; k < 2; ++k) {
      a.h[k] = oact_[k][nh - 1].p;
      a.w[k] = (k ? q2 : q1) + qnet_.w_off[nh];
      a.G[k] = G_[k][nh - 1].p;
    }
    a.ld_h = H;
    a.ld_g = H;
    a.dw_part = head_dw_.p;
    a.db_head_part = head_db_.p;
    a.db_part = head_cs_.p;
    a.B = B;
    a.H = H;
    a.tiles = ht;
    a.with_params = 1;
    steps_.push_back([a, ht](cudaStream_t st) {
      launch(critic::head_backward_kernel, dim3(dim3(ht, 2)), dim3(critic::kHeadThreads), 0, st, a);
    });
    if (dp_) dp_bucket(head_segs(), nh, true);
  }
  for (int l = nh - 1; l >= 0; --l) {
    const int in = l == 0 ? K0 : H;
    // wgrad: dW_l = act_{l-1}^T G_l  (act_{-1} = the critic input)
    const float* h0 = l == 0 ? Xon_.p : oact_[0][l - 1].p;
    const float* h1 = l == 0 ? Xon_.p : oact_[1][l - 1].p;
    const int64_t ldh = l == 0 ? Kp_ : H;
    steps_.push_back(mlp::wgrad(h0, h1, ldh, G_[0][l].p, G_[1][l].p, H, in, H, B, 2,
                                wsplits_[l], epi::Partial{}, wpart_[l].p));
    if (dp_) dp_bucket(layer_segs(l), l, false);
    if (l > 0) {
      // dgrad: G_{l-1} = (G_l W_l^T) * [act_{l-1} > 0], + bias colsums of layer l-1
      epi::DgradMask dm{};
      for (int k = 0; k < 2; ++k) dm.mask[k] = omask_[k][l - 1].p;
      dm.ld_mask = B;  // word-major masks
      dm.colsum = colsum_[l - 1].p;
      dm.ld_cs = H;
      dm.m_tiles = mt;
      dm.bn = bnH;
      dm.M = B;
      dm.N = H;
      steps_.push_back(mlp::dgrad(G_[0][l].p, G_[1][l].p, H, q1 + qnet_.w_off[l],
                                  q2 + qnet_.w_off[l], H, B, H, H, 2, dm, G_[0][l - 1].p,
                                  G_[1][l - 1].p, H));
    }
  }

  // --------------------------------------- gradient reduction + clip scale
  {
    optim::FinalizeArgs f{};
    int s = 0;
    if (comm_) {
      // the buckets hold the all-reduced full-batch gradient (each rank's
      // upstream already carries 1/(B*world)): the norm + clip scale
      // (clip_global_norm per critic, learners.cpp:182-183) as a
      // single-term pass over it, flagging a non-finite all-reduced loss
      steps_.push_back(dp_->join());
      f.seg[s++] = optim::Segment{0, P, grads_.p, Ps_, 1, 0};
      f.check = loss_.p;
    } else {
      for (int l = 0; l < nh; ++l)
        for (const auto& sg : layer_segs(l)) f.seg[s++] = sg;
      for (const auto& sg : head_segs()) f.seg[s++] = sg;
    }
    require(s <= optim::kMaxSegments, "vlearner: too many layers");
    f.n_seg = s;
    f.total = P;
    f.gstride = Ps_;
    f.grads = grads_.p;
    fin_blocks_ = optim::plan_finalize(f);
    block_sq_.alloc(2ull * fin_blocks_);
    fin_counter_.alloc(2);
    scale_.alloc(2);
    f.block_sq = block_sq_.p;
    f.counter = fin_counter_.p;
    f.scale = scale_.p;
    f.status = status_.p;
    f.max_norm = 0.5f;
    const int fb = fin_blocks_;
    steps_.push_back([f, fb](cudaStream_t st) {
      launch(optim::finalize_kernel, dim3(dim3(fb, 2)), dim3(optim::kFinalizeThreads), 0, st, f);
    });
  }
  // ------------------------------------------------ clip + Adam + Polyak
  {
    optim::AdamArgs a{};
    a.p = q_.p;
    a.g = grads_.p;
    a.m = m_.p;
    a.v = v_.p;
    a.target = qt_.p;
    a.n = P;
    a.gstride = Ps_;
    a.scale = scale_.p;
    a.status = status_.p;
    a.step = step_.p;
    a.bc = bc_.p;
    a.bc_len = static_cast<int64_t>(bc_.n);
    a.lr = static_cast<float>(cfg_.lr_critic);
    a.beta1 = 0.9f;
    a.beta2 = 0.999f;
    a.eps = 1e-8f;
    a.tau = static_cast<float>(cfg_.tau);
    const int blocks = static_cast<int>(std::min<int64_t>(4 * mlp::kSMs, (P + 255) / 256));
    steps_.push_back([a, blocks](cudaStream_t st) {
      launch(optim::adam_polyak_kernel, dim3(dim3(blocks, 2)), dim3(256), 0, st, a);
    });
  }
}

void VLearner::lagged_changed() {
  if (!wpack_.p) return;
  mlp::head_pack(lagged_.p + pnet_.w_off[pnet_.layers() - 1], wpack_n_, cfg_.hidden, wpack_n_,
                 reinterpret_cast<float4*>(wpack_.p), cfg_.precision == PQLG_PREC_3XTF32,
                 stream_);
}

void VLearner::adopt_policy(const float* flat, int64_t version) {
  if (version < lagged_version_) return;  // learners.cpp:37-42
  PQLG_CUDA(cudaMemcpyAsync(lagged_.p, flat, pnet_.params * 4, cudaMemcpyHostToDevice, stream_));
  lagged_changed();
  PQLG_CUDA(cudaStreamSynchronize(stream_));
  lagged_version_ = version;
}

void VLearner::adopt_policy_sac(const float* flat, float log_alpha, int64_t version) {
  require(sac_, "adopt_policy_sac: learner is not pql_sac");
  if (version < lagged_version_) return;
  PQLG_CUDA(cudaMemcpyAsync(lagged_.p, flat, pnet_.params * 4, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(lagged_.p + pnet_.params, &log_alpha, 4, cudaMemcpyHostToDevice,
                            stream_));
  lagged_changed();
  PQLG_CUDA(cudaStreamSynchronize(stream_));
  lagged_version_ = version;
}

void VLearner::adopt_policy_device(const float* flat, int64_t version) {
  if (version < lagged_version_) return;  // learners.cpp:37-42
  PQLG_CUDA(cudaMemcpyAsync(lagged_.p, flat, snapshot_len() * 4, cudaMemcpyDeviceToDevice,
                            stream_));
  lagged_changed();
  lagged_version_ = version;
}

void VLearner::adopt_norm(int64_t count, const double* mean, const double* m2) {
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

void VLearner::ingest(const replay::Slice& s) { nstep_->push(s, reward_scale_, *replay_, stream_); }

// Host StepSlice (CriticLearnerCore::ingest takes host matrices,
// learners.cpp:144-151): staged into device buffers on the learner's stream.
void VLearner::ingest_host(const pqlg_step_slice& h) {
  const int N = cfg_.n_envs, D = D_, A = A_;
  const int64_t lo = h.ld_obs > 0 ? h.ld_obs : D, la = h.ld_act > 0 ? h.ld_act : A;
  require(h.obs && h.act && h.boot_obs && h.rew && h.term && h.trunc, "ingest: null slice field");
  const int Dp = static_cast<int>(round_up(D, 4)), Ap = static_cast<int>(round_up(A, 4));  // 16-byte rows: vector gathers
  const size_t nf = static_cast<size_t>(N) * (2 * Dp + Ap + 1);
  if (in_f_.n < nf) in_f_.alloc(nf);
  if (in_u8_.n < 2u * N) in_u8_.alloc(2u * N);
  float* obs = in_f_.p;
  float* boot = obs + static_cast<size_t>(N) * Dp;
  float* act = boot + static_cast<size_t>(N) * Dp;
  float* rew = act + static_cast<size_t>(N) * Ap;
  auto h2d2 = [&](float* dst, int64_t ldd, int w, const float* src, int64_t ld) {
    PQLG_CUDA(cudaMemcpy2DAsync(dst, ldd * 4, src, ld * 4, w * 4, N, cudaMemcpyHostToDevice,
                                stream_));
  };
  h2d2(obs, Dp, D, h.obs, lo);
  h2d2(boot, Dp, D, h.boot_obs, lo);
  h2d2(act, Ap, A, h.act, la);
  PQLG_CUDA(cudaMemcpyAsync(rew, h.rew, N * 4, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(in_u8_.p, h.term, N, cudaMemcpyHostToDevice, stream_));
  PQLG_CUDA(cudaMemcpyAsync(in_u8_.p + N, h.trunc, N, cudaMemcpyHostToDevice, stream_));
  ingest(replay::Slice{obs, act, boot, rew, in_u8_.p, in_u8_.p + N, Dp, Ap});
  PQLG_CUDA(cudaStreamSynchronize(stream_));  // the host slice may be reused on return
}

bool VLearner::ready(int64_t c_a) {
  return c_a >= cfg_.warm_up && replay_->size() >= static_cast<uint64_t>(B_);
}

void VLearner::prepare_indices() {
  // The reference's own generator: uniform_int_distribution over
  // std::mt19937_64 make_rng(seed, sample, 1) (replay_buffer.hpp:58-59).
  const uint64_t count = replay_->size();
  std::uniform_int_distribution<std::size_t> pick(0, count - 1);
  for (int r = 0; r < B_; ++r) idx_host_[r] = pick(mt_);
  PQLG_CUDA(cudaMemcpyAsync(idx_.p, idx_host_.data(), B_ * sizeof(uint64_t),
                            cudaMemcpyHostToDevice, stream_));
}

void VLearner::enqueue() {
  const int skip = skip_step();
  for (size_t i = 0; i < steps_.size(); ++i)
    if (static_cast<int>(i) != skip) steps_[i](stream_);
}

std::string VLearner::time_update(int reps) {
  require(!mt_mode_, "time_update: graph replay needs the Philox sampler");
  if (replay_->size() < static_cast<uint64_t>(B_))
    throw Error(PQLG_NOT_READY, "critic update before buffer warm-up");
  return time_in_graph([&] { enqueue(); }, stream_, reps);
}

int VLearner::check_status() {
  uint32_t st = 0;
  PQLG_CUDA(cudaMemcpyAsync(&st, status_.p, 4, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
  if (st) {
    PQLG_CUDA(cudaMemsetAsync(status_.p, 0, 4, stream_));
    return PQLG_ENONFINITE;
  }
  return PQLG_OK;
}

float VLearner::update() {
  if (replay_->size() < static_cast<uint64_t>(B_))
    throw Error(PQLG_NOT_READY, "critic update before buffer warm-up");
  if (mt_mode_ || eager_updates()) {  // host-drawn indices / profiling: eager launches
    if (mt_mode_) prepare_indices();
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
    throw Error(PQLG_ENONFINITE, "ddpg critic update: non-finite");
  }
  float loss;
  std::memcpy(&loss, &hbuf_.p[0], 4);
  return loss;
}

void VLearner::update_n(int n) {
  require(!mt_mode_, "update_n: graph replay needs the Philox sampler");
  if (!graph_checked_) {
    if (replay_->size() < static_cast<uint64_t>(B_))
      throw Error(PQLG_NOT_READY, "critic update before buffer warm-up");
    graph_checked_ = true;
  }
  if (!graph_exec_) {
    capture_ = true;
    for (int reps = 1; reps <= 2; ++reps) {
      cudaGraph_t g;
      const uint64_t before = g_launches.load();
      PQLG_CUDA(cudaStreamBeginCapture(stream_, cudaStreamCaptureModeThreadLocal));
      for (int r = 0; r < reps; ++r) enqueue();
      PQLG_CUDA(cudaStreamEndCapture(stream_, &g));
      kpu_ = static_cast<int>(g_launches.load() - before) / reps;
      g_launches.fetch_sub(static_cast<uint64_t>(reps) * kpu_);  // captured, not launched
      PQLG_CUDA(cudaGraphInstantiate(reps == 1 ? &graph_exec_ : &graph2_exec_, g, 0));
      cudaGraphDestroy(g);
    }
    capture_ = false;
  }
  for (int i = 0; i + 1 < n; i += 2) PQLG_CUDA(cudaGraphLaunch(graph2_exec_, stream_));
  if (n % 2) PQLG_CUDA(cudaGraphLaunch(graph_exec_, stream_));
  count_launch(static_cast<uint64_t>(n) * kpu_);
}

int VLearner::kernels_per_update() {
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

float VLearner::last_loss() {
  float loss = 0.0f;
  PQLG_CUDA(cudaMemcpyAsync(&loss, loss_.p, 4, cudaMemcpyDeviceToHost, stream_));
  if (check_status() != PQLG_OK) throw Error(PQLG_ENONFINITE, "ddpg critic update: non-finite");
  return loss;
}

void VLearner::get_params(int which, float* out) {
  const int64_t P = qnet_.params;
  const float* src = nullptr;
  int64_t n = P;
  switch (which) {
    case 0: src = q_.p; break;
    case 1: src = q_.p + Ps_; break;
    case 2: src = qt_.p; break;
    case 3: src = qt_.p + Ps_; break;
    case 4: src = lagged_.p; n = pnet_.params; break;
    default: throw Error(PQLG_EINVAL, "get_params: which must be 0..4");
  }
  PQLG_CUDA(cudaMemcpyAsync(out, src, n * 4, cudaMemcpyDeviceToHost, stream_));
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

int64_t VLearner::param_count(int which) const {
  return which == 4 ? pnet_.params : qnet_.params;
}

void VLearner::set_params(int which, const float* flat) {
  const int64_t P = qnet_.params;
  float* dst = nullptr;
  int64_t n = P;
  switch (which) {
    case 0: dst = q_.p; break;
    case 1: dst = q_.p + Ps_; break;
    case 2: dst = qt_.p; break;
    case 3: dst = qt_.p + Ps_; break;
    case 4: dst = lagged_.p; n = pnet_.params; break;
    default: throw Error(PQLG_EINVAL, "set_params: which must be 0..4");
  }
  PQLG_CUDA(cudaMemcpyAsync(dst, flat, n * 4, cudaMemcpyHostToDevice, stream_));
  if (which == 4) lagged_changed();
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

float VLearner::log_alpha() {
  float v = 0.0f;
  if (sac_) {
    PQLG_CUDA(cudaMemcpyAsync(&v, lagged_.p + pnet_.params, 4, cudaMemcpyDeviceToHost, stream_));
    PQLG_CUDA(cudaStreamSynchronize(stream_));
  }
  return v;
}

void VLearner::debug_read(int what, float* out) {
  const int64_t P = qnet_.params;
  switch (what) {
    case 0:
      PQLG_CUDA(cudaMemcpyAsync(out, y_.p, B_ * 4, cudaMemcpyDeviceToHost, stream_));
      break;
    case 1:
      if (dist_)  // C51: dLoss/dlogits [2 x B x L]
        PQLG_CUDA(cudaMemcpy2DAsync(out, L_ * 4, up51_.p, Lp_ * 4, L_ * 4, 2ull * B_,
                                    cudaMemcpyDeviceToHost, stream_));
      else
        PQLG_CUDA(cudaMemcpyAsync(out, up_.p, 2ull * B_ * 4, cudaMemcpyDeviceToHost, stream_));
      break;
    case 2:
      PQLG_CUDA(cudaMemcpy2DAsync(out, P * 4, grads_.p, Ps_ * 4, P * 4, 2,
                                  cudaMemcpyDeviceToHost, stream_));
      break;
    case 3:
      PQLG_CUDA(cudaMemcpyAsync(out, scale_.p, 2 * 4, cudaMemcpyDeviceToHost, stream_));
      break;
    case 4:
      PQLG_CUDA(cudaMemcpy2DAsync(out, (D_ + A_) * 4, Xon_.p, Kp_ * 4, (D_ + A_) * 4, B_,
                                  cudaMemcpyDeviceToHost, stream_));
      break;
    case 5:  // pql_sac: this update's eps [B x A]
      require(sac_, "debug_read(5): pql_sac only");
      PQLG_CUDA(cudaMemcpyAsync(out, eps_.out.p, static_cast<size_t>(B_) * A_ * 4,
                                cudaMemcpyDeviceToHost, stream_));
      break;
    case 6:  // pql_sac: log pi(a'|s+) of the target actions [B]
      require(sac_, "debug_read(6): pql_sac only");
      PQLG_CUDA(cudaMemcpyAsync(out, logp_.p, B_ * 4, cudaMemcpyDeviceToHost, stream_));
      break;
    case 7:  // the target critics' input [B x (D + A)]: [norm(boot) | a']
      PQLG_CUDA(cudaMemcpy2DAsync(out, (D_ + A_) * 4, Xtg_.p, Kp_ * 4, (D_ + A_) * 4, B_,
                                  cudaMemcpyDeviceToHost, stream_));
      break;
    default: throw Error(PQLG_EINVAL, "debug_read: what must be 0..7");
  }
  PQLG_CUDA(cudaStreamSynchronize(stream_));
}

}  // namespace pqlg

// ------------------------------------------------------------------ C ABI
struct pqlg_vlearner_s {
  std::unique_ptr<pqlg::VLearner> v;
  pqlg_replay_s replay_view;
  cudaEvent_t ev = nullptr;  // record_event
  ~pqlg_vlearner_s() {
    if (ev) cudaEventDestroy(ev);
  }
};

namespace pqlg {
VLearner* vlearner_of(pqlg_vlearner h) {
  require(h != nullptr, "null vlearner handle");
  return h->v.get();
}
}  // namespace pqlg

using namespace pqlg;

extern "C" {

void pqlg_config_default(pqlg_config* c) {
  // RunConfig defaults (config.hpp:15-48) with Table B.1 values.
  *c = pqlg_config{};
  c->algo = PQLG_ALGO_DDPG;
  c->n_envs = 4096;
  c->batch_size = 8192;
  c->buffer_capacity = 5000000;
  c->gamma = 0.99;
  c->tau = 0.05;
  c->n_step = 3;
  c->lr_actor = 5e-4;
  c->lr_critic = 5e-4;
  c->warm_up = 32;
  c->sigma_min = 0.05;
  c->sigma_max = 0.8;
  c->sigma_fixed = -1.0;
  c->reward_scale = 1.0;
  c->seed = 0;
  c->hidden = 256;
  c->hidden_layers = 2;
  c->n_atoms = 51;
  c->vmin = -10.0;
  c->vmax = 10.0;
  c->max_episode_len = 1000;
  c->env_offset = 0;
  c->precision = PQLG_PREC_TF32;
}

int pqlg_vlearner_create(const pqlg_config* cfg, const pqlg_task_dims* dims,
                         uint64_t init_rng_seed, void* stream, pqlg_vlearner* out) {
  return guarded([&] {
    require(cfg && dims && out, "vlearner_create: null argument");
    auto h = std::make_unique<pqlg_vlearner_s>();
    h->v = std::make_unique<VLearner>(*cfg, *dims, init_rng_seed,
                                      static_cast<cudaStream_t>(stream));
    h->replay_view.r = h->v->replay();
    h->replay_view.norm.init(dims->obs_dim);
    *out = h.release();
  });
}

int pqlg_vlearner_create_dp(const pqlg_config* cfg, const pqlg_task_dims* dims,
                            uint64_t init_rng_seed, pqlg_comm comm, void* stream,
                            pqlg_vlearner* out) {
  return guarded([&] {
    require(cfg && dims && out && comm, "vlearner_create_dp: null argument");
    auto h = std::make_unique<pqlg_vlearner_s>();
    h->v = std::make_unique<VLearner>(*cfg, *dims, init_rng_seed,
                                      static_cast<cudaStream_t>(stream), comm);
    h->replay_view.r = h->v->replay();
    h->replay_view.norm.init(dims->obs_dim);
    *out = h.release();
  });
}

int pqlg_vlearner_wait_event(pqlg_vlearner h, void* event) {
  return guarded([&] {
    require(h && event, "vlearner_wait_event: null argument");
    PQLG_CUDA(cudaStreamWaitEvent(h->v->stream(), static_cast<cudaEvent_t>(event), 0));
  });
}

int pqlg_vlearner_record_event(pqlg_vlearner h, void** event_out) {
  return guarded([&] {
    require(h && event_out, "vlearner_record_event: null argument");
    if (!h->ev) PQLG_CUDA(cudaEventCreateWithFlags(&h->ev, cudaEventDisableTiming));
    PQLG_CUDA(cudaEventRecord(h->ev, h->v->stream()));
    *event_out = h->ev;
  });
}

int pqlg_vlearner_destroy(pqlg_vlearner h) {
  return guarded([&] { delete h; });
}

int pqlg_vlearner_adopt_policy(pqlg_vlearner h, const float* flat, int64_t version) {
  return guarded([&] { h->v->adopt_policy(flat, version); });
}

int pqlg_vlearner_adopt_policy_sac(pqlg_vlearner h, const float* flat, float log_alpha,
                                   int64_t version) {
  return guarded([&] { h->v->adopt_policy_sac(flat, log_alpha, version); });
}

int pqlg_vlearner_log_alpha(pqlg_vlearner h, float* out) {
  return guarded([&] { *out = h->v->log_alpha(); });
}

int pqlg_vlearner_adopt_norm(pqlg_vlearner h, const pqlg_norm_stats* n) {
  return guarded([&] { h->v->adopt_norm(n->count, n->mean, n->m2); });
}

int pqlg_vlearner_ingest(pqlg_vlearner h, const pqlg_step_slice* s) {
  return guarded([&] {
    const int D = h->v->obs_dim(), A = h->v->act_dim();
    replay::Slice sl{s->obs, s->act, s->boot_obs, s->rew, s->term, s->trunc,
                     s->ld_obs > 0 ? s->ld_obs : D, s->ld_act > 0 ? s->ld_act : A};
    h->v->ingest(sl);
  });
}

int pqlg_vlearner_ingest_host(pqlg_vlearner h, const pqlg_step_slice* s) {
  return guarded([&] {
    require(s != nullptr, "ingest_host: null slice");
    h->v->ingest_host(*s);
  });
}

int pqlg_vlearner_ready(pqlg_vlearner h, int64_t c_a, int* ready) {
  return guarded([&] { *ready = h->v->ready(c_a) ? 1 : 0; });
}

int pqlg_vlearner_update(pqlg_vlearner h, float* loss) {
  return guarded([&] {
    const float l = h->v->update();
    if (loss) *loss = l;
  });
}

int pqlg_vlearner_update_n(pqlg_vlearner h, int n) {
  return guarded([&] { h->v->update_n(n); });
}

int pqlg_vlearner_last_loss(pqlg_vlearner h, float* loss) {
  return guarded([&] { *loss = h->v->last_loss(); });
}

int pqlg_vlearner_get_params(pqlg_vlearner h, int which, float* out) {
  return guarded([&] { h->v->get_params(which, out); });
}

int pqlg_vlearner_param_count(pqlg_vlearner h, int which, int64_t* out) {
  return guarded([&] { *out = h->v->param_count(which); });
}

int pqlg_vlearner_snapshot(pqlg_vlearner h, float* q1, float* q2) {
  return guarded([&] {
    h->v->get_params(0, q1);
    h->v->get_params(1, q2);
  });
}

int pqlg_vlearner_buffer_size(pqlg_vlearner h, uint64_t* out) {
  return guarded([&] { *out = h->v->replay()->size(); });
}

int pqlg_vlearner_set_sampler(pqlg_vlearner h, int mode) {
  return guarded([&] {
    require(mode == PQLG_RNG_PHILOX || mode == PQLG_RNG_INDICES, "set_sampler: bad mode");
    h->v->set_mt_mode(mode == PQLG_RNG_INDICES);
  });
}

int pqlg_vlearner_replay(pqlg_vlearner h, pqlg_replay* out) {
  return guarded([&] { *out = &h->replay_view; });
}

int pqlg_vlearner_set_params(pqlg_vlearner h, int which, const float* flat) {
  return guarded([&] { h->v->set_params(which, flat); });
}

int pqlg_vlearner_debug_read(pqlg_vlearner h, int what, float* out) {
  return guarded([&] { h->v->debug_read(what, out); });
}

int pqlg_vlearner_kernels_per_update(pqlg_vlearner h, int* out) {
  return guarded([&] { *out = h->v->kernels_per_update(); });
}

int pqlg_vlearner_time_update(pqlg_vlearner h, int reps, char* out, int cap) {
  return guarded([&] {
    require(h && out && cap > 0, "vlearner_time_update: null argument");
    copy_cstr(h->v->time_update(reps), out, cap);
  });
}

}  // extern "C"
