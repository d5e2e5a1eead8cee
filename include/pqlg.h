/*
 * pqlg.h -- C ABI of the B200-native PQL learner/actor hot path (libpqlg.so).
 *
 * Drop-in boundary for the reference's runtime cores and replay objects
 * (reference paths are relative to /root/reference):
 *   ReplayBuffer / StateBuffer     proj/include/pql/replay/replay_buffer.hpp:17-119
 *   NStepAssembler / NStepBatch    proj/include/pql/replay/nstep.hpp:15-126
 *   ActorCore                      proj/include/pql/runtime/learners.hpp:52-73
 *   CriticLearnerCore              proj/include/pql/runtime/learners.hpp:77-106
 *   PolicyLearnerCore              proj/include/pql/runtime/learners.hpp:110-139
 *   kernels::* operator API        proj/include/pql/kernels/kernels.hpp:17-83
 *
 * Conventions
 *   - Every entry point returns an int status (PQLG_*); pqlg_last_error()
 *     returns the thread-local message of the last failure.
 *   - Pointers named *_dev are device pointers; *_host are host pointers.
 *   - Handles are owned by one host thread and run on one CUDA stream; all
 *     device work is asynchronous on that stream unless stated otherwise.
 *   - The library has no CPU fallback: without a CUDA device every compute
 *     entry point fails with PQLG_ECUDA.
 */
#ifndef PQLG_H_
#define PQLG_H_

#include <stddef.h>
#include <stdint.h>

#if defined(__GNUC__)
#define PQLG_API __attribute__((visibility("default")))
#else
#define PQLG_API
#endif

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------------ status */
enum {
  PQLG_OK = 0,
  PQLG_NOT_READY = 1,   /* empty std::optional / "before warm-up" runtime_error */
  PQLG_EINVAL = -1,     /* std::invalid_argument (shape / config)               */
  PQLG_ENONFINITE = -2, /* std::runtime_error for non-finite values             */
  PQLG_ECUDA = -3,
  PQLG_ENCCL = -4
};

PQLG_API const char* pqlg_last_error(void);
PQLG_API int pqlg_abi_version(void);
/* Number of kernels this library launched since load (evidence counter). */
PQLG_API uint64_t pqlg_launch_count(void);
/* Per-launch device timing for profiling: between begin and end every kernel
 * this library launches outside CUDA-graph capture is bracketed by events;
 * end synchronizes and writes "name\tms\n" lines into out (cap bytes). */
PQLG_API int pqlg_profile_begin(void);
PQLG_API int pqlg_profile_end(char* out, int cap);

/* ------------------------------------------------- operator-level test hooks
 * Device-pointer restatements of pql::kernels (kernels.hpp:25-60); there is
 * no backend dispatch -- these run the sm_100a kernels the learners use.
 */

/* D[M x N] = A x B (+ bias, ReLU) on tcgen05 tensor cores (tf32 inputs,
 * fp32 accumulate).  a_mn = 0: A is [M x K] row-major (K contiguous, stride
 * lda); a_mn = 1: A is stored transposed as [K x M] (stride lda).
 * b_mn = 0: B stored as [N x K] (stride ldb); b_mn = 1: B is [K x N].
 * splits > 1 splits K across CTAs with a fixed-order reduction.
 * round_mode: 0 = operands fed as fp32 bit patterns (hardware tf32 reads),
 *             1 = TMA tensor maps typed TFLOAT32. */
PQLG_API int pqlg_k_gemm_tf32(const float* A_dev, const float* B_dev, float* D_dev, const float* bias_dev,
                     int M, int N, int K, int a_mn, int b_mn, int lda, int ldb, int ldd, int relu,
                     int splits, int round_mode, void* stream);

/* `iters` back-to-back launches of the forward-layer GEMM (A K-major, B
 * [K x N] N-major, TFLOAT32 maps) for device-time measurement. */
PQLG_API int pqlg_k_gemm_tf32_repeat(const float* A_dev, const float* B_dev, float* D_dev,
                                     const float* bias_dev, int M, int N, int K, int lda, int ldb,
                                     int ldd, int relu, int iters, void* stream);

/* `iters` launches of the update's dominant GEMM: `groups` (<= 4) hidden
 * layers [M x K] x [K x N] in one persistent launch (Hidden epilogue: bias +
 * ReLU + TMA store), as the twin target + twin online critics run. */
PQLG_API int pqlg_k_gemm_tf32_repeat_groups(const float* A_dev, const float* B_dev, float* D_dev,
                                            const float* bias_dev, int M, int N, int K, int lda,
                                            int ldb, int ldd, int groups, int iters, void* stream);

/* ------------------------------------------------------------ data views */

/* StepSlice (proj/include/pql/runtime/messages.hpp:31-35) as device views.
 * ld_* are row strides in floats (0 = dense). */
typedef struct {
  const float* obs;      /* [N x obs_dim] raw observations s_t            */
  const float* act;      /* [N x act_dim] actions a_t                     */
  const float* boot_obs; /* [N x obs_dim] next obs, terminal obs on done  */
  const float* rew;      /* [N] unscaled task rewards                     */
  const uint8_t* term;   /* [N] terminated (done && !truncated)           */
  const uint8_t* trunc;  /* [N] time-limit truncation                     */
  int64_t ld_obs, ld_act;
} pqlg_step_slice;

/* NStepBatch (proj/include/pql/replay/nstep.hpp:15-29) as device views. */
typedef struct {
  float* obs;
  float* act;
  float* boot_obs;
  float* ret;
  float* eff_disc;
  int64_t ld_obs, ld_act;
} pqlg_nstep_batch;

/* NormStats (proj/include/pql/funcapprox/normalizer.hpp:14-21), host. */
typedef struct {
  int64_t count;
  const double* mean;
  const double* m2;
} pqlg_norm_stats;

/* Sampling generator.  PQLG_RNG_PHILOX: counter-based Philox4x32-10 draws
 * (key, counter), bit-exact against the reference's sample() driven by the
 * same URBG; the counter advances by the draws consumed.
 * PQLG_RNG_INDICES: explicit host indices (the reference's own
 * std::mt19937_64 stream generated on the host) -- the mt19937-compat mode. */
enum { PQLG_RNG_PHILOX = 0, PQLG_RNG_INDICES = 1 };
typedef struct {
  int mode;
  uint64_t key;
  uint64_t counter;
  const uint64_t* host_indices; /* [batch] when mode == PQLG_RNG_INDICES */
} pqlg_rng;

/* ------------------------------------------------------- replay buffers */
typedef struct pqlg_replay_s* pqlg_replay;
typedef struct pqlg_nstep_s* pqlg_nstep;
typedef struct pqlg_states_s* pqlg_states;

/* ReplayBuffer(capacity, obs_dim, act_dim)   replay_buffer.hpp:19-27 */
PQLG_API int pqlg_replay_create(uint64_t capacity, int obs_dim, int act_dim, void* stream,
                                pqlg_replay* out);
PQLG_API int pqlg_replay_destroy(pqlg_replay h);
/* size() / cursor() (replay_buffer.hpp:29-31); synchronize the stream. */
PQLG_API int pqlg_replay_size(pqlg_replay h, uint64_t* out);
PQLG_API int pqlg_replay_cursor(pqlg_replay h, uint64_t* out);
/* insert(batch)   replay_buffer.hpp:33-47 (n rows, device views) */
PQLG_API int pqlg_replay_insert(pqlg_replay h, const pqlg_nstep_batch* dev, uint64_t n);
/* sample(batch, rng, min_live)   replay_buffer.hpp:50-69.  Returns
 * PQLG_NOT_READY (empty optional) when size < min_live.  `norm` (nullable)
 * fuses RunningNormalizer::apply_stats on obs and boot_obs.  Synchronizes
 * and writes the advanced Philox counter back into *rng. */
PQLG_API int pqlg_replay_sample(pqlg_replay h, uint64_t batch, pqlg_rng* rng, uint64_t min_live,
                                const pqlg_norm_stats* norm, pqlg_nstep_batch* dev_out);
/* Appends n synthetic records generated on device (benchmark pre-fill,
 * SURVEY 8(d)): obs/boot ~ N(0,1), act ~ U(-1,1), ret ~ 0.1 N(0,1),
 * eff_disc = disc except every terminal_every-th record (0). */
PQLG_API int pqlg_replay_fill_synthetic(pqlg_replay h, uint64_t n, uint64_t seed, float disc,
                                        uint32_t terminal_every);
/* Ring rows [i0, i0+n) to host (obs_row / ret_at, replay_buffer.hpp:71-73);
 * any output pointer may be NULL. */
PQLG_API int pqlg_replay_read_rows(pqlg_replay h, uint64_t i0, uint64_t n, float* obs, float* act,
                                   float* boot_obs, float* ret, float* eff_disc);

/* NStepAssembler(n_envs, obs_dim, act_dim, gamma, horizon)  nstep.hpp:39-52 */
PQLG_API int pqlg_nstep_create(int n_envs, int obs_dim, int act_dim, float gamma, int horizon,
                               void* stream, pqlg_nstep* out);
PQLG_API int pqlg_nstep_destroy(pqlg_nstep h);
/* push_step fused with ReplayBuffer::insert (learners.cpp:144-151): rewards
 * are scaled by reward_scale first; the emitted records go straight into
 * `dst` in the reference's env-major order. */
PQLG_API int pqlg_nstep_push_step(pqlg_nstep h, const pqlg_step_slice* dev, float reward_scale,
                                  pqlg_replay dst);

/* StateBuffer(capacity, obs_dim)   replay_buffer.hpp:84-91 */
PQLG_API int pqlg_states_create(uint64_t capacity, int obs_dim, void* stream, pqlg_states* out);
PQLG_API int pqlg_states_destroy(pqlg_states h);
PQLG_API int pqlg_states_size(pqlg_states h, uint64_t* out);
PQLG_API int pqlg_states_insert(pqlg_states h, const float* rows_dev, int64_t ld, uint64_t n);
PQLG_API int pqlg_states_sample(pqlg_states h, uint64_t batch, pqlg_rng* rng, uint64_t min_live,
                                const pqlg_norm_stats* norm, float* out_dev, int64_t ld_out);

/* ------------------------------------------------------------ run config */

/* RunConfig fields the cores consume (proj/include/pql/config.hpp:15-48),
 * plus `hidden_layers` (the reference hard-codes 2: learners.cpp:22-23,
 * :127-130, :206-209; configs 2-5 need 3) and the synthetic env's time
 * limit.  pqlg_config_default() fills the Table B.1 defaults. */
/* pql_sac (algo.hpp:8, sac.hpp): the policy is a GaussianPolicy whose net
 * emits [mean | log_std] (2 x act_dim outputs, learners.cpp:20-22);
 * param_count / get_params / set_params of the policy are the net's.  The
 * snapshot's log_alpha (PolicySnapshot::log_alpha, messages.hpp:18-19)
 * travels beside it: pqlg_plearner_log_alpha reads the P-learner's,
 * pqlg_vlearner_adopt_policy_sac installs both in the V-learner, and the
 * run_parallel pipeline moves them together on the device. */
enum { PQLG_ALGO_DDPG = 0, PQLG_ALGO_C51 = 1, PQLG_ALGO_SAC = 2 };
/* GEMM precision of the MLP layers (the reference computes them in fp32,
 * scalar.hpp:12-55).  TF32: operands rounded to tf32 (10-bit mantissa), one
 * tcgen05 MMA per K step -- the speed mode.  3XTF32: each operand split into
 * tf32 hi + lo parts in shared memory and a_lo*b_hi + a_hi*b_lo + a_hi*b_hi
 * accumulated in fp32 -- products within a few fp32 ulps, 3x the MMA work;
 * the parity mode. */
enum { PQLG_PREC_TF32 = 0, PQLG_PREC_3XTF32 = 1 };
typedef struct {
  int algo;               /* PQLG_ALGO_DDPG (pql_ddpg), PQLG_ALGO_C51 (pql_d), PQLG_ALGO_SAC (pql_sac) */
  int n_envs;
  int batch_size;
  uint64_t buffer_capacity;
  double gamma;
  double tau;
  int n_step;
  double lr_actor;
  double lr_critic;
  int64_t warm_up;
  double sigma_min;
  double sigma_max;
  double sigma_fixed;     /* >= 0: same sigma for every env */
  double reward_scale;    /* effective_reward_scale() (> 0) */
  uint64_t seed;
  int hidden;             /* hidden width */
  int hidden_layers;      /* number of hidden layers */
  int n_atoms;
  double vmin;
  double vmax;
  int max_episode_len;    /* synthetic env time limit */
  int env_offset;         /* global index of this shard's first env (sharded actors) */
  int envs_total;         /* global env count of a sharded actor (0: n_envs)          */
  int precision;          /* PQLG_PREC_TF32 (speed) or PQLG_PREC_3XTF32 (fp32-faithful) */
} pqlg_config;

/* TaskDims (learners.hpp:23-26) */
typedef struct {
  int obs_dim;
  int act_dim;
  float low;
  float high;
} pqlg_task_dims;

PQLG_API void pqlg_config_default(pqlg_config* cfg);

/* ------------------------------------------------ data-parallel communicator
 * NCCL communicator for the data-parallel critic / policy updates of config 5
 * (SURVEY 8(e)): one process per GPU, one rank per process.  The 128-byte
 * id is created on rank 0 and shipped to the other ranks by the caller (any
 * host channel; the benchmark uses torch.distributed).  pqlg_comm_init must
 * run with the rank's CUDA device current.  NCCL failures -> PQLG_ENCCL. */
#define PQLG_COMM_ID_BYTES 128
typedef struct pqlg_comm_s* pqlg_comm;
PQLG_API int pqlg_comm_unique_id(uint8_t* id_out /* [PQLG_COMM_ID_BYTES] */);
PQLG_API int pqlg_comm_init(int rank, int world, const uint8_t* id, pqlg_comm* out);
PQLG_API int pqlg_comm_destroy(pqlg_comm c);
PQLG_API int pqlg_comm_rank(pqlg_comm c, int* rank, int* world);
/* In-place sum all-reduce of n floats on `stream` (device pointer). */
PQLG_API int pqlg_comm_allreduce_f32(pqlg_comm c, float* buf_dev, uint64_t n, void* stream);

/* ------------------------------------------------ V-learner (critic core) */
typedef struct pqlg_vlearner_s* pqlg_vlearner;

/* CriticLearnerCore(cfg, dims, init_rng)  learners.hpp:79, learners.cpp:122-139.
 * Critics are initialised exactly as CriticPair::create with
 * std::mt19937_64(init_rng_seed); the lagged policy as PolicyHandle::create
 * with make_rng(seed, init, 0).  Sampling uses Philox keyed by
 * derive_seed(seed, sample, 1) unless pqlg_vlearner_set_sampler selects the
 * reference's mt19937_64 stream. */
PQLG_API int pqlg_vlearner_create(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                  uint64_t init_rng_seed, void* stream, pqlg_vlearner* out);
/* Data-parallel CriticLearnerCore (SURVEY 8(e) option i): every rank samples
 * cfg->batch_size rows from its own replay shard (Philox key
 * derive_seed(seed, sample, 1 + 2*rank)), scales dLoss/dQ by
 * 1/(batch_size*world), and one NCCL all-reduce per update sums the twin
 * critics' gradients and the loss before clip + Adam + Polyak, so every rank
 * applies the full-batch update.  world == 1 is bit-identical to
 * pqlg_vlearner_create.  `comm` must outlive the learner. */
PQLG_API int pqlg_vlearner_create_dp(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                     uint64_t init_rng_seed, pqlg_comm comm, void* stream,
                                     pqlg_vlearner* out);
PQLG_API int pqlg_vlearner_destroy(pqlg_vlearner h);
/* adopt_policy: equal-or-newer version replaces (learners.cpp:37-42) */
PQLG_API int pqlg_vlearner_adopt_policy(pqlg_vlearner h, const float* flat_host, int64_t version);
/* pql_sac: adopt a PolicySnapshot's net and log_alpha (learners.cpp:37-42) */
PQLG_API int pqlg_vlearner_adopt_policy_sac(pqlg_vlearner h, const float* flat_host,
                                            float log_alpha, int64_t version);
/* pql_sac: the lagged policy's log_alpha (0 for other algos) */
PQLG_API int pqlg_vlearner_log_alpha(pqlg_vlearner h, float* out);
PQLG_API int pqlg_vlearner_adopt_norm(pqlg_vlearner h, const pqlg_norm_stats* norm);
/* ingest(StepSlice): reward scale + n-step + insert (learners.cpp:144-151) */
PQLG_API int pqlg_vlearner_ingest(pqlg_vlearner h, const pqlg_step_slice* dev);
/* The learner's stream waits for a cudaEvent_t (e.g. pqlg_actor_step_event)
 * before its next work: orders cross-stream reads of a device StepSlice. */
PQLG_API int pqlg_vlearner_wait_event(pqlg_vlearner h, void* event);
/* Records (and returns) the handle's event at the current end of its stream. */
PQLG_API int pqlg_vlearner_record_event(pqlg_vlearner h, void** event_out);
/* ingest from HOST buffers (a CPU-produced StepSlice): copied in on the
 * learner's stream; returns once the slice may be reused. */
PQLG_API int pqlg_vlearner_ingest_host(pqlg_vlearner h, const pqlg_step_slice* host);
PQLG_API int pqlg_vlearner_ready(pqlg_vlearner h, int64_t c_a, int* ready);
/* update(): one critic update; synchronizes and returns the loss
 * (PQLG_NOT_READY before warm-up, PQLG_ENONFINITE on non-finite). */
PQLG_API int pqlg_vlearner_update(pqlg_vlearner h, float* loss_host);
/* n updates replayed from a CUDA graph, asynchronous (no host sync). */
PQLG_API int pqlg_vlearner_update_n(pqlg_vlearner h, int n);
/* loss of the last completed update + sticky status; synchronizes. */
PQLG_API int pqlg_vlearner_last_loss(pqlg_vlearner h, float* loss_host);
/* which: 0 q1, 1 q2, 2 q1_target, 3 q2_target, 4 lagged policy (host copy) */
PQLG_API int pqlg_vlearner_get_params(pqlg_vlearner h, int which, float* flat_host);
PQLG_API int pqlg_vlearner_param_count(pqlg_vlearner h, int which, int64_t* out);
/* make_snapshot(version) -> online nets (learners.cpp:190-196) */
PQLG_API int pqlg_vlearner_snapshot(pqlg_vlearner h, float* q1_host, float* q2_host);
PQLG_API int pqlg_vlearner_buffer_size(pqlg_vlearner h, uint64_t* out);
/* Sampler: PQLG_RNG_PHILOX (default) or PQLG_RNG_INDICES = the reference's
 * own std::mt19937_64 make_rng(seed, sample, 1) stream drawn on the host. */
PQLG_API int pqlg_vlearner_set_sampler(pqlg_vlearner h, int mode);
/* The owned replay buffer (for direct inserts / inspection). */
PQLG_API int pqlg_vlearner_replay(pqlg_vlearner h, pqlg_replay* out);
/* Overwrite parameters (which as in get_params; CriticPair::hard_sync_online
 * for 0/1, critic.hpp:33-36); resets nothing else. */
PQLG_API int pqlg_vlearner_set_params(pqlg_vlearner h, int which, const float* flat_host);
/* Intermediates of the last update for parity checks: 0 TD target y [B],
 * 1 dLoss/dQ [2 x B] (C51: dLoss/dlogits [2 x B x n_atoms]),
 * 2 flat gradients before clipping [2 x P],
 * 3 clip scales [2], 4 sampled critic input [B x (obs_dim+act_dim)],
 * 5 (pql_sac) eps [B x act_dim], 6 (pql_sac) log pi(a'|s+) [B],
 * 7 target critic input [B x (obs_dim+act_dim)] = [norm(boot) | a']. */
PQLG_API int pqlg_vlearner_debug_read(pqlg_vlearner h, int what, float* host_out);
/* Number of kernels one update launches (graph nodes). */
PQLG_API int pqlg_vlearner_kernels_per_update(pqlg_vlearner h, int* out);
/* Measurement hook: the update graph captured with an event-record node
 * around every kernel, replayed `reps` times (after two warm-up replays, each
 * a real update); writes "kernel\tavg_ms\tshape\n" per launch in order and
 * a final "__graph__\tavg_ms\t\n" line (NUL-terminated, cap bytes).  The
 * event nodes remove programmatic-dependent-launch overlap between kernels. */
PQLG_API int pqlg_vlearner_time_update(pqlg_vlearner h, int reps, char* out, int cap);

/* ------------------------------------------------ P-learner (policy core) */
typedef struct pqlg_plearner_s* pqlg_plearner;

/* PolicyLearnerCore(cfg, dims, init_rng)  learners.hpp:112, learners.cpp:202-217.
 * Critic replicas initialised as CriticPair::create(std::mt19937_64(init_rng_seed)),
 * the policy as PolicyHandle::create(make_rng(seed, init, 0)); sampling keyed by
 * derive_seed(seed, sample, 2). */
PQLG_API int pqlg_plearner_create(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                  uint64_t init_rng_seed, void* stream, pqlg_plearner* out);
/* Data-parallel PolicyLearnerCore: as pqlg_vlearner_create_dp (sample key
 * derive_seed(seed, sample, 2 + 2*rank); one all-reduce of the policy
 * gradient and the loss per update). */
PQLG_API int pqlg_plearner_create_dp(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                     uint64_t init_rng_seed, pqlg_comm comm, void* stream,
                                     pqlg_plearner* out);
PQLG_API int pqlg_plearner_destroy(pqlg_plearner h);
/* adopt_critics(snapshot): equal-or-newer version replaces (learners.cpp:222-227) */
PQLG_API int pqlg_plearner_adopt_critics(pqlg_plearner h, const float* q1_host,
                                         const float* q2_host, int64_t version);
PQLG_API int pqlg_plearner_adopt_norm(pqlg_plearner h, const pqlg_norm_stats* norm);
/* ingest(states) = StateBuffer::insert (learners.hpp:117) */
PQLG_API int pqlg_plearner_ingest(pqlg_plearner h, const float* states_dev, int64_t ld,
                                  uint64_t n);
PQLG_API int pqlg_plearner_wait_event(pqlg_plearner h, void* event);
PQLG_API int pqlg_plearner_record_event(pqlg_plearner h, void** event_out);
PQLG_API int pqlg_plearner_ingest_host(pqlg_plearner h, const float* states_host, int64_t ld,
                                       uint64_t n);
PQLG_API int pqlg_plearner_ready(pqlg_plearner h, int64_t c_a, int* ready);
/* update(): one policy update; synchronizes and returns the actor loss. */
PQLG_API int pqlg_plearner_update(pqlg_plearner h, float* loss_host);
PQLG_API int pqlg_plearner_update_n(pqlg_plearner h, int n);
PQLG_API int pqlg_plearner_last_loss(pqlg_plearner h, float* loss_host);
/* make_snapshot(): the policy's flat parameters (host copy). */
PQLG_API int pqlg_plearner_snapshot(pqlg_plearner h, float* flat_host);
/* which: 0 policy, 1 critic replica q1, 2 critic replica q2 */
PQLG_API int pqlg_plearner_get_params(pqlg_plearner h, int which, float* flat_host);
PQLG_API int pqlg_plearner_set_params(pqlg_plearner h, int which, const float* flat_host);
PQLG_API int pqlg_plearner_param_count(pqlg_plearner h, int which, int64_t* out);
/* pql_sac: the learned log alpha (alpha_param_[0], learners.cpp:218, :254-257) */
PQLG_API int pqlg_plearner_log_alpha(pqlg_plearner h, float* out);
PQLG_API int pqlg_plearner_buffer_size(pqlg_plearner h, uint64_t* out);
PQLG_API int pqlg_plearner_set_sampler(pqlg_plearner h, int mode);
PQLG_API int pqlg_plearner_kernels_per_update(pqlg_plearner h, int* out);
/* As pqlg_vlearner_time_update, for the policy update graph. */
PQLG_API int pqlg_plearner_time_update(pqlg_plearner h, int reps, char* out, int cap);

/* ------------------------------------------------------------ actor */
typedef struct pqlg_actor_s* pqlg_actor;
typedef struct pqlg_env_s* pqlg_env;

/* ActorCore(cfg, dims)  learners.hpp:54, learners.cpp:62-76, with the
 * synthetic vectorised environment of SURVEY 8(d) in place of make_env.
 * Env/noise streams use global env indices env_offset + i. */
PQLG_API int pqlg_actor_create(const pqlg_config* cfg, const pqlg_task_dims* dims, void* stream,
                               pqlg_actor* out);
/* A shard of a multi-GPU actor: cfg->env_offset / envs_total
 * place its envs in the global index space (streams, noise schedule), and
 * the running normalizer is merged over the communicator every step (an
 * all-gather of each shard's batch mean / M2 / n, combined in rank order),
 * so every shard normalises with the statistics of all envs.  A world-1
 * communicator reproduces pqlg_actor_create bit for bit. */
PQLG_API int pqlg_actor_create_sharded(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                       pqlg_comm comm, void* stream, pqlg_actor* out);
PQLG_API int pqlg_actor_destroy(pqlg_actor h);
/* adopt_policy: PolicyHandle::adopt, equal-or-newer (learners.cpp:37-42) */
PQLG_API int pqlg_actor_adopt_policy(pqlg_actor h, const float* flat_host, int64_t version);
/* rollout_step() (learners.cpp:80-116): enqueues one step; *out receives
 * device views of the StepSlice, valid for the next two rollout_steps (the
 * actor rotates three output buffer sets), so consumers on other streams can
 * read step t while step t+1 runs; order them before step t+2 (events). */
PQLG_API int pqlg_actor_rollout_step(pqlg_actor h, pqlg_step_slice* out);
/* The cudaEvent_t (as void*) recorded on the actor's stream after the last
 * rollout_step: a consumer on another stream orders its reads of the slice
 * after it with pqlg_{vlearner,plearner}_wait_event (the threading contract's
 * exported events).  NULL before the first rollout_step. */
PQLG_API int pqlg_actor_step_event(pqlg_actor h, void** event_out);
/* The actor's stream waits for an event (e.g. a learner's record_event after
 * ingesting step t) before reusing step t's buffers at step t + 3. */
PQLG_API int pqlg_actor_wait_event(pqlg_actor h, void* event);
/* n steps replayed from CUDA graphs (no slices returned). */
PQLG_API int pqlg_actor_rollout_n(pqlg_actor h, int n);
/* norm(): the running NormStats (host copies); synchronizes. */
PQLG_API int pqlg_actor_norm(pqlg_actor h, int64_t* count, double* mean_host, double* m2_host);
PQLG_API int pqlg_actor_policy_version(pqlg_actor h, int64_t* out);
/* what: 0 obs [N x D] f32, 1 actions [N x A] f32, 2 noise streams [N] u64,
 * 3 episode steps [N] i64, 4 env streams [N] u64, 5 policy params, 6 status */
PQLG_API int pqlg_actor_read(pqlg_actor h, int what, void* host_out);
/* The last rollout_step's StepSlice (messages.hpp:31-35) as dense host rows:
 * obs / boot_obs [N x obs_dim], act [N x act_dim], rew [N], term / trunc [N]
 * (any pointer may be NULL); synchronizes.  The copy-out path of a host
 * consumer (the reference's StepSlice-by-value ActorCore::rollout_step). */
PQLG_API int pqlg_actor_read_slice(pqlg_actor h, float* obs, float* act, float* boot_obs,
                                   float* rew, uint8_t* term, uint8_t* trunc);
PQLG_API int pqlg_actor_kernels_per_step(pqlg_actor h, int* out);
/* As pqlg_vlearner_time_update for the rollout-step graphs; one replay runs
 * three consecutive steps (every output buffer set once). */
PQLG_API int pqlg_actor_time_steps(pqlg_actor h, int reps, char* out, int cap);

/* ------------------------------------------------ run_parallel (pipeline)
 * The three PQL processes (Actor, V-learner, P-learner; SPEC.md:438-501,
 * run.hpp:38) as three host threads on one GPU, each core on its own CUDA
 * stream, paced by RatioGate's counter rule (ratio_gate.hpp:17-112) and
 * exchanging device-resident data / snapshots through bounded channels and
 * latest-wins slots (mailbox.hpp) with the actor as the hub. */
typedef struct pqlg_pipeline_s* pqlg_pipeline;

enum { PQLG_PROC_ACTOR = 0, PQLG_PROC_VLEARNER = 1, PQLG_PROC_PLEARNER = 2 };

/* RatioConfig (ratio_gate.hpp:17-25) + the run_parallel design constants
 * (SPEC.md:486-492): rollout horizon H, channel capacity, K_pub. */
typedef struct {
  double beta_av;       /* c_a / c_v target (1/8) */
  double beta_pv;       /* c_p / c_v target (1/2) */
  double slack_a, slack_p, slack_v;
  int64_t warm_up;      /* rollout steps before any gating (32) */
  int free_running;
  int horizon;          /* rollout steps per actor iteration (4) */
  int channel_capacity; /* batches in flight per channel (8) */
  int publish_every;    /* learner updates per snapshot (8) */
} pqlg_ratio_config;

/* RunReport (run.hpp:11-31), the fields this pipeline produces. */
typedef struct {
  int ok;
  int64_t c_a, c_v, c_p, env_steps;
  double wall_s, ratio_av, ratio_pv;
  int64_t batches_sent, batches_consumed_v, batches_consumed_p;
  int64_t seq_duplicates, seq_gaps;
  int64_t max_policy_staleness; /* publish intervals */
  int64_t policy_version, critic_version;
  float last_critic_loss, last_actor_loss;
} pqlg_run_report;

PQLG_API void pqlg_ratio_config_default(pqlg_ratio_config* cfg);
/* RatioGate::may_proceed (ratio_gate.hpp:44-60): 1 proceed, 0 wait, -1 bad args. */
PQLG_API int pqlg_ratio_may_proceed(int proc, int64_t c_a, int64_t c_v, int64_t c_p,
                                    const pqlg_ratio_config* cfg);
PQLG_API int pqlg_pipeline_create(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                  const pqlg_ratio_config* ratio, uint64_t init_rng_seed,
                                  pqlg_pipeline* out);
/* Runs until c_a >= actor_steps or max_seconds elapsed; joins all threads.
 * A non-finite update aborts the run with PQLG_ENONFINITE. Once per pipeline. */
PQLG_API int pqlg_pipeline_run(pqlg_pipeline h, int64_t actor_steps, double max_seconds,
                               pqlg_run_report* out);
PQLG_API int pqlg_pipeline_destroy(pqlg_pipeline h);
/* Test hooks for the snapshot exchange: before run, record a host copy of
 * every critic snapshot the V-learner publishes; after run, the P-learner's
 * critic replicas vs the snapshot published under the version it holds
 * (*max_abs_diff = 0 when they are that snapshot; -1 when it holds none). */
PQLG_API int pqlg_pipeline_record_snapshots(pqlg_pipeline h, int on);
PQLG_API int pqlg_pipeline_check_critics(pqlg_pipeline h, int64_t* p_version,
                                         double* max_abs_diff);

/* ------------------------------------------------------------ metrics CSV
 * MetricsRow / MetricsWriter (metrics.hpp:9-32, metrics.cpp:8-29):
 * header "wall_clock_s,env_steps,c_a,c_v,c_p,eval_return_mean,
 * eval_return_stderr,critic_loss_ema,actor_loss_ema", then one flushed line
 * per row formatted "%.3f,%lld,%lld,%lld,%lld,%.6g,%.6g,%.6g,%.6g" --
 * byte-identical to the reference writer.  Host only (no GPU work). */
typedef struct {
  double wall_clock_s;
  int64_t env_steps, c_a, c_v, c_p;
  double eval_return_mean, eval_return_stderr;
  double critic_loss_ema, actor_loss_ema;
} pqlg_metrics_row;
typedef struct pqlg_metrics_s* pqlg_metrics;
PQLG_API const char* pqlg_metrics_header(void);
/* Truncates `path` and writes the header; PQLG_EINVAL if it cannot be opened. */
PQLG_API int pqlg_metrics_open(const char* path, pqlg_metrics* out);
PQLG_API int pqlg_metrics_append(pqlg_metrics h, const pqlg_metrics_row* row);
PQLG_API int pqlg_metrics_close(pqlg_metrics h);

/* The evaluator + metrics writer of run_parallel / run_synchronous
 * (SPEC.md:461, :494): every interval_s of wall clock (parallel) or every
 * every_actor_steps rollout steps (synchronous) the actor's current policy
 * and normalizer are evaluated (evaluate_policy, eval_episodes episodes,
 * eval_seed) and a row is appended; a last row is written at the end of the
 * run.  Loss EMAs: the first sample seeds them, then ema = f*ema + (1-f)*x
 * with f = `ema`, sampled at every snapshot publication (K_pub updates). */
typedef struct {
  const char* path;
  double interval_s;
  int64_t every_actor_steps;
  int eval_episodes;
  uint64_t eval_seed;
  double ema;
} pqlg_metrics_config;
PQLG_API void pqlg_metrics_config_default(pqlg_metrics_config* m);
/* Before pqlg_pipeline_run; path == NULL disables. */
PQLG_API int pqlg_pipeline_set_metrics(pqlg_pipeline h, const pqlg_metrics_config* m);

/* run_synchronous (algos sync_ddpg_n / sync_sac_n): the
 * same three cores on one stream in one host thread, in Algorithm order:
 * roll out H steps (ingest into both learners), then H / beta_av critic
 * updates, a policy update after every critic update that keeps
 * c_p <= beta_pv * c_v, critic snapshot -> P-learner and policy snapshot ->
 * actor + V-learner every publish_every updates.  Bit-deterministic for a
 * fixed seed (the metrics CSV differs only in its wall_clock_s column).
 * metrics nullable. */
PQLG_API int pqlg_run_synchronous(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                  const pqlg_ratio_config* ratio, uint64_t init_rng_seed,
                                  int64_t actor_steps, const pqlg_metrics_config* metrics,
                                  pqlg_run_report* out);

/* evaluate_policy (learners.cpp:280-325) on the synthetic task: a fresh env
 * of `episodes` rows seeded with eval_seed, each row one full episode of the
 * deterministic policy (flat host params, cfg->hidden / hidden_layers /
 * max_episode_len) on apply_stats(norm, obs); mean and standard error of the
 * undiscounted returns (returns_host nullable [episodes]).  episodes < 1 ->
 * PQLG_EINVAL. */
PQLG_API int pqlg_evaluate(const pqlg_config* cfg, const pqlg_task_dims* dims,
                           const float* policy_host, const pqlg_norm_stats* norm, int episodes,
                           uint64_t eval_seed, double* returns_host, double* mean,
                           double* stderr_out);

/* The synthetic EnvBatch on its own (vecenv.hpp:44-81 contract). */
PQLG_API int pqlg_env_create(int n_envs, int obs_dim, int act_dim, uint64_t seed,
                             int max_episode_len, int env_offset, float low, float high,
                             void* stream, pqlg_env* out);
PQLG_API int pqlg_env_destroy(pqlg_env h);
/* reset_all() (vecenv.cpp:53-60); writes the observations. */
PQLG_API int pqlg_env_reset_all(pqlg_env h, float* obs_dev, int64_t ld);
/* step(actions) (vecenv.cpp:84-106): next obs, terminal obs (valid on done
 * rows), rewards, dones, truncated.  Non-finite action -> PQLG_ENONFINITE. */
PQLG_API int pqlg_env_step(pqlg_env h, const float* act_dev, int64_t ld_act, float* next_obs_dev,
                           float* terminal_obs_dev, float* rew_dev, uint8_t* done_dev,
                           uint8_t* trunc_dev, int64_t ld_obs);

/* explore::apply_noise (noise.hpp:56-72) on device, bit-exact: per-row
 * polar-method normals from the row's SplitMix state (advanced in place). */
PQLG_API int pqlg_k_apply_noise(float* act_dev, int64_t ld, int n, int act_dim,
                                const float* sigma_dev, float low, float high,
                                uint64_t* states_dev, void* stream);
/* The replay sampler's index draw alone (test hook): B indices of
 * uniform_int_distribution<size_t>(0, count-1) over the Philox URBG
 * (key, *counter), drawn by the device sampler (parallel draws, and the
 * sequential Lemire redo when a draw is rejected) for any virtual live count;
 * *counter advances by the draws consumed; *rejected (nullable) = 1 when the
 * redo path ran.  Synchronizes. */
PQLG_API int pqlg_k_sample_indices(uint64_t key, uint64_t* counter, uint64_t count,
                                   uint64_t batch, uint64_t* out_host, uint32_t* rejected);
/* RunningNormalizer::update (normalizer.hpp:33-50, :73-83) on device; also
 * writes the fp32 apply constants.  Synchronizes. */
PQLG_API int pqlg_k_normalizer_update(int64_t* count_dev, double* mean_dev, double* m2_dev,
                                      const float* batch_dev, int64_t ld, int rows, int dim,
                                      float* mean_f_dev, float* inv_f_dev, void* stream);

/* One evaluation context (the metrics loops' reusable Evaluator) run over
 * n_policies policy vectors in turn, all with `norm`: returns
 * [n_policies x episodes] and the per-policy mean / stderr, each equal to a
 * fresh pqlg_evaluate of that policy (test hook).  Synchronizes. */
PQLG_API int pqlg_k_evaluate_seq(const pqlg_config* cfg, const pqlg_task_dims* dims,
                                 const float* policies_host, int n_policies,
                                 const pqlg_norm_stats* norm, int episodes, uint64_t eval_seed,
                                 double* returns_host, double* mean, double* stderr_out);

/* ------------------------------------------------------------ checkpoints
 * The reference's on-disk format, byte for byte (fa::save_checkpoint /
 * load_checkpoint, src/funcapprox/checkpoint.cpp:35-91): "PQLCKPT\x01",
 * named nets (layer sizes, u8 activations: ReLU hidden, identity output,
 * flat f32 params in Mlp layout), then the normalizer (dim, count, mean, m2).
 * IO / format errors -> PQLG_EINVAL. */
PQLG_API int pqlg_checkpoint_write(const char* path, int n_nets, const char* const* names,
                                   const int32_t* n_layers, const int32_t* const* sizes,
                                   const float* const* flats, int64_t count, const double* mean,
                                   const double* m2, int dim);
/* Reads every net's parameters concatenated in file order into flat_out
 * (nullable: sizes only) and the normalizer (mean / m2 nullable). */
PQLG_API int pqlg_checkpoint_read(const char* path, int* n_nets, int64_t* n_params,
                                  float* flat_out, int64_t* count, double* mean, double* m2,
                                  int* dim);
/* Cores: V-learner nets "q1" "q2" "q1_target" "q2_target" "policy" (lagged),
 * P-learner "policy" "q1" "q2", actor "policy"; the normalizer is the one the
 * core last adopted (the actor's own running stats).  load restores the nets
 * by name (shape-checked) and adopts the normalizer. */
PQLG_API int pqlg_vlearner_save(pqlg_vlearner h, const char* path);
PQLG_API int pqlg_vlearner_load(pqlg_vlearner h, const char* path);
PQLG_API int pqlg_plearner_save(pqlg_plearner h, const char* path);
PQLG_API int pqlg_plearner_load(pqlg_plearner h, const char* path);
PQLG_API int pqlg_actor_save(pqlg_actor h, const char* path);
PQLG_API int pqlg_actor_load(pqlg_actor h, const char* path);

#ifdef __cplusplus
}
#endif

#endif /* PQLG_H_ */
