/*
 * pql_oracle.h -- CPU restatement of the reference's learner/actor hot path.
 *
 * TEST INFRASTRUCTURE ONLY.  This is the checker the GPU path is compared
 * against; nothing in the product (libpqlg.so, the Python mirror) links or
 * calls it.  Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline
 * leg may load it.
 *
 * Every function cites the reference file:line it restates (paths relative
 * to /root/reference/proj).  Arithmetic follows the reference's scalar
 * ground truth (include/pql/kernels/scalar.hpp) compiled with
 * -ffp-contract=off (CMakeLists.txt:13), i.e. no FMA contraction.
 *
 * Third-party arithmetic on the path (not under /root/reference) is
 * restated from GCC 13.3 libstdc++ and glibc 2.39 (the toolchain of this
 * image): std::mt19937_64, std::uniform_int_distribution<size_t> (Lemire
 * nearly-divisionless, bits/uniform_int_dist.h:257-276),
 * std::normal_distribution<float> (polar method, bits/random.tcc),
 * std::generate_canonical<float>, glibc logf.
 */
#ifndef PQL_ORACLE_H_
#define PQL_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

/* ------------------------------------------------------------ rng.hpp */
enum { ORC_STREAM_ENV = 1, ORC_STREAM_NOISE = 2, ORC_STREAM_INIT = 3, ORC_STREAM_SAMPLE = 4,
       ORC_STREAM_EVAL = 5, ORC_STREAM_SAC = 6 };
uint64_t orc_splitmix64(uint64_t x);
uint64_t orc_derive_seed(uint64_t master, uint64_t stream, uint64_t index);

/* std::mt19937_64 */
typedef struct { uint64_t mt[312]; int idx; } orc_mt64;
void orc_mt64_seed(orc_mt64* g, uint64_t seed);
uint64_t orc_mt64_next(orc_mt64* g);

/* Philox4x32-10 (Salmon et al. 2011) and the counter URBG the GPU sampler
 * uses: draw i = out[0] | out[1] << 32 of philox(ctr = {i_lo, i_hi, 0, 0},
 * key = {key_lo, key_hi}). */
void orc_philox4x32_10(const uint32_t ctr[4], const uint32_t key[2], uint32_t out[4]);
uint64_t orc_philox_draw(uint64_t key, uint64_t counter);

/* uniform_int_distribution<size_t>(0, count-1) with a 64-bit URBG.
 * kind 0: mt19937_64 state `mt`; kind 1: philox (key, *counter advanced). */
void orc_sample_indices_mt(orc_mt64* g, uint64_t count, size_t n, uint64_t* out);
void orc_sample_indices_philox(uint64_t key, uint64_t* counter, uint64_t count, size_t n,
                               uint64_t* out);

/* ------------------------------------------------------ replay (nstep.hpp) */
typedef struct {
  size_t n_envs, obs_dim, act_dim, horizon;
  float gamma;
  float* obs; /* [n_envs*horizon x obs_dim] */
  float* act; /* [n_envs*horizon x act_dim] */
  float* rew; /* [n_envs*horizon] */
  size_t* head;
  size_t* count;
} orc_nstep;

typedef struct { /* growable NStepBatch (nstep.hpp:15-29) */
  size_t rows, cap, obs_dim, act_dim;
  float *obs, *act, *boot, *ret, *eff;
} orc_batch;

orc_nstep* orc_nstep_create(size_t n_envs, size_t obs_dim, size_t act_dim, float gamma,
                            size_t horizon);
void orc_nstep_destroy(orc_nstep* a);
orc_batch* orc_batch_create(size_t obs_dim, size_t act_dim);
void orc_batch_destroy(orc_batch* b);
void orc_batch_clear(orc_batch* b);
/* NStepAssembler::push_step (nstep.hpp:58-68); rewards already scaled. */
void orc_nstep_push_step(orc_nstep* a, const float* obs, const float* act, const float* rew,
                         const uint8_t* term, const uint8_t* trunc, const float* boot,
                         orc_batch* out);

typedef struct { /* ReplayBuffer (replay_buffer.hpp:17-81) */
  size_t capacity, obs_dim, act_dim, cursor, count;
  float *obs, *act, *boot, *ret, *eff;
} orc_replay;
orc_replay* orc_replay_create(size_t capacity, size_t obs_dim, size_t act_dim);
void orc_replay_destroy(orc_replay* r);
void orc_replay_insert(orc_replay* r, const orc_batch* b);
/* ReplayBuffer::sample given precomputed indices: gathers rows into out. */
void orc_replay_gather(const orc_replay* r, const uint64_t* idx, size_t n, float* obs, float* act,
                       float* boot, float* ret, float* eff);

typedef struct { /* StateBuffer (replay_buffer.hpp:84-119) */
  size_t capacity, obs_dim, cursor, count;
  float* obs;
} orc_states;
orc_states* orc_states_create(size_t capacity, size_t obs_dim);
void orc_states_destroy(orc_states* s);
void orc_states_insert(orc_states* s, const float* rows, size_t n);

/* ------------------------------------------- normalizer.hpp / scalar.hpp */
/* apply_stats: identity if count <= 1 (normalizer.hpp:56-70). */
void orc_norm_stats_to_f32(int64_t count, const double* mean, const double* m2, size_t d,
                           float* mean_f, float* inv_f);
void orc_normalize_clip(const float* x, const float* mean, const float* inv, float* out, size_t B,
                        size_t D, float clip);
void orc_normalize_apply(int64_t count, const double* mean, const double* m2, const float* x,
                         float* out, size_t B, size_t D);
/* RunningNormalizer::update (normalizer.hpp:33-50, 73-83). */
void orc_norm_update(int64_t* count, double* mean, double* m2, const float* batch, size_t rows,
                     size_t d);

/* Sharded normalizer: a shard's batch (mean, M2), and Chan's merge of a
 * batch into (count, mean, m2) (normalizer.hpp:33-50, :73-83). */
void orc_norm_batch_stats(const float* batch, size_t rows, size_t d, double* bmean, double* bm2);
void orc_norm_merge(double* count, double* mean, double* m2, size_t d, double nb,
                    const double* bmean, const double* bm2);

/* ---------------------------------------------------------- optim.hpp */
void orc_adam_bias_corrections(int64_t t, float* bc1, float* bc2);
void orc_adam_update(float* p, const float* g, float* m, float* v, size_t n, float lr, float beta1,
                     float beta2, float eps, float bc1, float bc2);
double orc_sum_squares(const float* x, size_t n);
/* Returns the fp32 scale applied (1 if no clipping). */
float orc_clip_global_norm(float* g, size_t n, float max_norm);
void orc_lerp_towards(float* target, const float* online, size_t n, float tau);

/* ---------------------------------------------------------- noise.hpp */
void orc_build_schedule(float sigma_min, float sigma_max, size_t n, float* sigma);
/* apply_noise with per-row SplitMix streams (state advanced in place). */
void orc_apply_noise(float* actions, size_t n, size_t act_dim, const float* sigma, float low,
                     float high, uint64_t* states);
/* glibc 2.39 logf restated (table + degree-3 polynomial in double). */
float orc_glibc_logf(float x);

/* --------------------------------------------------------------- MLP */
/* Flat layout of fa::Mlp (mlp.hpp:83-88): per layer W [in x out] then b.
 * sizes has n_layers+1 entries; acts[l] = 1 for ReLU. */
size_t orc_mlp_param_count(const size_t* sizes, size_t n_layers);
/* forward; if cache != NULL it receives post-activations of every layer
 * concatenated ([B x sizes[1]], [B x sizes[2]], ...). */
void orc_mlp_forward(const float* flat, const size_t* sizes, const uint8_t* acts,
                     size_t n_layers, const float* in, size_t B, float* out, float* cache);
/* fa::backward (mlp.hpp:161-184) given cache from forward; grads accumulate
 * into `grads` (zeroed by caller); dinput optional ([B x sizes[0]]). */
void orc_mlp_backward(const float* flat, const size_t* sizes, const uint8_t* acts,
                      size_t n_layers, const float* in, const float* cache, const float* upstream,
                      size_t B, float* grads, float* dinput);

/* --------------------------------------------------------- agents */
/* DeterministicPolicy::act (policy.hpp:33-38): a = mid + half*tanh(y). */
void orc_policy_act(const float* flat, const size_t* sizes, size_t n_layers, const float* obs,
                    size_t B, float low, float high, float* act);
/* ddpg_critic_target (ddpg.hpp:24-40); returns 0 or -2 if non-finite. */
int orc_ddpg_target(const float* pol, const size_t* psizes, const float* q1t, const float* q2t,
                    const size_t* qsizes, size_t n_layers, const float* boot_norm, const float* ret,
                    const float* eff, size_t B, size_t obs_dim, size_t act_dim, float low,
                    float high, float* y);
/* ddpg_critic_loss (ddpg.hpp:50-76): loss and flat grads dq1/dq2 (zeroed
 * here). obs_norm/act are the sampled rows. Returns 0 or -2. */
int orc_ddpg_critic_loss(const float* pol, const size_t* psizes, const float* q1, const float* q2,
                         const float* q1t, const float* q2t, const size_t* qsizes,
                         size_t n_layers, const float* obs_norm, const float* act,
                         const float* boot_norm, const float* ret, const float* eff, size_t B,
                         size_t obs_dim, size_t act_dim, float low, float high, float* loss,
                         float* y_out, float* dq1, float* dq2);
/* ddpg_actor_loss (ddpg.hpp:86-118): loss and dpolicy (zeroed here). */
int orc_ddpg_actor_loss(const float* pol, const size_t* psizes, const float* q1, const float* q2,
                        const size_t* qsizes, size_t n_layers, const float* states, size_t B,
                        size_t obs_dim, size_t act_dim, float low, float high, float* loss,
                        float* dpolicy);

/* C51 (c51.hpp) */
void orc_c51_atoms(size_t n_atoms, float vmin, float vmax, float* atoms);
int orc_c51_project(const float* probs, const float* ret, const float* eff, size_t B,
                    size_t n_atoms, float vmin, float vmax, const float* atoms, float* out);
int orc_c51_critic_loss(const float* pol, const size_t* psizes, const float* q1, const float* q2,
                        const float* q1t, const float* q2t, const size_t* qsizes,
                        size_t n_layers, const float* obs_norm, const float* act,
                        const float* boot_norm, const float* ret, const float* eff, size_t B,
                        size_t obs_dim, size_t act_dim, float low, float high, size_t n_atoms,
                        float vmin, float vmax, float* loss, float* dq1, float* dq2);
int orc_c51_actor_loss(const float* pol, const size_t* psizes, const float* q1, const float* q2,
                       const size_t* qsizes, size_t n_layers, const float* states, size_t B,
                       size_t obs_dim, size_t act_dim, float low, float high, size_t n_atoms,
                       float vmin, float vmax, float* loss, float* dpolicy);

/* SAC (sac.hpp, policy.hpp:54-153) */
/* n draws of one normal_distribution<float> over mt19937_64 (kind 0, `g`)
 * or the Philox counter URBG (kind 1, key, *ctr advanced). */
void orc_normals(int kind, orc_mt64* g, uint64_t key, uint64_t* ctr, size_t n, float* out);
/* fresh normal_distribution<float> per row over SplitMix states. */
void orc_normals_rows(uint64_t* states, size_t n_rows, size_t dim, float* out);
/* GaussianPolicy::sample: psizes[n_layers] = 2 * act_dim. */
int orc_gauss_sample(const float* pol, const size_t* psizes, size_t n_layers, const float* obs,
                     const float* eps, size_t B, float low, float high, float* act, float* logp);
int orc_sac_critic_loss(const float* pol, const size_t* psizes, const float* q1p,
                        const float* q2p, const float* q1t, const float* q2t,
                        const size_t* qsizes, size_t n_layers, const float* obs_norm,
                        const float* act, const float* boot_norm, const float* ret,
                        const float* eff, size_t B, size_t obs_dim, size_t act_dim, float low,
                        float high, float alpha, const float* eps, float* loss_out,
                        float* y_out, float* dq1, float* dq2);
int orc_sac_actor_loss(const float* pol, const size_t* psizes, const float* q1p,
                       const float* q2p, const size_t* qsizes, size_t n_layers,
                       const float* states, size_t B, size_t obs_dim, size_t act_dim, float low,
                       float high, float alpha, const float* eps, float* loss_out,
                       float* mean_logp, float* dpolicy);

/* ---------------------------------------------- synthetic env */
typedef struct {
  size_t n_envs, obs_dim, act_dim, max_len;
  uint64_t seed;
  float low, high;
  float* M;           /* [obs_dim x act_dim] coupling, fixed from seed   */
  float* s;           /* [n_envs x obs_dim] state                        */
  int64_t* episode_step;
  uint64_t* rng;      /* per-env SplitMix state (vecenv.cpp:66)          */
} orc_env;
orc_env* orc_env_create(size_t n_envs, size_t obs_dim, size_t act_dim, uint64_t seed,
                        size_t max_len);
void orc_env_destroy(orc_env* e);
/* evaluate_policy (learners.cpp:280-325) on the synthetic task: a fresh env
 * of `episodes` rows (seed eval_seed, episode steps from 0), deterministic
 * policy on apply_stats(norm, obs), one episode per row; returns[episodes]
 * (double), mean and standard error as the reference computes them. */
int orc_evaluate(const float* pol, const size_t* psizes, size_t n_layers, int64_t count,
                 const double* mean, const double* m2, size_t episodes, uint64_t eval_seed,
                 size_t obs_dim, size_t act_dim, float low, float high, size_t max_len,
                 double* returns, double* mean_out, double* stderr_out);
void orc_env_observe(const orc_env* e, float* obs);
/* EnvBatch::step contract (vecenv.cpp:84-106); returns -2 on non-finite
 * action (runtime_error in the reference). */
int orc_env_step(orc_env* e, const float* actions, float* next_obs, float* terminal_obs,
                 float* rewards, uint8_t* dones, uint8_t* truncated);

#ifdef __cplusplus
}
#endif

#endif /* PQL_ORACLE_H_ */
