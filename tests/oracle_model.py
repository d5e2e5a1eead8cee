"""Composition of the oracle restatement into the reference's runtime-core
steps (tests only).  The arithmetic is in oracle/pql_oracle.c; this file only
sequences the calls the way proj/src/runtime/learners.cpp does."""
from __future__ import annotations

import numpy as np

from oracle_lib import (MT64, STREAM_SAC, STREAM_SAMPLE, acts_arr, derive_seed, orc, param_count,
                        ptr, sizes_arr)


def f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def normalize(count, mean, m2, x):
    x = f32(x)
    out = np.empty_like(x)
    orc().orc_normalize_apply(int(count), ptr(np.ascontiguousarray(mean, np.float64)),
                              ptr(np.ascontiguousarray(m2, np.float64)), ptr(x), ptr(out),
                              x.shape[0], x.shape[1])
    return out


def mlp_forward(flat, sizes, x):
    L = len(sizes) - 1
    y = np.zeros((x.shape[0], sizes[-1]), np.float32)
    orc().orc_mlp_forward(ptr(f32(flat)), ptr(sizes_arr(sizes)), ptr(acts_arr(L)), L,
                          ptr(f32(x)), x.shape[0], ptr(y), None)
    return y


def policy_act(flat, sizes, x, low=-1.0, high=1.0):
    y = np.zeros((x.shape[0], sizes[-1]), np.float32)
    orc().orc_policy_act(ptr(f32(flat)), ptr(sizes_arr(sizes)), len(sizes) - 1, ptr(f32(x)),
                         x.shape[0], np.float32(low), np.float32(high), ptr(y))
    return y


class EpsStream:
    """The learners' eps draws (one normal_distribution<float> per update,
    learners.cpp:171-173, :247-249) over make_rng(seed, sac, learner)
    (mt19937_64) or the device's Philox URBG with the same key."""

    def __init__(self, seed, learner, philox=False):
        self.key = derive_seed(seed, STREAM_SAC, learner)
        self.philox = philox
        self.mt = MT64(self.key)
        self.ctr = np.zeros(1, np.uint64)

    def draw(self, B, A):
        out = np.zeros((B, A), np.float32)
        orc().orc_normals(1 if self.philox else 0, None if self.philox else self.mt.handle,
                          self.key, ptr(self.ctr), B * A, ptr(out))
        return out


def adam(p, g, m, v, t, lr):
    bc1 = np.zeros(1, np.float32)
    bc2 = np.zeros(1, np.float32)
    orc().orc_adam_bias_corrections(t, ptr(bc1), ptr(bc2))
    orc().orc_adam_update(ptr(p), ptr(g), ptr(m), ptr(v), p.size, np.float32(lr), np.float32(0.9),
                          np.float32(0.999), np.float32(1e-8), bc1[0], bc2[0])


class OracleVUpdate:
    """CriticLearnerCore::update (learners.cpp:157-188) on explicit state,
    sampling with mt19937_64 (make_rng(seed, sample, 1)) or Philox."""

    def __init__(self, D, A, hidden, n_hidden, B, q1, q2, policy, seed=0, lr=5e-4, tau=0.05,
                 philox=False, distributional=False, n_atoms=51, vmin=-10.0, vmax=10.0,
                 sac=False, log_alpha=0.0):
        self.D, self.A, self.B = D, A, B
        self.ps = [D] + [hidden] * n_hidden + [2 * A if sac else A]
        self.qs = [D + A] + [hidden] * n_hidden + [n_atoms if distributional else 1]
        self.L = n_hidden + 1
        self.sac, self.log_alpha = sac, np.float32(log_alpha)
        self.eps = EpsStream(seed, 1, philox) if sac else None
        self.q = [f32(q1).copy(), f32(q2).copy()]
        self.qt = [self.q[0].copy(), self.q[1].copy()]
        self.pol = f32(policy).copy()
        P = param_count(self.qs)
        self.m = [np.zeros(P, np.float32) for _ in range(2)]
        self.v = [np.zeros(P, np.float32) for _ in range(2)]
        self.t = 0
        self.lr, self.tau = lr, tau
        self.philox = philox
        self.key = derive_seed(seed, STREAM_SAMPLE, 1)
        self.ctr = np.zeros(1, np.uint64)
        self.mt = MT64(self.key)
        self.rows = None
        self.norm = (0, np.zeros(D), np.zeros(D))
        self.distributional = distributional
        self.n_atoms, self.vmin, self.vmax = n_atoms, vmin, vmax

    def set_rows(self, obs, act, boot, ret, eff):
        self.rows = [f32(obs), f32(act), f32(boot), f32(ret), f32(eff)]

    def sample(self):
        count = self.rows[3].shape[0]
        idx = np.zeros(self.B, np.uint64)
        if self.philox:
            orc().orc_sample_indices_philox(self.key, ptr(self.ctr), count, self.B, ptr(idx))
        else:
            orc().orc_sample_indices_mt(self.mt.handle, count, self.B, ptr(idx))
        return idx

    def step(self):
        idx = self.sample().astype(np.int64)
        obs, act, boot, ret, eff = (r[idx] for r in self.rows)
        c, mean, m2 = self.norm
        obs_n = normalize(c, mean, m2, obs)
        boot_n = normalize(c, mean, m2, boot)
        P = param_count(self.qs)
        dq = [np.zeros(P, np.float32), np.zeros(P, np.float32)]
        loss = np.zeros(1, np.float32)
        y = np.zeros(self.B, np.float32)
        args = (ptr(self.pol), ptr(sizes_arr(self.ps)), ptr(self.q[0]), ptr(self.q[1]),
                ptr(self.qt[0]), ptr(self.qt[1]), ptr(sizes_arr(self.qs)), self.L, ptr(obs_n),
                ptr(f32(act)), ptr(boot_n), ptr(f32(ret)), ptr(f32(eff)), self.B, self.D, self.A,
                np.float32(-1), np.float32(1))
        if self.sac:
            eps = self.eps.draw(self.B, self.A)
            alpha = np.float32(np.exp(self.log_alpha))
            rc = orc().orc_sac_critic_loss(*args, alpha, ptr(eps), ptr(loss), ptr(y), ptr(dq[0]),
                                           ptr(dq[1]))
        elif self.distributional:
            rc = orc().orc_c51_critic_loss(*args, self.n_atoms, np.float32(self.vmin),
                                           np.float32(self.vmax), ptr(loss), ptr(dq[0]),
                                           ptr(dq[1]))
        else:
            rc = orc().orc_ddpg_critic_loss(*args, ptr(loss), ptr(y), ptr(dq[0]), ptr(dq[1]))
        if rc != 0:
            raise FloatingPointError("non-finite target/loss")
        scales = []
        for k in range(2):
            scales.append(orc().orc_clip_global_norm(ptr(dq[k]), P, np.float32(0.5)))
        self.t += 1
        for k in range(2):
            adam(self.q[k], dq[k], self.m[k], self.v[k], self.t, self.lr)
        for k in range(2):
            orc().orc_lerp_towards(ptr(self.qt[k]), ptr(self.q[k]), P, np.float32(self.tau))
        return float(loss[0]), dict(idx=idx, y=y, dq=dq, scales=scales)


class OraclePUpdate:
    """PolicyLearnerCore::update (learners.cpp:239-270) on explicit state."""

    def __init__(self, D, A, hidden, n_hidden, B, policy, q1, q2, seed=0, lr=5e-4, philox=False,
                 distributional=False, n_atoms=51, vmin=-10.0, vmax=10.0, sac=False):
        self.D, self.A, self.B = D, A, B
        self.ps = [D] + [hidden] * n_hidden + [2 * A if sac else A]
        self.sac = sac
        self.eps = EpsStream(seed, 2, philox) if sac else None
        # log alpha and its Adam state (learners.cpp:217-219)
        self.alpha_p = np.zeros(1, np.float32)
        self.alpha_m = np.zeros(1, np.float32)
        self.alpha_v = np.zeros(1, np.float32)
        self.qs = [D + A] + [hidden] * n_hidden + [n_atoms if distributional else 1]
        self.L = n_hidden + 1
        self.pol = f32(policy).copy()
        self.q = [f32(q1).copy(), f32(q2).copy()]
        P = param_count(self.ps)
        self.m = np.zeros(P, np.float32)
        self.v = np.zeros(P, np.float32)
        self.t = 0
        self.lr = lr
        self.philox = philox
        self.key = derive_seed(seed, STREAM_SAMPLE, 2)
        self.ctr = np.zeros(1, np.uint64)
        self.mt = MT64(self.key)
        self.states = None
        self.norm = (0, np.zeros(D), np.zeros(D))
        self.distributional = distributional
        self.n_atoms, self.vmin, self.vmax = n_atoms, vmin, vmax

    def step(self):
        count = self.states.shape[0]
        idx = np.zeros(self.B, np.uint64)
        if self.philox:
            orc().orc_sample_indices_philox(self.key, ptr(self.ctr), count, self.B, ptr(idx))
        else:
            orc().orc_sample_indices_mt(self.mt.handle, count, self.B, ptr(idx))
        c, mean, m2 = self.norm
        s = normalize(c, mean, m2, self.states[idx.astype(np.int64)])
        P = param_count(self.ps)
        dp = np.zeros(P, np.float32)
        loss = np.zeros(1, np.float32)
        args = (ptr(self.pol), ptr(sizes_arr(self.ps)), ptr(self.q[0]), ptr(self.q[1]),
                ptr(sizes_arr(self.qs)), self.L, ptr(s), self.B, self.D, self.A, np.float32(-1),
                np.float32(1))
        if self.sac:
            eps = self.eps.draw(self.B, self.A)
            alpha = np.float32(np.exp(self.alpha_p[0]))
            mean_logp = np.zeros(1, np.float32)
            rc = orc().orc_sac_actor_loss(*args, alpha, ptr(eps), ptr(loss), ptr(mean_logp),
                                          ptr(dp))
            if rc != 0:
                raise FloatingPointError("non-finite actor loss")
            # sac_alpha_loss (sac.hpp:117-125) + adam_step on log alpha
            drift = np.float32(mean_logp[0] + np.float32(-self.A))
            self.t += 1
            adam(self.alpha_p, f32([-drift]), self.alpha_m, self.alpha_v, self.t, self.lr)
            orc().orc_clip_global_norm(ptr(dp), P, np.float32(0.5))
            adam(self.pol, dp, self.m, self.v, self.t, self.lr)
            return float(loss[0]), dict(idx=idx, dp=dp, qscale=1.0, mean_logp=float(mean_logp[0]))
        if self.distributional:
            rc = orc().orc_c51_actor_loss(*args, self.n_atoms, np.float32(self.vmin),
                                          np.float32(self.vmax), ptr(loss), ptr(dp))
        else:
            rc = orc().orc_ddpg_actor_loss(*args, ptr(loss), ptr(dp))
        if rc != 0:
            raise FloatingPointError("non-finite actor loss")
        # scale of the objective's terms: mean_b |min(Q1, Q2)(s, pi(s))| -- the
        # loss itself is a mean of terms that largely cancel, so tolerances on
        # it are stated relative to this scale
        a = policy_act(self.pol, self.ps, s)
        xq = np.concatenate([s, a], axis=1)
        q1 = mlp_forward(self.q[0], self.qs, xq)
        q2 = mlp_forward(self.q[1], self.qs, xq)
        qscale = float(np.mean(np.abs(np.minimum(q1, q2)))) if not self.distributional else 1.0
        orc().orc_clip_global_norm(ptr(dp), P, np.float32(0.5))
        self.t += 1
        adam(self.pol, dp, self.m, self.v, self.t, self.lr)
        return float(loss[0]), dict(idx=idx, dp=dp, qscale=qscale)


class OracleEnv:
    """The synthetic EnvBatch of the restatement (pql_oracle.c orc_env_*)."""

    def __init__(self, N, D, A, seed, max_len):
        self.N, self.D, self.A = N, D, A
        self.h = orc().orc_env_create(N, D, A, seed, max_len)

    def observe(self):
        o = np.zeros((self.N, self.D), np.float32)
        orc().orc_env_observe(self.h, ptr(o))
        return o

    def step(self, act):
        act = f32(act)
        nxt = np.zeros((self.N, self.D), np.float32)
        term_obs = np.zeros((self.N, self.D), np.float32)
        rew = np.zeros(self.N, np.float32)
        done = np.zeros(self.N, np.uint8)
        trunc = np.zeros(self.N, np.uint8)
        rc = orc().orc_env_step(self.h, ptr(act), ptr(nxt), ptr(term_obs), ptr(rew), ptr(done),
                                ptr(trunc))
        if rc:
            raise FloatingPointError("non-finite action")
        return nxt, term_obs, rew, done, trunc

    def __del__(self):
        try:
            orc().orc_env_destroy(self.h)
        except Exception:
            pass


class OracleActor:
    """ActorCore::rollout_step (learners.cpp:80-116) over the synthetic env."""

    def __init__(self, N, D, A, hidden, n_hidden, policy, seed=0, max_len=1000,
                 sigma_min=0.05, sigma_max=0.8):
        from oracle_lib import STREAM_NOISE
        self.N, self.D, self.A = N, D, A
        self.ps = [D] + [hidden] * n_hidden + [A]
        self.pol = f32(policy).copy()
        self.env = OracleEnv(N, D, A, seed, max_len)
        self.obs = self.env.observe()
        self.count = np.zeros(1, np.int64)
        self.mean = np.zeros(D)
        self.m2 = np.zeros(D)
        self.sigma = np.zeros(N, np.float32)
        orc().orc_build_schedule(np.float32(sigma_min), np.float32(sigma_max), N, ptr(self.sigma))
        self.noise = np.array([derive_seed(seed, STREAM_NOISE, i) for i in range(N)], np.uint64)

    def step(self):
        obs_norm = normalize(int(self.count[0]), self.mean, self.m2, self.obs)
        act = policy_act(self.pol, self.ps, obs_norm)
        pre_noise = act.copy()
        orc().orc_apply_noise(ptr(act), self.N, self.A, ptr(self.sigma), np.float32(-1),
                              np.float32(1), ptr(self.noise))
        nxt, term_obs, rew, done, trunc = self.env.step(act)
        term = (done.astype(bool) & ~trunc.astype(bool)).astype(np.uint8)
        boot = np.where(done[:, None].astype(bool), term_obs, nxt)
        obs = self.obs
        orc().orc_norm_update(ptr(self.count), ptr(self.mean), ptr(self.m2), ptr(obs), self.N,
                              self.D)
        self.obs = nxt
        return dict(obs=obs, act=act, pre_noise=pre_noise, boot=f32(boot), rew=rew, term=term,
                    trunc=trunc)
