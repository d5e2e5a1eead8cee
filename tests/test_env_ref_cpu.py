"""The synthetic task, the actor step and evaluation pinned to the reference
itself (CPU, no GPU needed).

oracle/ref_harness.cpp defines SyntheticEnv, an EnvBatch subclass built
through the reference's protected constructor and virtuals
(vecenv.hpp:62-69), and hands it to the reference's own code through the
`make_env` link seam, so these fixtures come from the unmodified
EnvBatch::reset_all / step (vecenv.cpp:73-106), rt::ActorCore
(learners.cpp:62-116) and rt::evaluate_policy (learners.cpp:280-325):
  tests/golden/env.npz, actor_core.npz, evaluate.npz  (oracle/make_golden.py)
Here the C restatement (pql_oracle.c: orc_env_*, orc_evaluate, and the
OracleActor composition) is checked against them bit for bit; the GPU tests
(test_actor_gpu.py, test_evaluate_gpu.py) check the device against the same
fixtures.
"""
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import orc, ptr, ref, sizes_arr, traj_hash
from oracle_model import OracleActor, OracleEnv, f32

GOLDEN = Path(__file__).resolve().parent / "golden"


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


@pytest.mark.parametrize("k", [0, 1, 2])
def test_oracle_env_matches_reference_env_golden(k):
    G = np.load(GOLDEN / "env.npz")
    N, D, A, max_len, T, seed = (int(x) for x in G[f"env{k}_args"])
    o = OracleEnv(N, D, A, seed, max_len)
    assert np.array_equal(bits(o.observe()), bits(G[f"env{k}_obs0"]))
    for t in range(T):
        nxt, term_obs, rew, done, trunc = o.step(G[f"env{k}_act"][t])
        assert np.array_equal(done, G[f"env{k}_done"][t]), t
        assert np.array_equal(trunc, G[f"env{k}_trunc"][t]), t
        assert np.array_equal(bits(rew), bits(G[f"env{k}_rew"][t])), t
        term_obs[done == 0] = 0.0
        assert traj_hash(nxt) == G[f"env{k}_hash"][t, 0], t
        assert traj_hash(term_obs) == G[f"env{k}_hash"][t, 1], t
        if f"env{k}_next" in G:
            assert np.array_equal(bits(nxt), bits(G[f"env{k}_next"][t]))
    assert np.array_equal(bits(nxt), bits(G[f"env{k}_last"]))
    # non-finite action: EnvBatch::step throws runtime_error (vecenv.cpp:87-89)
    assert int(G[f"env{k}_nan_rc"][0]) == -2
    with pytest.raises(FloatingPointError):
        o.step(np.full((N, A), np.nan, np.float32))


def test_env_golden_exercises_terminals_and_truncations():
    G = np.load(GOLDEN / "env.npz")
    terms = sum(int(np.sum(G[f"env{k}_done"] & (1 - G[f"env{k}_trunc"]))) for k in range(3))
    truncs = sum(int(np.sum(G[f"env{k}_trunc"])) for k in range(3))
    assert terms > 0 and truncs > 0


@pytest.mark.parametrize("k", [0, 1])
def test_oracle_actor_matches_reference_actor_core(k):
    """OracleActor (normalize -> policy -> apply_noise -> env.step -> term /
    boot -> normalizer.update) reproduces the reference's ActorCore
    rollout_step StepSlices and normalizer bit for bit."""
    G = np.load(GOLDEN / "actor_core.npz")
    N, D, A, H, seed, max_len, T, sac = (int(x) for x in G[f"ac{k}_args"])
    if f"ac{k}_policy" in G:
        pol = G[f"ac{k}_policy"]
    else:
        R = ref()
        if R is None:
            pytest.skip("oracle/_ref not built")
        from oracle_lib import param_count
        pol = np.zeros(param_count([D, H, H, A]), np.float32)
        R.ref_policy_init(D, A, H, seed, ptr(pol))
        assert traj_hash(pol) == G[f"ac{k}_policy_hash"][0]
    o = OracleActor(N, D, A, H, 2, pol, seed=seed, max_len=max_len)
    for t in range(T):
        w = o.step()
        for key in ("obs", "act", "boot", "rew"):
            assert np.array_equal(bits(w[key]), bits(G[f"ac{k}_{key}"][t])), (t, key)
        for key in ("term", "trunc"):
            assert np.array_equal(w[key], G[f"ac{k}_{key}"][t]), (t, key)
    norm = G[f"ac{k}_norm"]
    assert o.count[0] == int(norm[0])
    assert np.array_equal(o.mean, norm[1:1 + D]) and np.array_equal(o.m2, norm[1 + D:])


@pytest.mark.parametrize("k", [0, 1, 2])
def test_oracle_evaluate_matches_reference_evaluate_policy(k):
    G = np.load(GOLDEN / "evaluate.npz")
    D, A, H, nh, M, seed, max_len, sac, count = (int(x) for x in G[f"ev{k}_args"])
    assert not sac
    ps = [D] + [H] * nh + [A]
    ret = np.zeros(M)
    mu, se = np.zeros(1), np.zeros(1)
    assert orc().orc_evaluate(ptr(G[f"ev{k}_policy"]), ptr(sizes_arr(ps)), nh + 1, count,
                              ptr(G[f"ev{k}_mean"]), ptr(G[f"ev{k}_m2"]), M, seed, D, A,
                              np.float32(-1), np.float32(1), max_len, ptr(ret), ptr(mu),
                              ptr(se)) == 0
    assert mu[0] == G[f"ev{k}_result"][0] and se[0] == G[f"ev{k}_result"][1]


def test_live_reference_env_matches_oracle_random_configs():
    """Fresh configurations (not in the fixtures): the reference's
    EnvBatch::step on SyntheticEnv vs the restatement, bit for bit."""
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    rng = np.random.default_rng(9)
    for N, D, A, max_len, seed in ((17, 3, 1, 5, 11), (50, 33, 7, 9, 12), (8, 211, 20, 3, 13)):
        obs0 = np.zeros((N, D), np.float32)
        h = R.ref_synth_env_create(N, D, A, seed, max_len, np.float32(-1), np.float32(1), 1,
                                   ptr(obs0))
        o = OracleEnv(N, D, A, seed, max_len)
        assert np.array_equal(bits(obs0), bits(o.observe()))
        for t in range(25):
            a = f32(rng.uniform(-2, 2, (N, A)))
            nxt, term_obs = np.zeros((N, D), np.float32), np.zeros((N, D), np.float32)
            rew = np.zeros(N, np.float32)
            done, trunc = np.zeros(N, np.uint8), np.zeros(N, np.uint8)
            assert R.ref_synth_env_step(h, ptr(a), ptr(nxt), ptr(term_obs), ptr(rew), ptr(done),
                                        ptr(trunc)) == 0
            w = o.step(a)
            assert np.array_equal(bits(nxt), bits(w[0]))
            assert np.array_equal(bits(rew), bits(w[2]))
            assert np.array_equal(done, w[3]) and np.array_equal(trunc, w[4])
            d = done.astype(bool)
            assert np.array_equal(bits(term_obs[d]), bits(w[1][d]))
        ep = np.zeros(N, np.int64)
        R.ref_synth_env_episode_steps(h, ptr(ep))
        R.ref_synth_env_destroy(h)
