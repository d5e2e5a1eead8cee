"""pql_sac restatement (oracle/pql_oracle.c, sac.hpp / policy.hpp:54-153)
pinned against the compiled reference's outputs (tests/golden/sac.npz,
oracle/make_golden.py gen_sac)."""
import numpy as np

from oracle_lib import (MT64, STREAM_NOISE, STREAM_SAC, derive_seed, orc, ptr, sizes_arr)
from oracle_model import EpsStream, OraclePUpdate, OracleVUpdate, f32, normalize
from test_oracle_cpu import golden


def test_eps_stream_matches_normal_distribution_over_mt19937():
    """normal_distribution<float> over make_rng(0, sac, 1): bit-exact,
    including the cached second value of the last pair (1001 draws)."""
    G = golden("sac")
    out = np.zeros(1001, np.float32)
    g = MT64(derive_seed(0, STREAM_SAC, 1))
    orc().orc_normals(0, g.handle, 0, None, 1001, ptr(out))
    np.testing.assert_array_equal(out.view(np.uint32), G["sac_normals"].view(np.uint32))


def test_eps_stream_split_calls_restart_the_distribution():
    """Each update builds a fresh normal_distribution (learners.cpp:172): a
    second call must not reuse the first call's cached value, so two
    draws of 5 differ from one draw of 10 exactly when 5 is odd."""
    e1 = EpsStream(3, 1)
    a = np.concatenate([e1.draw(1, 5).ravel(), e1.draw(1, 5).ravel()])
    e2 = EpsStream(3, 1)
    b = e2.draw(1, 10).ravel()
    np.testing.assert_array_equal(a[:5], b[:5])
    assert not np.array_equal(a[5:], b[5:])
    e3, e4 = EpsStream(3, 1), EpsStream(3, 1)
    np.testing.assert_array_equal(np.concatenate([e3.draw(1, 4).ravel(), e3.draw(1, 6).ravel()]),
                                  e4.draw(1, 10).ravel())


def test_philox_eps_stream_counter_advances_by_two_per_candidate_pair():
    e = EpsStream(0, 1, philox=True)
    x = e.draw(7, 3)  # 21 normals = 11 accepted pairs (last value's partner discarded)
    assert np.isfinite(x).all()
    used = int(e.ctr[0])
    assert used % 2 == 0 and used >= 22
    # recomputing from the same key and counter 0 reproduces the stream
    e2 = EpsStream(0, 1, philox=True)
    np.testing.assert_array_equal(e2.draw(7, 3), x)
    assert int(e2.ctr[0]) == used


def test_gauss_sample_matches_reference():
    G = golden("sac")
    D, A, H, nh = 9, 4, 32, 2
    ps = [D] + [H] * nh + [2 * A]
    act = np.zeros((64, A), np.float32)
    logp = np.zeros(64, np.float32)
    assert orc().orc_gauss_sample(ptr(G["su_pol"]), ptr(sizes_arr(ps)), nh + 1, ptr(G["gs_obs"]),
                                  ptr(G["gs_eps"]), 64, np.float32(-1), np.float32(1), ptr(act),
                                  ptr(logp)) == 0
    # the reference's affine loops are AVX2 (FMA, lane reassociation)
    np.testing.assert_allclose(act, G["gs_act"], rtol=1e-5, atol=1e-6)
    np.testing.assert_allclose(logp, G["gs_logp"], rtol=1e-5, atol=1e-5)


def test_sac_update_k_steps_match_reference_golden():
    """3 SAC critic updates (lagged log alpha -0.7) + 3 SAC policy/alpha
    updates of the restatement vs the compiled reference."""
    G = golden("sac")
    D, A, H, nh, B, cap = (int(v) for v in G["su_dims"])
    o = OracleVUpdate(D, A, H, nh, B, G["su_q1"], G["su_q2"], G["su_pol"], sac=True,
                      log_alpha=float(G["su_log_alpha"][0]))
    o.set_rows(G["su_obs"], G["su_act"], G["su_boot"], G["su_ret"], G["su_eff"])
    o.norm = (int(G["su_norm"][0]), G["su_mean"], G["su_m2"])
    losses = [o.step()[0] for _ in range(3)]
    np.testing.assert_allclose(losses, G["su_losses"], rtol=1e-5)
    for w, arr in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        want = G["su_params"][w]
        assert np.linalg.norm(arr - want) / np.linalg.norm(want) < 1e-4
    p = OraclePUpdate(D, A, H, nh, B, G["su_pol"], G["su_q1"], G["su_q2"], sac=True)
    p.states = G["su_obs"]
    p.norm = o.norm
    pl, la = [], []
    for _ in range(3):
        pl.append(p.step()[0])
        la.append(float(p.alpha_p[0]))
    np.testing.assert_allclose(pl, G["sp_losses"], rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(la, G["sp_log_alpha"], rtol=1e-5, atol=1e-7)
    assert np.linalg.norm(p.pol - G["sp_params"]) / np.linalg.norm(G["sp_params"]) < 1e-4


def test_stochastic_actor_step_matches_reference():
    """ActorCore::rollout_step for pql_sac (learners.cpp:87-94): per-env
    fresh normal_distribution over the noise streams, squashed sample."""
    G = golden("sac")
    D, A, H, nh = 9, 4, 32, 2
    N = G["sa_obs0"].shape[0]
    ps = [D] + [H] * nh + [2 * A]
    count = np.zeros(1, np.int64)
    mean = np.zeros(D)
    m2 = np.zeros(D)
    orc().orc_norm_update(ptr(count), ptr(mean), ptr(m2), ptr(G["sa_obs0"]), N, D)
    x = normalize(int(count[0]), mean, m2, G["sa_obs1"])
    states = np.array([derive_seed(0, STREAM_NOISE, i) for i in range(N)], np.uint64)
    eps = np.zeros((N, A), np.float32)
    orc().orc_normals_rows(ptr(states), N, A, ptr(eps))
    act = np.zeros((N, A), np.float32)
    logp = np.zeros(N, np.float32)
    orc().orc_gauss_sample(ptr(G["su_pol"]), ptr(sizes_arr(ps)), nh + 1, ptr(x), ptr(eps), N,
                           np.float32(-1), np.float32(1), ptr(act), ptr(logp))
    np.testing.assert_allclose(act, G["sa_act"], rtol=1e-5, atol=1e-6)
