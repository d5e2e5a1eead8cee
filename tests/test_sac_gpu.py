"""pql_sac on the GPU (sac.hpp, policy.hpp:54-153, learners.cpp:87-94,
:168-176, :246-258) vs the oracle and the reference's golden vectors.

Bars: the eps streams (learners' Philox polar draws, the actor's per-env
normal_distribution over SplitMix) bit-exact, stream counters exact; TF32
quantities as elsewhere (losses rel 2e-3, gradients norm-wise 1e-2, weights
norm-wise 2e-3 with |dw| <= 2 lr k + 1e-3 |w|); log alpha after k updates
within 2e-3 lr-steps (the alpha gradient is the mean log-prob, a TF32
quantity)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import STREAM_NOISE, STREAM_SAC, derive_seed, orc, param_count, ptr, sizes_arr
from oracle_model import EpsStream, OraclePUpdate, OracleVUpdate, f32, normalize
from paper_2307_12983_b200 import _lib
from test_c51_gpu import pl_get, pl_ingest, pl_put
from test_vlearner_gpu import (adopt_norm, check_weights, insert_rows, params, random_rows, rel,
                               set_params)

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def cfg_sac(**kw):
    return _lib.default_config(algo=_lib.ALGO_SAC, **kw)


def make_vl(D, A, H, nh, B, cap, seed=0, init_seed=12345, n_envs=4):
    cfg = cfg_sac(batch_size=B, buffer_capacity=cap, hidden=H, hidden_layers=nh, n_envs=n_envs,
                  seed=seed)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), init_seed, None, C.byref(h))
    return h


def make_pl(D, A, H, nh, B, cap, seed=0):
    cfg = cfg_sac(batch_size=B, buffer_capacity=cap, hidden=H, hidden_layers=nh, seed=seed)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 12345, None, C.byref(h))
    return h


def v_update(h):
    l = C.c_float()
    _lib.call("pqlg_vlearner_update", h, C.byref(l))
    return l.value


def p_update(h):
    l = C.c_float()
    _lib.call("pqlg_plearner_update", h, C.byref(l))
    return l.value


def v_adopt(h, pol, log_alpha, version=1):
    _lib.call("pqlg_vlearner_adopt_policy_sac", h, ptr(f32(pol)), np.float32(log_alpha), version)


@pytest.mark.parametrize("B,A", [(64, 3), (1024, 8), (8192, 20), (1, 1), (37, 32)])
def test_eps_stream_bit_exact_and_counter_advance(B, A):
    """The device's parallel polar draws equal the sequential
    normal_distribution over the same Philox URBG (orc_normals, kind 1), for
    3 consecutive updates: the counter advance is exact too.  B*A odd for
    (64, 3) -> the last pair's cached value is discarded."""
    D, H, nh, n = 6, 32, 2, B + 400
    rng = np.random.default_rng(5)
    h = make_vl(D, A, H, nh, B, n)
    insert_rows(h, *random_rows(rng, n, D, A))
    es = EpsStream(0, 1, philox=True)
    for _ in range(3):
        v_update(h)
        got = np.zeros(B * A, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 5, ptr(got))
        want = es.draw(B, A).ravel()
        np.testing.assert_array_equal(got.view(np.uint32), want.view(np.uint32))
    _lib.call("pqlg_vlearner_destroy", h)


def test_sac_vlearner_k_steps_vs_reference_golden():
    G = np.load(GOLDEN / "sac.npz")
    D, A, H, nh, B, cap = (int(v) for v in G["su_dims"])
    h = make_vl(D, A, H, nh, B, cap)
    set_params(h, 0, G["su_q1"]); set_params(h, 1, G["su_q2"])
    set_params(h, 2, G["su_q1"]); set_params(h, 3, G["su_q2"])
    v_adopt(h, G["su_pol"], G["su_log_alpha"][0])
    la = C.c_float()
    _lib.call("pqlg_vlearner_log_alpha", h, C.byref(la))
    assert la.value == np.float32(G["su_log_alpha"][0])
    insert_rows(h, G["su_obs"], G["su_act"], G["su_boot"], G["su_ret"], G["su_eff"])
    adopt_norm(h, int(G["su_norm"][0]), G["su_mean"], G["su_m2"])
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)  # + the reference's eps stream
    losses = [v_update(h) for _ in range(3)]
    print("losses gpu", losses, "ref", G["su_losses"])
    np.testing.assert_allclose(losses, G["su_losses"], rtol=2e-3)
    P = param_count([D + A] + [H] * nh + [1])
    for w in range(4):
        check_weights(params(h, w, P), G["su_params"][w], 5e-4, 3)
    _lib.call("pqlg_vlearner_destroy", h)


def test_sac_plearner_k_steps_vs_reference_golden():
    G = np.load(GOLDEN / "sac.npz")
    D, A, H, nh, B, cap = (int(v) for v in G["su_dims"])
    h = make_pl(D, A, H, nh, B, cap)
    pl_put(h, 0, G["su_pol"]); pl_put(h, 1, G["su_q1"]); pl_put(h, 2, G["su_q2"])
    pl_ingest(h, G["su_obs"])
    mean = np.ascontiguousarray(G["su_mean"], np.float64)
    m2 = np.ascontiguousarray(G["su_m2"], np.float64)
    ns = _lib.NormStats(int(G["su_norm"][0]), ptr(mean), ptr(m2))
    _lib.call("pqlg_plearner_adopt_norm", h, C.byref(ns))
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    losses, las = [], []
    for _ in range(3):
        losses.append(p_update(h))
        la = C.c_float()
        _lib.call("pqlg_plearner_log_alpha", h, C.byref(la))
        las.append(la.value)
    print("actor losses gpu", losses, "ref", G["sp_losses"], "log alpha", las, G["sp_log_alpha"])
    assert np.max(np.abs(np.array(losses) - G["sp_losses"])) <= 2e-3 * (
        1.0 + np.max(np.abs(G["sp_losses"])))
    # Adam moves log alpha by ~lr per step whatever the gradient's size
    assert np.max(np.abs(np.array(las) - G["sp_log_alpha"])) <= 2e-3 * 5e-4 * 3 + 1e-7
    check_weights(pl_get(h, 0, param_count([D] + [H] * nh + [2 * A])), G["sp_params"], 5e-4, 3)
    _lib.call("pqlg_plearner_destroy", h)


@pytest.mark.parametrize("cfg", ["small", "c3"])
def test_sac_vlearner_intermediates_vs_oracle(cfg):
    D, A, H, nh, B, n = {"small": (32, 8, 256, 2, 1024, 20000),
                         "c3": (211, 20, 512, 3, 8192, 30000)}[cfg]
    rng = np.random.default_rng(21)
    h = make_vl(D, A, H, nh, B, n + 10)
    P = param_count([D + A] + [H] * nh + [1])
    Pp = param_count([D] + [H] * nh + [2 * A])
    q1, q2 = params(h, 0, P), params(h, 1, P)
    pol = params(h, 4, Pp)
    log_alpha = -0.3
    v_adopt(h, pol, log_alpha)
    obs, act, boot, ret, eff = random_rows(rng, n, D, A)
    insert_rows(h, obs, act, boot, ret, eff)
    count = 10**6
    mean, m2 = adopt_norm(h, count, rng.standard_normal(D) * 0.1,
                          np.abs(rng.standard_normal(D)) * count + count * 0.5)
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)
    o = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, sac=True, log_alpha=log_alpha)
    o.set_rows(obs, act, boot, ret, eff)
    o.norm = (count, mean, m2)
    k = 2
    for step in range(k):
        loss_o, info = o.step()
        lg = v_update(h)
        y = np.zeros(B, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 0, ptr(y))
        g = np.zeros(2 * P, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 2, ptr(g))
        sc = np.zeros(2, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 3, ptr(sc))
        r = [rel(g[kk * P:(kk + 1) * P] * sc[kk], info["dq"][kk]) for kk in range(2)]
        ry = rel(y, info["y"])
        print(f"\n{cfg} step {step}: loss gpu={lg:.6f} oracle={loss_o:.6f} y_rel={ry:.2e} g_rel={r}")
        assert abs(lg - loss_o) <= 2e-3 * abs(loss_o)
        assert ry <= 2e-3
        for kk in range(2):
            assert r[kk] <= 1e-2, r
    for w, want in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        check_weights(params(h, w, P), want, 5e-4, k)
    _lib.call("pqlg_vlearner_destroy", h)


def test_sac_target_sample_vs_oracle():
    """debug_read 6/7: log pi(a'|s+) and a' of the target policy vs
    GaussianPolicy::sample on the same normalised boot rows and eps."""
    D, A, H, nh, B, n = 24, 6, 128, 2, 512, 3000
    rng = np.random.default_rng(22)
    h = make_vl(D, A, H, nh, B, n)
    Pp = param_count([D] + [H] * nh + [2 * A])
    pol = params(h, 4, Pp)  # orthogonal init; log_std biases spread over both clamps
    pol[Pp - A:] = np.linspace(-6.0, 3.0, A, dtype=np.float32)
    v_adopt(h, pol, 0.2)
    insert_rows(h, *random_rows(rng, n, D, A))
    v_update(h)
    X = np.zeros((B, D + A), np.float32)
    _lib.call("pqlg_vlearner_debug_read", h, 7, ptr(X))
    eps = np.zeros((B, A), np.float32)
    _lib.call("pqlg_vlearner_debug_read", h, 5, ptr(eps))
    logp = np.zeros(B, np.float32)
    _lib.call("pqlg_vlearner_debug_read", h, 6, ptr(logp))
    act = np.zeros((B, A), np.float32)
    lo = np.zeros(B, np.float32)
    ps = [D] + [H] * nh + [2 * A]
    boot = np.ascontiguousarray(X[:, :D])
    orc().orc_gauss_sample(ptr(pol), ptr(sizes_arr(ps)), nh + 1, ptr(boot), ptr(eps), B,
                           np.float32(-1), np.float32(1), ptr(act), ptr(lo))
    print("act max err", np.max(np.abs(X[:, D:] - act)), "logp rel", rel(logp, lo))
    assert np.max(np.abs(X[:, D:] - act)) <= 2e-3
    assert rel(logp, lo) <= 2e-3
    _lib.call("pqlg_vlearner_destroy", h)


@pytest.mark.parametrize("cfg", ["small", "c3"])
def test_sac_plearner_vs_oracle(cfg):
    D, A, H, nh, B, n = {"small": (31, 7, 256, 2, 1024, 5000),
                         "c3": (211, 20, 512, 3, 8192, 20000)}[cfg]
    rng = np.random.default_rng(23)
    h = make_pl(D, A, H, nh, B, n)
    Pp = param_count([D] + [H] * nh + [2 * A])
    Pq = param_count([D + A] + [H] * nh + [1])
    pol, q1, q2 = pl_get(h, 0, Pp), pl_get(h, 1, Pq), pl_get(h, 2, Pq)
    states = f32(rng.standard_normal((n, D)))
    pl_ingest(h, states)
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    o = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, sac=True)
    o.states = states
    k = 2
    for _ in range(k):
        lo, info = o.step()
        lg = p_update(h)
        print(f"\n{cfg}: actor loss gpu={lg:.6f} oracle={lo:.6f}")
        assert abs(lg - lo) <= 2e-3 * (1.0 + abs(lo))
    la = C.c_float()
    _lib.call("pqlg_plearner_log_alpha", h, C.byref(la))
    assert abs(la.value - o.alpha_p[0]) <= 2e-3 * 5e-4 * k + 1e-7
    check_weights(pl_get(h, 0, Pp), o.pol, 5e-4, k)
    _lib.call("pqlg_plearner_destroy", h)


def test_sac_graph_replay_philox_vs_oracle():
    """update_n (CUDA graph, device eps stream) for V and P vs the oracle on
    the Philox streams."""
    D, A, H, nh, B, n = 32, 8, 256, 2, 1024, 5000
    rng = np.random.default_rng(24)
    h = make_vl(D, A, H, nh, B, n)
    P = param_count([D + A] + [H] * nh + [1])
    Pp = param_count([D] + [H] * nh + [2 * A])
    q1, q2, pol = params(h, 0, P), params(h, 1, P), params(h, 4, Pp)
    v_adopt(h, pol, -0.5)
    rows = random_rows(rng, n, D, A)
    insert_rows(h, *rows)
    o = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, philox=True, sac=True, log_alpha=-0.5)
    o.set_rows(*rows)
    k = 4
    _lib.call("pqlg_vlearner_update_n", h, k)
    losses = [o.step()[0] for _ in range(k)]
    l = C.c_float()
    _lib.call("pqlg_vlearner_last_loss", h, C.byref(l))
    assert abs(l.value - losses[-1]) <= 2e-3 * abs(losses[-1])
    for w, want in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        check_weights(params(h, w, P), want, 5e-4, k)
    _lib.call("pqlg_vlearner_destroy", h)

    hp = make_pl(D, A, H, nh, B, n)
    pol, q1, q2 = pl_get(hp, 0, Pp), pl_get(hp, 1, P), pl_get(hp, 2, P)
    states = f32(rng.standard_normal((n, D)))
    pl_ingest(hp, states)
    op = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, philox=True, sac=True)
    op.states = states
    _lib.call("pqlg_plearner_update_n", hp, k)
    for _ in range(k):
        op.step()
    la = C.c_float()
    _lib.call("pqlg_plearner_log_alpha", hp, C.byref(la))
    assert abs(la.value - op.alpha_p[0]) <= 2e-3 * 5e-4 * k + 1e-7
    check_weights(pl_get(hp, 0, Pp), op.pol, 5e-4, k)
    _lib.call("pqlg_plearner_destroy", hp)


@pytest.mark.parametrize("N,D,A", [(40, 9, 4), (4096, 211, 20), (300, 17, 7), (64, 7, 1),
                                   (96, 40, 32)])
def test_sac_actor_step_vs_oracle(N, D, A):
    """ActorCore::rollout_step for pql_sac: the per-env eps draws (fresh
    normal_distribution over the noise streams) bit-exact -- checked through
    the stream states -- and the squashed sample within TF32 tolerance."""
    H, nh = 64, 2
    conf = cfg_sac(n_envs=N, hidden=H, hidden_layers=nh, seed=0)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(conf), C.byref(dims), None, C.byref(h))
    ps = [D] + [H] * nh + [2 * A]
    pol = np.zeros(param_count(ps), np.float32)
    _lib.call("pqlg_actor_read", h, 5, ptr(pol))
    obs0 = np.zeros((N, D), np.float32)
    _lib.call("pqlg_actor_read", h, 0, ptr(obs0))
    sl = _lib.StepSlice()
    _lib.call("pqlg_actor_rollout_step", h, C.byref(sl))
    act = np.zeros((N, A), np.float32)
    _lib.call("pqlg_actor_read", h, 1, ptr(act))
    ns = np.zeros(N, np.uint64)
    _lib.call("pqlg_actor_read", h, 2, ptr(ns))
    states = np.array([derive_seed(0, STREAM_NOISE, i) for i in range(N)], np.uint64)
    eps = np.zeros((N, A), np.float32)
    orc().orc_normals_rows(ptr(states), N, A, ptr(eps))
    np.testing.assert_array_equal(ns, states)
    want = np.zeros((N, A), np.float32)
    lp = np.zeros(N, np.float32)
    x = normalize(0, np.zeros(D), np.zeros(D), obs0)
    orc().orc_gauss_sample(ptr(pol), ptr(sizes_arr(ps)), nh + 1, ptr(x), ptr(eps), N,
                           np.float32(-1), np.float32(1), ptr(want), ptr(lp))
    print("max |da|", np.max(np.abs(act - want)))
    assert np.max(np.abs(act - want)) <= 2e-3
    _lib.call("pqlg_actor_destroy", h)


def test_sac_evaluate_uses_the_squashed_mean():
    """evaluate_policy with a stochastic snapshot acts with mean_act
    (policy.hpp:110-118): a SAC net whose mean half equals a DDPG net gives
    the DDPG evaluation exactly (the log_std half is ignored)."""
    D, A, H, nh, E = 12, 3, 64, 2, 16
    rng = np.random.default_rng(25)
    ps_d = [D] + [H] * nh + [A]
    det = f32(rng.standard_normal(param_count(ps_d)) * 0.2)
    # build the SAC net: hidden layers equal, head W [H x 2A] = [W_det | random]
    ps_s = [D] + [H] * nh + [2 * A]
    sac = np.zeros(param_count(ps_s), np.float32)
    off_d = off_s = 0
    for l in range(nh + 1):
        i, o_d, o_s = ps_d[l], ps_d[l + 1], ps_s[l + 1]
        Wd = det[off_d:off_d + i * o_d].reshape(i, o_d)
        bd = det[off_d + i * o_d:off_d + i * o_d + o_d]
        if o_s == o_d:
            Ws, bs = Wd, bd
        else:
            Ws = np.concatenate([Wd, f32(rng.standard_normal((i, A)))], axis=1)
            bs = np.concatenate([bd, f32(rng.standard_normal(A))])
        sac[off_s:off_s + i * o_s] = Ws.ravel()
        sac[off_s + i * o_s:off_s + i * o_s + o_s] = bs
        off_d += i * o_d + o_d
        off_s += i * o_s + o_s
    mean = np.zeros(D)
    m2 = np.zeros(D)
    res = {}
    for algo, flat in [(_lib.ALGO_DDPG, det), (_lib.ALGO_SAC, sac)]:
        conf = _lib.default_config(algo=algo, hidden=H, hidden_layers=nh, max_episode_len=50)
        dims = _lib.TaskDims(D, A, -1.0, 1.0)
        ret = np.zeros(E, np.float64)
        mu, se = C.c_double(), C.c_double()
        ns = _lib.NormStats(0, ptr(mean), ptr(m2))
        _lib.call("pqlg_evaluate", C.byref(conf), C.byref(dims), ptr(flat), C.byref(ns), E, 7,
                  ptr(ret), C.byref(mu), C.byref(se))
        res[algo] = ret
    np.testing.assert_array_equal(res[_lib.ALGO_DDPG], res[_lib.ALGO_SAC])
