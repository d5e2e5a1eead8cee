"""Actor path on the GPU: the synthetic EnvBatch bit-exact against the
reference's own EnvBatch::step on SyntheticEnv (tests/golden/env.npz) and
the oracle, the exploration noise bit-exact against the reference's noise
fixtures, the normalizer update to 1e-10, and rollout_step end to end
against the reference's own rt::ActorCore (tests/golden/actor_core.npz):
initial observations and policy, termination / truncation flags and episode
counters exact; actions, observations and rewards within the precision
mode's bar (TF32 2e-3, 3xTF32 2e-5 norm-wise)."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import STREAM_NOISE, derive_seed, orc, param_count, ptr
from oracle_model import OracleActor, OracleEnv, f32
from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def u32(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def d2h(ptr_dev, ld, rows, cols, dtype=np.float32):
    """Rows of a device view (a StepSlice field) to host."""
    from cuda.bindings import runtime as rt
    out = np.zeros((rows, cols), dtype)
    w = cols * out.itemsize
    err, = rt.cudaMemcpy2D(out.ctypes.data, w, ptr_dev, (ld or cols) * out.itemsize, w, rows,
                           rt.cudaMemcpyKind.cudaMemcpyDeviceToHost)
    assert err == rt.cudaError_t.cudaSuccess, err
    return out


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / (np.linalg.norm(b) + 1e-30))


@pytest.mark.parametrize("k", [0, 1, 2])
def test_env_bit_exact_vs_reference_golden(k):
    """The device env replays the actions of tests/golden/env.npz and matches
    the reference's EnvBatch::step on SyntheticEnv bit for bit: rewards,
    dones, truncations, next and terminal observations (full arrays or
    per-step digests), episode counters, and the non-finite-action error."""
    import torch
    from oracle_lib import traj_hash
    G = np.load(GOLDEN / "env.npz")
    N, D, A, max_len, T, seed = (int(x) for x in G[f"env{k}_args"])
    h = C.c_void_p()
    _lib.call("pqlg_env_create", N, D, A, seed, max_len, 0, np.float32(-1), np.float32(1), None,
              C.byref(h))
    obs = torch.zeros(N, D, device="cuda")
    _lib.call("pqlg_env_reset_all", h, obs.data_ptr(), 0)
    torch.cuda.synchronize()
    assert np.array_equal(u32(host(obs)), u32(G[f"env{k}_obs0"]))
    nxt = torch.zeros(N, D, device="cuda")
    term_obs = torch.zeros(N, D, device="cuda")
    rew = torch.zeros(N, device="cuda")
    done = torch.zeros(N, dtype=torch.uint8, device="cuda")
    trunc = torch.zeros(N, dtype=torch.uint8, device="cuda")
    for t in range(T):
        ad = dev(G[f"env{k}_act"][t])
        _lib.call("pqlg_env_step", h, ad.data_ptr(), 0, nxt.data_ptr(), term_obs.data_ptr(),
                  rew.data_ptr(), done.data_ptr(), trunc.data_ptr(), 0)
        torch.cuda.synchronize()
        dn = host(done)
        assert np.array_equal(dn, G[f"env{k}_done"][t]), t
        assert np.array_equal(host(trunc), G[f"env{k}_trunc"][t]), t
        assert np.array_equal(u32(host(rew)), u32(G[f"env{k}_rew"][t])), t
        to = host(term_obs).copy()
        to[dn == 0] = 0.0
        assert traj_hash(host(nxt)) == G[f"env{k}_hash"][t, 0], t
        assert traj_hash(to) == G[f"env{k}_hash"][t, 1], t
    assert np.array_equal(u32(host(nxt)), u32(G[f"env{k}_last"]))
    bad = dev(f32(np.full((N, A), np.nan)))
    with pytest.raises(_lib.NonFinite):
        _lib.call("pqlg_env_step", h, bad.data_ptr(), 0, nxt.data_ptr(), term_obs.data_ptr(),
                  rew.data_ptr(), done.data_ptr(), trunc.data_ptr(), 0)
    _lib.call("pqlg_env_destroy", h)


@pytest.mark.parametrize("k,prec", [(0, _lib.PREC_TF32), (0, _lib.PREC_3XTF32),
                                    (1, _lib.PREC_TF32), (1, _lib.PREC_3XTF32),
                                    (2, _lib.PREC_TF32), (2, _lib.PREC_3XTF32)])
def test_rollout_vs_reference_actor_core(k, prec):
    """pqlg_actor_rollout_step vs the reference's rt::ActorCore::rollout_step
    on the synthetic task (tests/golden/actor_core.npz; DDPG with mixed
    noise at c1 and c3-width dims, and pql_sac).  Both start from the same
    state by construction: the device's initial policy must equal
    PolicyHandle::create's bit for bit."""
    from oracle_lib import traj_hash
    G = np.load(GOLDEN / "actor_core.npz")
    N, D, A, H, seed, max_len, T, sac = (int(x) for x in G[f"ac{k}_args"])
    conf = _lib.default_config(n_envs=N, hidden=H, hidden_layers=2, seed=seed,
                               max_episode_len=max_len, precision=prec,
                               algo=_lib.ALGO_SAC if sac else _lib.ALGO_DDPG)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(conf), C.byref(dims), None, C.byref(h))
    pol = np.zeros(param_count([D, H, H, 2 * A if sac else A]), np.float32)
    _lib.call("pqlg_actor_read", h, 5, ptr(pol))
    if f"ac{k}_policy" in G:
        assert np.array_equal(u32(pol), u32(G[f"ac{k}_policy"]))
    else:
        assert traj_hash(pol) == G[f"ac{k}_policy_hash"][0]
    bar = 2e-3 if prec == _lib.PREC_TF32 else 2e-5
    worst = {}
    for t in range(T):
        sl = _lib.StepSlice()
        _lib.call("pqlg_actor_rollout_step", h, C.byref(sl))
        got = dict(obs=d2h(sl.obs, sl.ld_obs, N, D), act=d2h(sl.act, sl.ld_act, N, A),
                   boot=d2h(sl.boot_obs, sl.ld_obs, N, D), rew=d2h(sl.rew, 0, N, 1)[:, 0],
                   term=d2h(sl.term, 0, N, 1, np.uint8)[:, 0],
                   trunc=d2h(sl.trunc, 0, N, 1, np.uint8)[:, 0])
        if t == 0:  # reset_all observations: exact
            assert np.array_equal(u32(got["obs"]), u32(G[f"ac{k}_obs"][0]))
        for key in ("obs", "act", "boot", "rew"):
            r = rel(got[key], G[f"ac{k}_{key}"][t])
            worst[key] = max(worst.get(key, 0.0), r)
            assert r <= bar, (t, key, r)
        assert np.array_equal(got["term"], G[f"ac{k}_term"][t]), t
        assert np.array_equal(got["trunc"], G[f"ac{k}_trunc"][t]), t
    ep = np.zeros(N, np.int64)
    _lib.call("pqlg_actor_read", h, 3, ptr(ep))
    assert np.array_equal(ep, G[f"ac{k}_episode_step"])
    cnt = C.c_int64()
    mean, m2 = np.zeros(D), np.zeros(D)
    _lib.call("pqlg_actor_norm", h, C.byref(cnt), ptr(mean), ptr(m2))
    norm = G[f"ac{k}_norm"]
    assert cnt.value == int(norm[0]) == N * T
    std = np.sqrt(norm[1 + D:] / norm[0])
    assert np.all(np.abs(mean - norm[1:1 + D]) <= bar * std)
    np.testing.assert_allclose(m2, norm[1 + D:], rtol=bar)
    print(f"\nactor_core case {k} precision {prec}: worst rel {worst}")
    _lib.call("pqlg_actor_destroy", h)


@pytest.mark.parametrize("N,D,A,max_len", [(64, 5, 2, 7), (96, 211, 20, 1000), (40, 60, 8, 13)])
def test_env_bit_exact_vs_oracle(N, D, A, max_len):
    import torch
    seed = 3
    h = C.c_void_p()
    _lib.call("pqlg_env_create", N, D, A, seed, max_len, 0, np.float32(-1), np.float32(1), None,
              C.byref(h))
    o = OracleEnv(N, D, A, seed, max_len)
    obs = torch.zeros(N, D, device="cuda")
    _lib.call("pqlg_env_reset_all", h, obs.data_ptr(), 0)
    torch.cuda.synchronize()
    assert np.array_equal(u32(host(obs)), u32(o.observe()))
    rng = np.random.default_rng(N + D)
    # constant push on some envs so |s_0| crosses 9 (terminal) within the run
    M = None
    drive = np.sign(rng.standard_normal((N, A))).astype(np.float32)
    saw_term = saw_trunc = False
    for t in range(60):
        a = f32(np.where(rng.uniform(size=(N, 1)) < 0.5, drive,
                         rng.uniform(-1.5, 1.5, (N, A))))  # includes out-of-range actions
        ad = dev(a)
        nxt = torch.zeros(N, D, device="cuda"); term_obs = torch.zeros(N, D, device="cuda")
        rew = torch.zeros(N, device="cuda")
        done = torch.zeros(N, dtype=torch.uint8, device="cuda")
        trunc = torch.zeros(N, dtype=torch.uint8, device="cuda")
        _lib.call("pqlg_env_step", h, ad.data_ptr(), 0, nxt.data_ptr(), term_obs.data_ptr(),
                  rew.data_ptr(), done.data_ptr(), trunc.data_ptr(), 0)
        torch.cuda.synchronize()
        w_nxt, w_term, w_rew, w_done, w_trunc = o.step(a)
        assert np.array_equal(host(done), w_done) and np.array_equal(host(trunc), w_trunc)
        assert np.array_equal(u32(host(nxt)), u32(w_nxt)), t
        assert np.array_equal(u32(host(rew)), u32(w_rew)), t
        d = w_done.astype(bool)
        assert np.array_equal(u32(host(term_obs)[d]), u32(w_term[d]))
        saw_term |= bool(np.any(d & ~w_trunc.astype(bool)))
        saw_trunc |= bool(np.any(w_trunc))
    if max_len <= 60:
        assert saw_trunc
    # non-finite action -> runtime_error (vecenv.cpp:87-89)
    bad = dev(f32(np.full((N, A), np.nan)))
    with pytest.raises(_lib.NonFinite):
        _lib.call("pqlg_env_step", h, bad.data_ptr(), 0, nxt.data_ptr(), term_obs.data_ptr(),
                  rew.data_ptr(), done.data_ptr(), trunc.data_ptr(), 0)
    _lib.call("pqlg_env_destroy", h)


def test_noise_bit_exact_vs_reference_golden():
    G = np.load(GOLDEN / "noise.npz")
    for N, A, steps in ((64, 8, 3), (33, 20, 2), (5, 1, 4)):
        a = G[f"noise_{N}_{A}_in"].copy()
        sig = np.zeros(N, np.float32)
        orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), N, ptr(sig))
        st = dev(np.array([derive_seed(0, STREAM_NOISE, i) for i in range(N)], np.uint64))
        sd = dev(sig)
        out = []
        for s in range(steps):
            ad = dev(a[s])
            _lib.call("pqlg_k_apply_noise", ad.data_ptr(), 0, N, A, sd.data_ptr(),
                      np.float32(-1), np.float32(1), st.data_ptr(), None)
            out.append(host(ad))
        assert np.array_equal(u32(np.stack(out)), u32(G[f"noise_{N}_{A}_out"])), (N, A)


def test_noise_bit_exact_wide_random_vs_oracle():
    # many rows -> many glibc-logf evaluations, incl. 1-ulp-sensitive inputs
    N, A = 20000, 20
    rng = np.random.default_rng(1)
    a = f32(rng.uniform(-1, 1, (N, A)))
    sig = np.zeros(N, np.float32)
    orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), N, ptr(sig))
    states = np.array([derive_seed(9, STREAM_NOISE, i) for i in range(N)], np.uint64)
    ad, sd, st = dev(a), dev(sig), dev(states)
    _lib.call("pqlg_k_apply_noise", ad.data_ptr(), 0, N, A, sd.data_ptr(), np.float32(-1),
              np.float32(1), st.data_ptr(), None)
    want = a.copy()
    ws = states.copy()
    orc().orc_apply_noise(ptr(want), N, A, ptr(sig), np.float32(-1), np.float32(1), ptr(ws))
    assert np.array_equal(u32(host(ad)), u32(want))
    assert np.array_equal(host(st), ws)


def test_normalizer_update_vs_oracle():
    import torch
    rng = np.random.default_rng(2)
    D = 211
    cnt = torch.zeros(1, dtype=torch.int64, device="cuda")
    mean = torch.zeros(D, dtype=torch.float64, device="cuda")
    m2 = torch.zeros(D, dtype=torch.float64, device="cuda")
    mf = torch.zeros(D, device="cuda"); inv = torch.zeros(D, device="cuda")
    oc = np.zeros(1, np.int64); om = np.zeros(D); om2 = np.zeros(D)
    for rows in (1, 300, 16384, 5):
        x = f32(rng.standard_normal((rows, D)) * 3 + 2)
        xd = dev(x)
        _lib.call("pqlg_k_normalizer_update", cnt.data_ptr(), mean.data_ptr(), m2.data_ptr(),
                  xd.data_ptr(), 0, rows, D, mf.data_ptr(), inv.data_ptr(), None)
        orc().orc_norm_update(ptr(oc), ptr(om), ptr(om2), ptr(x), rows, D)
        assert int(host(cnt)[0]) == oc[0]
        np.testing.assert_allclose(host(mean), om, rtol=1e-10, atol=1e-12)
        np.testing.assert_allclose(host(m2), om2, rtol=1e-10)
    mf_o = np.zeros(D, np.float32); inv_o = np.zeros(D, np.float32)
    orc().orc_norm_stats_to_f32(int(oc[0]), ptr(om), ptr(om2), D, ptr(mf_o), ptr(inv_o))
    np.testing.assert_allclose(host(mf), mf_o, rtol=1e-6)
    np.testing.assert_allclose(host(inv), inv_o, rtol=1e-6)


@pytest.mark.parametrize("cfg", ["small", "c3"])
def test_rollout_steps_vs_oracle(cfg):
    N, D, A, H, nh, T = {"small": (300, 13, 3, 64, 2, 6), "c3": (2048, 211, 20, 512, 3, 4)}[cfg]
    conf = _lib.default_config(n_envs=N, hidden=H, hidden_layers=nh, seed=5, max_episode_len=50)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(conf), C.byref(dims), None, C.byref(h))
    P = param_count([D] + [H] * nh + [A])
    pol = np.zeros(P, np.float32)
    _lib.call("pqlg_actor_read", h, 5, ptr(pol))
    # a policy with visible actions (the orthogonal init's 1e-2 head is near zero)
    rng = np.random.default_rng(3)
    pol = f32(pol + rng.standard_normal(P).astype(np.float32) * 0.02)
    _lib.call("pqlg_actor_adopt_policy", h, ptr(pol), 1)
    o = OracleActor(N, D, A, H, nh, pol, seed=5, max_len=50)
    obs0 = np.zeros((N, D), np.float32)
    _lib.call("pqlg_actor_read", h, 0, ptr(obs0))
    assert np.array_equal(u32(obs0), u32(o.obs))
    for t in range(T):
        s = _lib.StepSlice()
        _lib.call("pqlg_actor_rollout_step", h, C.byref(s))
        w = o.step()
        act = np.zeros((N, A), np.float32)
        _lib.call("pqlg_actor_read", h, 1, ptr(act))
        ns = np.zeros(N, np.uint64)
        _lib.call("pqlg_actor_read", h, 2, ptr(ns))
        ep = np.zeros(N, np.int64)
        _lib.call("pqlg_actor_read", h, 3, ptr(ep))
        # noise streams advance identically (polar rejections depend only on the stream)
        assert np.array_equal(ns, o.noise), t
        rel = np.linalg.norm(act - w["act"]) / np.linalg.norm(w["act"])
        print(f"\n{cfg} t={t}: actions rel={rel:.2e} max={np.max(np.abs(act - w['act'])):.2e}")
        assert rel <= 2e-3
        obs = np.zeros((N, D), np.float32)
        _lib.call("pqlg_actor_read", h, 0, ptr(obs))  # next observation
        # next obs = 0.95 s + 0.05 M a: inherits the TF32 action error
        orel = np.linalg.norm(obs - o.obs) / np.linalg.norm(o.obs)
        assert orel <= 1e-3, orel
    cnt = C.c_int64()
    mean = np.zeros(D); m2 = np.zeros(D)
    _lib.call("pqlg_actor_norm", h, C.byref(cnt), ptr(mean), ptr(m2))
    assert cnt.value == o.count[0] == N * T
    # the observations themselves carry the TF32 action error (1e-4 rel), so
    # the stats are compared on the scale of the data: |dmean| <= 1e-3 std
    std = np.sqrt(o.m2 / o.count[0])
    assert np.all(np.abs(mean - o.mean) <= 1e-3 * std)
    np.testing.assert_allclose(m2, o.m2, rtol=2e-3)
    _lib.call("pqlg_actor_destroy", h)


def test_cross_stream_ingest_ordered_by_exported_events():
    """Actor and V-learner on different streams, ordered only by the ABI's
    events (pqlg_actor_step_event -> pqlg_vlearner_wait_event, and
    pqlg_vlearner_record_event -> pqlg_actor_wait_event): the replay ring
    equals the one built with everything on one stream."""
    import torch
    N, D, A, steps = 1024, 23, 6, 9
    cfg = _lib.default_config(n_envs=N, hidden=64, hidden_layers=2, batch_size=256,
                              buffer_capacity=20000, seed=2, max_episode_len=5)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)

    def run(shared):
        s0 = torch.cuda.Stream()
        s1 = s0 if shared else torch.cuda.Stream()
        act, vl = C.c_void_p(), C.c_void_p()
        _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), C.c_void_p(s0.cuda_stream),
                  C.byref(act))
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1,
                  C.c_void_p(s1.cuda_stream), C.byref(vl))
        sl = _lib.StepSlice()
        for _ in range(steps):
            _lib.call("pqlg_actor_rollout_step", act, C.byref(sl))
            if not shared:
                ev = C.c_void_p()
                _lib.call("pqlg_actor_step_event", act, C.byref(ev))
                _lib.call("pqlg_vlearner_wait_event", vl, ev)
            _lib.call("pqlg_vlearner_ingest", vl, C.byref(sl))
            if not shared:
                ev2 = C.c_void_p()
                _lib.call("pqlg_vlearner_record_event", vl, C.byref(ev2))
                _lib.call("pqlg_actor_wait_event", act, ev2)
        rp = C.c_void_p()
        _lib.call("pqlg_vlearner_replay", vl, C.byref(rp))
        n = C.c_uint64()
        _lib.call("pqlg_replay_size", rp, C.byref(n))
        out = [np.zeros((n.value, D), np.float32), np.zeros((n.value, A), np.float32),
               np.zeros((n.value, D), np.float32), np.zeros(n.value, np.float32),
               np.zeros(n.value, np.float32)]
        _lib.call("pqlg_replay_read_rows", rp, 0, n.value, *(ptr(x) for x in out))
        for h, fn in ((act, "pqlg_actor_destroy"), (vl, "pqlg_vlearner_destroy")):
            _lib.call(fn, h)
        return out

    a, b = run(True), run(False)
    assert a[3].size > 0
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def test_zero_sigma_rows_draw_no_noise():
    """build_fixed_schedule(0) (noise.hpp:44-50): sigma = 0 on every env, so
    apply_noise draws nothing -- the noise streams do not advance and the
    actions are the squashed policy output (clamped)."""
    N, D, A, H, nh = 256, 11, 4, 64, 2
    conf = _lib.default_config(n_envs=N, hidden=H, hidden_layers=nh, seed=6, sigma_fixed=0.0)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(conf), C.byref(dims), None, C.byref(h))
    ps = [D] + [H] * nh + [A]
    pol = np.zeros(param_count(ps), np.float32)
    _lib.call("pqlg_actor_read", h, 5, ptr(pol))
    obs0 = np.zeros((N, D), np.float32)
    _lib.call("pqlg_actor_read", h, 0, ptr(obs0))
    ns0 = np.zeros(N, np.uint64)
    _lib.call("pqlg_actor_read", h, 2, ptr(ns0))
    sl = _lib.StepSlice()
    _lib.call("pqlg_actor_rollout_step", h, C.byref(sl))
    act = np.zeros((N, A), np.float32)
    _lib.call("pqlg_actor_read", h, 1, ptr(act))
    ns1 = np.zeros(N, np.uint64)
    _lib.call("pqlg_actor_read", h, 2, ptr(ns1))
    np.testing.assert_array_equal(ns0, ns1)
    want = np.zeros((N, A), np.float32)
    orc().orc_policy_act(ptr(pol), ptr(np.asarray(ps, np.uintp)), nh + 1, ptr(obs0), N,
                         np.float32(-1), np.float32(1), ptr(want))
    assert np.max(np.abs(act - want)) <= 2e-3
    _lib.call("pqlg_actor_destroy", h)
