"""Pins the CPU restatement (oracle/pql_oracle.c) before it is trusted as the
checker: spec known-answer tests, the survey's golden vectors, and the
fixtures generated from the compiled reference (tests/golden, made by
oracle/make_golden.py).  When oracle/_ref is present the restatement is also
checked against the live reference on fresh random inputs."""
import ctypes as C
import math
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import (MT64, STREAM_NOISE, STREAM_SAMPLE, acts_arr, derive_seed, orc,
                        param_count, ptr, ref, sizes_arr)
from oracle_model import OraclePUpdate, OracleVUpdate, f32

GOLDEN = Path(__file__).resolve().parent / "golden"


def golden(name):
    return np.load(GOLDEN / f"{name}.npz")


# ------------------------------------------------------------------ KATs
def test_kat_sample_indices_survey_golden_vector():
    # make_rng(0, sample, 1), 100 live rows -> 88 69 52 49 34 3 88 15
    g = MT64(derive_seed(0, STREAM_SAMPLE, 1))
    idx = np.zeros(8, np.uint64)
    orc().orc_sample_indices_mt(g.handle, 100, 8, ptr(idx))
    assert idx.tolist() == [88, 69, 52, 49, 34, 3, 88, 15]


def run_nstep(rews, terms, truncs, n=3, gamma=0.99):
    a = orc().orc_nstep_create(1, 1, 1, np.float32(gamma), n)
    b = orc().orc_batch_create(1, 1)
    out = []
    for r, te, tr in zip(rews, terms, truncs):
        orc().orc_batch_clear(b)
        o = np.zeros(1, np.float32)
        rr = np.array([r], np.float32)
        t1 = np.array([te], np.uint8)
        t2 = np.array([tr], np.uint8)
        orc().orc_nstep_push_step(a, ptr(o), ptr(o), ptr(rr), ptr(t1), ptr(t2), ptr(o), b)
        rows = C.cast(b, C.POINTER(C.c_size_t))[0]
        if rows:
            # struct orc_batch {rows, cap, obs_dim, act_dim, obs*, act*, boot*, ret*, eff*}
            fp = C.cast(b, C.POINTER(C.c_void_p))
            ret = np.ctypeslib.as_array(C.cast(fp[7], C.POINTER(C.c_float)), (rows,)).copy()
            eff = np.ctypeslib.as_array(C.cast(fp[8], C.POINTER(C.c_float)), (rows,)).copy()
            out += list(zip(ret.tolist(), eff.tolist()))
    orc().orc_batch_destroy(b)
    orc().orc_nstep_destroy(a)
    return out


def test_kat_nstep_spec():
    # SPEC.md:193 n=3, r=(1,1,1) -> G=2.9701, disc 0.970299 (f32: 2.97009993, 0.970299065)
    recs = run_nstep([1, 1, 1], [0, 0, 0], [0, 0, 0])
    assert len(recs) == 1
    assert np.float32(recs[0][0]) == np.float32(2.97009993)
    assert np.float32(recs[0][1]) == np.float32(0.970299065)
    # SPEC.md:194 termination after rewards (1, 1) -> (1.99, 0) and (1.0, 0)
    recs = run_nstep([1, 1], [0, 1], [0, 0])
    assert [(np.float32(g), e) for g, e in recs] == [(np.float32(1.99), 0.0), (np.float32(1.0), 0.0)]
    # n=1 degenerate horizon: (r, gamma) per step
    recs = run_nstep([2.0], [0], [0], n=1)
    assert recs == [(2.0, np.float32(0.99))]


def test_kat_schedule_clip_adam():
    s = np.zeros(4, np.float32)
    orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), 4, ptr(s))
    assert s.tolist() == [np.float32(0.0500000007), np.float32(0.300000012),
                          np.float32(0.550000012), np.float32(0.800000012)]
    s1 = np.zeros(1, np.float32)
    orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), 1, ptr(s1))
    assert s1[0] == np.float32(0.05)
    g = np.array([3, 4], np.float32)
    orc().orc_clip_global_norm(ptr(g), 2, np.float32(0.5))
    assert g.tolist() == [np.float32(0.299999684), np.float32(0.399999589)]
    p = np.zeros(1, np.float32); gg = np.ones(1, np.float32)
    m = np.zeros(1, np.float32); v = np.zeros(1, np.float32)
    bc1 = np.zeros(1, np.float32); bc2 = np.zeros(1, np.float32)
    orc().orc_adam_bias_corrections(1, ptr(bc1), ptr(bc2))
    orc().orc_adam_update(ptr(p), ptr(gg), ptr(m), ptr(v), 1, np.float32(1e-3), np.float32(0.9),
                          np.float32(0.999), np.float32(1e-8), bc1[0], bc2[0])
    assert p[0] == np.float32(-0.00100000668)


def test_kat_ddpg_zero_critics_and_c51_projection():
    # zero critics, y = 1 -> loss 2 (Q=0, G=1, eff=0)
    D, A, H, L, B = 2, 1, 4, 3, 1
    ps, qs = [D, H, H, A], [D + A, H, H, 1]
    pol = np.zeros(param_count(ps), np.float32)
    q = np.zeros(param_count(qs), np.float32)
    obs = np.zeros((B, D), np.float32); act = np.zeros((B, A), np.float32)
    ret = np.ones(B, np.float32); eff = np.zeros(B, np.float32)
    loss = np.zeros(1, np.float32); y = np.zeros(B, np.float32)
    dq1 = np.zeros_like(q); dq2 = np.zeros_like(q)
    rc = orc().orc_ddpg_critic_loss(ptr(pol), ptr(sizes_arr(ps)), ptr(q), ptr(q), ptr(q), ptr(q),
                                    ptr(sizes_arr(qs)), L, ptr(obs), ptr(act), ptr(obs), ptr(ret),
                                    ptr(eff), B, D, A, np.float32(-1), np.float32(1), ptr(loss),
                                    ptr(y), ptr(dq1), ptr(dq2))
    assert rc == 0 and loss[0] == 2.0 and y[0] == 1.0
    # l=3 on [-1,1], mass at 0, G=0.5 -> (0, 0.5, 0.5)
    atoms = np.zeros(3, np.float32)
    orc().orc_c51_atoms(3, np.float32(-1), np.float32(1), ptr(atoms))
    p = np.array([[0, 1, 0]], np.float32)
    out = np.zeros_like(p)
    assert orc().orc_c51_project(ptr(p), ptr(np.array([0.5], np.float32)),
                                 ptr(np.array([1.0], np.float32)), 1, 3, np.float32(-1),
                                 np.float32(1), ptr(atoms), ptr(out)) == 0
    assert out.tolist() == [[0.0, 0.5, 0.5]]


def test_philox_known_answer_vectors():
    # Random123 kat_vectors, philox4x32_10
    cases = [
        ([0, 0, 0, 0], [0, 0], [0x6627e8d5, 0xe169c58d, 0xbc57ac4c, 0x9b00dbd8]),
        ([0xffffffff] * 4, [0xffffffff] * 2, [0x408f276d, 0x41c83b0e, 0xa20bc7c6, 0x6d5451fd]),
        ([0x243f6a88, 0x85a308d3, 0x13198a2e, 0x03707344], [0xa4093822, 0x299f31d0],
         [0xd16cfe09, 0x94fdcceb, 0x5001e420, 0x24126ea1]),
    ]
    for ctr, key, want in cases:
        c = np.array(ctr, np.uint32); k = np.array(key, np.uint32); o = np.zeros(4, np.uint32)
        orc().orc_philox4x32_10(ptr(c), ptr(k), ptr(o))
        assert o.tolist() == want


def test_glibc_logf_restatement_sampled():
    # Exhaustively verified over all 2^31 positive floats during development
    # (80 s); here a strided sample over (0, 1] -- the polar method's range --
    # plus edge cases.
    bits = np.arange(1, 0x3F800001, 9973, dtype=np.uint32)
    xs = bits.view(np.float32)
    lib = orc()
    got = np.array([lib.orc_glibc_logf(float(x)) for x in xs[::7]], np.float32)
    want = np.array([math.log(float(x)) for x in xs[::7]], np.float64).astype(np.float32)
    # glibc logf is not correctly rounded everywhere; compare against libm logf via ctypes
    libm = C.CDLL("libm.so.6")
    libm.logf.restype = C.c_float
    libm.logf.argtypes = [C.c_float]
    ref_vals = np.array([libm.logf(float(x)) for x in xs[::7]], np.float32)
    assert np.array_equal(got.view(np.uint32), ref_vals.view(np.uint32))
    nz = want != 0
    assert np.max(np.abs(got[nz] - want[nz]) / np.abs(want[nz])) < 2.5e-7  # <= 1 ulp


# -------------------------------------------- restatement vs golden (ref)
def test_indices_and_mt64_match_reference_golden():
    G = golden("indices")
    g = MT64(derive_seed(0, STREAM_SAMPLE, 1))
    d = np.array([g() for _ in range(1000)], np.uint64)
    assert np.array_equal(d, G["mt64_draws"])
    for k in range(10):
        if f"idx{k}" not in G:
            continue
        seed, learner, count, B, n = (int(v) for v in G[f"idx{k}_args"])
        gg = MT64(derive_seed(seed, STREAM_SAMPLE, learner))
        idx = np.zeros(B * n, np.uint64)
        orc().orc_sample_indices_mt(gg.handle, count, B * n, ptr(idx))
        assert np.array_equal(idx, G[f"idx{k}"]), k


def oracle_nstep_replay(obs, act, boot, rew, term, trunc, n, cap, gamma=0.99):
    T, N, D = obs.shape
    A = act.shape[2]
    a = orc().orc_nstep_create(N, D, A, np.float32(gamma), n)
    b = orc().orc_batch_create(D, A)
    r = orc().orc_replay_create(cap, D, A)
    counts = []
    rows = {k: [] for k in ("obs", "act", "boot", "ret", "eff")}
    for t in range(T):
        orc().orc_batch_clear(b)
        orc().orc_nstep_push_step(a, ptr(obs[t]), ptr(act[t]), ptr(rew[t]), ptr(term[t]),
                                  ptr(trunc[t]), ptr(boot[t]), b)
        nr = C.cast(b, C.POINTER(C.c_size_t))[0]
        counts.append(nr)
        fp = C.cast(b, C.POINTER(C.c_void_p))
        if nr:
            for j, (k, w) in enumerate([("obs", D), ("act", A), ("boot", D), ("ret", 1),
                                        ("eff", 1)]):
                arr = np.ctypeslib.as_array(C.cast(fp[4 + j], C.POINTER(C.c_float)), (nr * w,))
                rows[k].append(arr.reshape(nr, w).copy() if w > 1 else arr.copy())
        orc().orc_replay_insert(r, b)
    fr = C.cast(r, C.POINTER(C.c_void_p))
    st = C.cast(r, C.POINTER(C.c_size_t))
    ring_obs = np.ctypeslib.as_array(C.cast(fr[5], C.POINTER(C.c_float)), (cap * D,)).copy()
    ring_ret = np.ctypeslib.as_array(C.cast(fr[8], C.POINTER(C.c_float)), (cap,)).copy()
    cursor, count = st[3], st[4]
    orc().orc_replay_destroy(r)
    orc().orc_batch_destroy(b)
    orc().orc_nstep_destroy(a)
    cat = {k: (np.concatenate(v) if v else np.zeros(0, np.float32)) for k, v in rows.items()}
    return counts, cat, ring_obs.reshape(cap, D), ring_ret, (cursor, count)


def test_nstep_ring_match_reference_golden():
    G = golden("nstep")
    for k in range(3):
        T, N, D, A, n, cap = (int(v) for v in G[f"c{k}_args"])
        counts, cat, ring_obs, ring_ret, cc = oracle_nstep_replay(
            G[f"c{k}_obs"], G[f"c{k}_act"], G[f"c{k}_boot"], G[f"c{k}_rew"], G[f"c{k}_term"],
            G[f"c{k}_trunc"], n, cap)
        assert counts == G[f"c{k}_counts"].tolist()
        for name in ("obs", "act", "boot", "ret", "eff"):
            want = G[f"c{k}_e_{name}"]
            assert np.array_equal(cat[name].reshape(want.shape).view(np.uint32),
                                  want.view(np.uint32)), (k, name)
        assert np.array_equal(ring_obs, G[f"c{k}_ring_obs"])
        assert np.array_equal(ring_ret, G[f"c{k}_ring_ret"])
        assert tuple(G[f"c{k}_cursor_count"].tolist()) == cc


def test_elementwise_match_reference_golden():
    G = golden("elementwise")
    n = G["adam_p"].size
    for t in (0, 1, 9, 99):
        p, m, v = G["adam_p"].copy(), G["adam_m"].copy(), G["adam_v"].copy()
        bc1 = np.zeros(1, np.float32); bc2 = np.zeros(1, np.float32)
        orc().orc_adam_bias_corrections(t + 1, ptr(bc1), ptr(bc2))
        orc().orc_adam_update(ptr(p), ptr(G["adam_g"]), ptr(m), ptr(v), n, np.float32(5e-4),
                              np.float32(0.9), np.float32(0.999), np.float32(1e-8), bc1[0], bc2[0])
        assert np.array_equal(np.stack([p, m, v]), G[f"adam_t{t}"]), t
    for scale in (0.01, 1.0, 30.0):
        g = f32(G["adam_g"] * scale)
        orc().orc_clip_global_norm(ptr(g), n, np.float32(0.5))
        assert np.array_equal(g, G[f"clip_{scale}"]), scale
    t = G["lerp_t"].copy()
    orc().orc_lerp_towards(ptr(t), ptr(G["adam_p"]), n, np.float32(0.05))
    assert np.array_equal(t, G["lerp_out"])
    for N in (1, 2, 4, 7, 4096):
        s = np.zeros(N, np.float32)
        orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), N, ptr(s))
        assert np.array_equal(s, G[f"sched_{N}"])
    # fp64 sum of squares: order may differ from the AVX2 backend by ulps
    assert orc().orc_sum_squares(ptr(G["adam_g"]), n) == pytest.approx(float(G["sumsq"][0]),
                                                                       rel=1e-14)


def test_normalizer_match_reference_golden():
    G = golden("norm")
    D = G["norm_mean"].size
    cnt = np.zeros(1, np.int64); mean = np.zeros(D); m2 = np.zeros(D)
    off = 0
    for r in G["norm_rows"]:
        r = int(r)
        orc().orc_norm_update(ptr(cnt), ptr(mean), ptr(m2), ptr(G["norm_data"][off:off + r].copy()),
                              r, D)
        off += r
    assert cnt[0] == G["norm_count"][0]
    assert np.array_equal(mean, G["norm_mean"]) and np.array_equal(m2, G["norm_m2"])
    x = G["norm_x"]
    out = np.zeros_like(x)
    orc().orc_normalize_apply(int(cnt[0]), ptr(mean), ptr(m2), ptr(x), ptr(out), x.shape[0], D)
    want = G["norm_xn"]
    # scalar.hpp keeps NaN; the AVX2 backend the reference runs maps NaN to a
    # clip bound.  Compare bit-exactly everywhere else.
    finite = np.isfinite(x)
    assert np.array_equal(out[finite], want[finite])


def test_noise_match_reference_golden_bit_exact():
    G = golden("noise")
    for N, A, steps in ((64, 8, 3), (33, 20, 2), (5, 1, 4)):
        a = G[f"noise_{N}_{A}_in"].copy()
        sig = np.zeros(N, np.float32)
        orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), N, ptr(sig))
        st = np.array([derive_seed(0, STREAM_NOISE, i) for i in range(N)], np.uint64)
        for s in range(steps):
            orc().orc_apply_noise(ptr(a[s]), N, A, ptr(sig), np.float32(-1), np.float32(1),
                                  ptr(st))
        assert np.array_equal(a.view(np.uint32), G[f"noise_{N}_{A}_out"].view(np.uint32))


def test_mlp_match_reference_golden():
    G = golden("mlp")
    sizes = G["mlp_sizes"].tolist()
    L = len(sizes) - 1
    x = G["mlp_x"]
    B = x.shape[0]
    y = np.zeros_like(G["mlp_y"])
    cache = np.zeros(sum(B * s for s in sizes[1:]), np.float32)
    orc().orc_mlp_forward(ptr(G["mlp_flat"]), ptr(sizes_arr(sizes)), ptr(acts_arr(L)), L, ptr(x),
                          B, ptr(y), ptr(cache))
    np.testing.assert_allclose(y, G["mlp_y"], rtol=1e-5, atol=1e-5)
    gr = np.zeros_like(G["mlp_grads"]); din = np.zeros_like(G["mlp_din"])
    orc().orc_mlp_backward(ptr(G["mlp_flat"]), ptr(sizes_arr(sizes)), ptr(acts_arr(L)), L,
                           ptr(x), ptr(cache), ptr(G["mlp_up"]), B, ptr(gr), ptr(din))
    np.testing.assert_allclose(gr, G["mlp_grads"], rtol=1e-4, atol=1e-5)
    np.testing.assert_allclose(din, G["mlp_din"], rtol=1e-4, atol=1e-5)


def test_agents_match_reference_golden():
    G = golden("agents")
    D, A, H, L, B = (int(v) for v in G["ag_dims"])
    ps, qs = [D] + [H] * (L - 1) + [A], [D + A] + [H] * (L - 1) + [1]
    P = param_count(qs)
    loss = np.zeros(1, np.float32); y = np.zeros(B, np.float32)
    dq1 = np.zeros(P, np.float32); dq2 = np.zeros(P, np.float32)
    rc = orc().orc_ddpg_critic_loss(
        ptr(G["ag_pol"]), ptr(sizes_arr(ps)), ptr(G["ag_q1"]), ptr(G["ag_q2"]), ptr(G["ag_q1t"]),
        ptr(G["ag_q2t"]), ptr(sizes_arr(qs)), L, ptr(G["ag_obs"]), ptr(G["ag_act"]),
        ptr(G["ag_boot"]), ptr(G["ag_ret"]), ptr(G["ag_eff"]), B, D, A, np.float32(-1),
        np.float32(1), ptr(loss), ptr(y), ptr(dq1), ptr(dq2))
    assert rc == 0
    np.testing.assert_allclose(y, G["ag_y"], rtol=1e-5, atol=1e-5)
    np.testing.assert_allclose(loss, G["ag_loss"], rtol=1e-5)
    np.testing.assert_allclose(dq1, G["ag_dq1"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(dq2, G["ag_dq2"], rtol=1e-4, atol=1e-6)
    dp = np.zeros(param_count(ps), np.float32)
    rc = orc().orc_ddpg_actor_loss(ptr(G["ag_pol"]), ptr(sizes_arr(ps)), ptr(G["ag_q1"]),
                                   ptr(G["ag_q2"]), ptr(sizes_arr(qs)), L, ptr(G["ag_obs"]), B, D,
                                   A, np.float32(-1), np.float32(1), ptr(loss), ptr(dp))
    assert rc == 0
    np.testing.assert_allclose(loss, G["ag_aloss"], rtol=1e-5)
    np.testing.assert_allclose(dp, G["ag_dpol"], rtol=1e-4, atol=1e-6)
    # C51
    La = int(G["c51_L"][0])
    qs = [D + A] + [H] * (L - 1) + [La]
    P = param_count(qs)
    dq1 = np.zeros(P, np.float32); dq2 = np.zeros(P, np.float32)
    rc = orc().orc_c51_critic_loss(
        ptr(G["c51_pol"]), ptr(sizes_arr(ps)), ptr(G["c51_q1"]), ptr(G["c51_q2"]),
        ptr(G["c51_q1t"]), ptr(G["c51_q2t"]), ptr(sizes_arr(qs)), L, ptr(G["ag_obs"]),
        ptr(G["ag_act"]), ptr(G["ag_boot"]), ptr(G["c51_ret"]), ptr(G["ag_eff"]), B, D, A,
        np.float32(-1), np.float32(1), La, np.float32(-10), np.float32(10), ptr(loss), ptr(dq1),
        ptr(dq2))
    assert rc == 0
    np.testing.assert_allclose(loss, G["c51_loss"], rtol=1e-5)
    np.testing.assert_allclose(dq1, G["c51_dq1"], rtol=1e-4, atol=1e-6)
    np.testing.assert_allclose(dq2, G["c51_dq2"], rtol=1e-4, atol=1e-6)
    rc = orc().orc_c51_actor_loss(ptr(G["c51_pol"]), ptr(sizes_arr(ps)), ptr(G["c51_q1"]),
                                  ptr(G["c51_q2"]), ptr(sizes_arr(qs)), L, ptr(G["ag_obs"]), B, D,
                                  A, np.float32(-1), np.float32(1), La, np.float32(-10),
                                  np.float32(10), ptr(loss), ptr(dp))
    assert rc == 0
    np.testing.assert_allclose(loss, G["c51_aloss"], rtol=1e-5)
    np.testing.assert_allclose(dp, G["c51_dpol"], rtol=1e-4, atol=1e-6)
    # projection: same double-precision arithmetic -> bit exact
    probs = G["proj_probs"]
    out = np.zeros_like(probs)
    atoms = np.zeros(La, np.float32)
    orc().orc_c51_atoms(La, np.float32(-10), np.float32(10), ptr(atoms))
    assert orc().orc_c51_project(ptr(probs), ptr(G["proj_ret"]), ptr(G["proj_eff"]),
                                 probs.shape[0], La, np.float32(-10), np.float32(10), ptr(atoms),
                                 ptr(out)) == 0
    assert np.array_equal(out, G["proj_out"])
    assert np.array_equal(out[0], probs[0])  # G=0, eff=1 is an exact identity


def test_vupdate_k_steps_match_reference_golden():
    G = golden("vupdate")
    D, A, H, nh, B, cap = (int(v) for v in G["vu_dims"])
    o = OracleVUpdate(D, A, H, nh, B, G["vu_q1"], G["vu_q2"], G["vu_pol"])
    o.set_rows(G["vu_obs"], G["vu_act"], G["vu_boot"], G["vu_ret"], G["vu_eff"])
    o.norm = (int(G["vu_norm"][0]), G["vu_mean"], G["vu_m2"])
    losses = [o.step()[0] for _ in range(3)]
    np.testing.assert_allclose(losses, G["vu_losses"], rtol=1e-5)
    for w, arr in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        want = G["vu_params"][w]
        # Adam sign amplification: norm-wise + per-element bound
        assert np.linalg.norm(arr - want) / np.linalg.norm(want) < 1e-4
        assert np.max(np.abs(arr - want)) <= 2 * 5e-4 * 3 * 0.01 + 1e-4
    p = OraclePUpdate(D, A, H, nh, B, G["vu_pol"], G["vu_q1"], G["vu_q2"])
    p.states = G["vu_obs"]
    p.norm = o.norm
    pl = [p.step()[0] for _ in range(3)]
    np.testing.assert_allclose(pl, G["pu_losses"], rtol=1e-5)
    assert np.linalg.norm(p.pol - G["pu_params"]) / np.linalg.norm(G["pu_params"]) < 1e-4


def test_c51_update_k_steps_match_reference_golden():
    """PQL-D: 3 c51 critic updates + 3 c51 policy updates (51 atoms) of the
    restatement vs the compiled reference (tests/golden/c51update.npz)."""
    G = golden("c51update")
    D, A, H, nh, B, cap, L = (int(v) for v in G["cu_dims"])
    o = OracleVUpdate(D, A, H, nh, B, G["cu_q1"], G["cu_q2"], G["cu_pol"], distributional=True,
                      n_atoms=L)
    o.set_rows(G["cu_obs"], G["cu_act"], G["cu_boot"], G["cu_ret"], G["cu_eff"])
    o.norm = (int(G["cu_norm"][0]), G["cu_mean"], G["cu_m2"])
    losses = [o.step()[0] for _ in range(3)]
    np.testing.assert_allclose(losses, G["cu_losses"], rtol=1e-5)
    for w, arr in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        want = G["cu_params"][w]
        assert np.linalg.norm(arr - want) / np.linalg.norm(want) < 1e-4
    p = OraclePUpdate(D, A, H, nh, B, G["cu_pol"], G["cu_q1"], G["cu_q2"], distributional=True,
                      n_atoms=L)
    p.states = G["cu_obs"]
    p.norm = o.norm
    pl = [p.step()[0] for _ in range(3)]
    np.testing.assert_allclose(pl, G["cpu_losses"], rtol=1e-5)
    assert np.linalg.norm(p.pol - G["cpu_params"]) / np.linalg.norm(G["cpu_params"]) < 1e-4


def test_init_orthogonal_golden_present():
    G = golden("mlp")
    assert G["init_policy"].size == param_count([6, 16, 16, 3])
    assert np.isfinite(G["init_critics"]).all()


# ---------------------------------------- live reference on fresh inputs
needs_ref = pytest.mark.skipif(ref() is None, reason="oracle/_ref not built here")


@needs_ref
def test_live_reference_sampling_many_counts():
    rng = np.random.default_rng(123)
    for _ in range(6):
        count = int(rng.integers(1, 300_000))
        seed = int(rng.integers(0, 2**63))
        B = 257
        want = np.zeros(2 * B, np.uint64)
        ref().ref_sample_indices(seed, 1, count, B, 2, ptr(want))
        g = MT64(derive_seed(seed, STREAM_SAMPLE, 1))
        got = np.zeros(2 * B, np.uint64)
        orc().orc_sample_indices_mt(g.handle, count, 2 * B, ptr(got))
        assert np.array_equal(got, want)


@needs_ref
def test_live_reference_noise_wide_rows():
    rng = np.random.default_rng(9)
    N, A, steps = 300, 20, 3
    a = f32(rng.uniform(-1, 1, (steps, N, A)))
    want = a.copy()
    ref().ref_apply_noise(np.float32(0.05), np.float32(0.8), N, A, 42, steps, np.float32(-1),
                          np.float32(1), ptr(want))
    sig = np.zeros(N, np.float32)
    orc().orc_build_schedule(np.float32(0.05), np.float32(0.8), N, ptr(sig))
    st = np.array([derive_seed(42, STREAM_NOISE, i) for i in range(N)], np.uint64)
    for s in range(steps):
        orc().orc_apply_noise(ptr(a[s]), N, A, ptr(sig), np.float32(-1), np.float32(1), ptr(st))
    assert np.array_equal(a.view(np.uint32), want.view(np.uint32))
