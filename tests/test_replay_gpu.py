"""Replay path on the GPU vs the oracle: bit-exact n-step records, ring
contents/cursor/count, state ring, and sampled + normalized minibatches in
both generator modes (reference mt19937_64 indices and Philox)."""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import MT64, STREAM_SAMPLE, derive_seed, orc, ptr
from oracle_model import f32, normalize
from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu
GOLDEN = __import__("pathlib").Path(__file__).resolve().parent / "golden"


def dev(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def host(t):
    return t.cpu().numpy()


def new_replay(cap, D, A):
    h = C.c_void_p()
    _lib.call("pqlg_replay_create", cap, D, A, None, C.byref(h))
    return h


def read_ring(h, cap, D, A, i0=0, n=None):
    n = cap - i0 if n is None else n
    obs = np.zeros((n, D), np.float32); act = np.zeros((n, A), np.float32)
    boot = np.zeros((n, D), np.float32); ret = np.zeros(n, np.float32)
    eff = np.zeros(n, np.float32)
    _lib.call("pqlg_replay_read_rows", h, i0, n, ptr(obs), ptr(act), ptr(boot), ptr(ret), ptr(eff))
    return obs, act, boot, ret, eff


def state_of(h):
    c = C.c_uint64(); s = C.c_uint64()
    _lib.call("pqlg_replay_cursor", h, C.byref(c))
    _lib.call("pqlg_replay_size", h, C.byref(s))
    return c.value, s.value


@pytest.mark.parametrize("case", [0, 1, 2])
def test_nstep_insert_bit_exact_vs_reference_golden(case):
    G = np.load(GOLDEN / "nstep.npz")
    T, N, D, A, n, cap = (int(v) for v in G[f"c{case}_args"])
    h = new_replay(cap, D, A)
    a = C.c_void_p()
    _lib.call("pqlg_nstep_create", N, D, A, np.float32(0.99), n, None, C.byref(a))
    e_off = 0
    for t in range(T):
        obs, act, boot = dev(G[f"c{case}_obs"][t]), dev(G[f"c{case}_act"][t]), dev(G[f"c{case}_boot"][t])
        rew, term, trunc = dev(G[f"c{case}_rew"][t]), dev(G[f"c{case}_term"][t]), dev(G[f"c{case}_trunc"][t])
        cur0, _ = state_of(h)
        s = _lib.StepSlice(obs.data_ptr(), act.data_ptr(), boot.data_ptr(), rew.data_ptr(),
                           term.data_ptr(), trunc.data_ptr(), 0, 0)
        _lib.call("pqlg_nstep_push_step", a, C.byref(s), np.float32(1.0), h)
        k = int(G[f"c{case}_counts"][t])
        if 0 < k <= cap:
            rows = [(cur0 + j) % cap for j in range(k)]
            got = [read_ring(h, cap, D, A, r, 1) for r in rows]
            for j, (o, ac, b, r, e) in enumerate(got):
                assert np.array_equal(o[0], G[f"c{case}_e_obs"][e_off + j])
                assert np.array_equal(ac[0], G[f"c{case}_e_act"][e_off + j])
                assert np.array_equal(b[0], G[f"c{case}_e_boot"][e_off + j])
                assert r[0].view(np.uint32) == G[f"c{case}_e_ret"][e_off + j].view(np.uint32)
                assert e[0].view(np.uint32) == G[f"c{case}_e_eff"][e_off + j].view(np.uint32)
        e_off += k
    obs, _, _, ret, _ = read_ring(h, cap, D, A)
    assert np.array_equal(obs, G[f"c{case}_ring_obs"])
    assert np.array_equal(ret.view(np.uint32), G[f"c{case}_ring_ret"].view(np.uint32))
    assert state_of(h) == tuple(int(v) for v in G[f"c{case}_cursor_count"])
    _lib.call("pqlg_nstep_destroy", a)
    _lib.call("pqlg_replay_destroy", h)


def test_nstep_large_batch_random_vs_oracle():
    # 16384 envs, config-3 dims, staggered dones, several steps incl. ring wrap
    rng = np.random.default_rng(11)
    N, D, A, n, cap, T = 4096, 211, 20, 3, 20000, 9
    h = new_replay(cap, D, A)
    a = C.c_void_p()
    _lib.call("pqlg_nstep_create", N, D, A, np.float32(0.99), n, None, C.byref(a))
    oa = orc().orc_nstep_create(N, D, A, np.float32(0.99), n)
    ob = orc().orc_batch_create(D, A)
    orr = orc().orc_replay_create(cap, D, A)
    scale = np.float32(0.1)
    for t in range(T):
        obs = f32(rng.standard_normal((N, D))); act = f32(rng.uniform(-1, 1, (N, A)))
        boot = f32(rng.standard_normal((N, D))); rew = f32(rng.standard_normal(N))
        u = rng.uniform(size=N)
        term = (u < 0.03).astype(np.uint8); trunc = ((u > 0.97)).astype(np.uint8)
        d = [dev(x) for x in (obs, act, boot, rew, term, trunc)]
        s = _lib.StepSlice(*(x.data_ptr() for x in d), 0, 0)
        _lib.call("pqlg_nstep_push_step", a, C.byref(s), scale, h)
        rs = f32(rew * scale)
        orc().orc_batch_clear(ob)
        orc().orc_nstep_push_step(oa, ptr(obs), ptr(act), ptr(rs), ptr(term), ptr(trunc), ptr(boot), ob)
        orc().orc_replay_insert(orr, ob)
    got = read_ring(h, cap, D, A)
    fr = C.cast(orr, C.POINTER(C.c_void_p))
    st = C.cast(orr, C.POINTER(C.c_size_t))
    want = []
    for j, w in enumerate([D, A, D, 1, 1]):
        arr = np.ctypeslib.as_array(C.cast(fr[5 + j], C.POINTER(C.c_float)), (cap * w,)).copy()
        want.append(arr.reshape(cap, w) if w > 1 else arr)
    for g, w in zip(got, want):
        assert np.array_equal(g.view(np.uint32), w.view(np.uint32))
    assert state_of(h) == (st[3], st[4])


def fill_random(h, rng, n, D, A):
    obs = f32(rng.standard_normal((n, D)) * 3); act = f32(rng.uniform(-1, 1, (n, A)))
    boot = f32(rng.standard_normal((n, D)) * 3); ret = f32(rng.standard_normal(n))
    eff = f32(rng.uniform(size=n))
    d = [dev(x) for x in (obs, act, boot, ret, eff)]
    b = _lib.NStepBatch(*(x.data_ptr() for x in d), 0, 0)
    _lib.call("pqlg_replay_insert", h, C.byref(b), n)
    return obs, act, boot, ret, eff


@pytest.mark.parametrize("mode", ["indices", "philox"])
def test_sample_gather_normalize_bit_exact(mode):
    import torch
    rng = np.random.default_rng(5)
    D, A, cap, n, B = 211, 20, 7000, 5000, 1024
    h = new_replay(cap, D, A)
    rows = fill_random(h, rng, n, D, A)
    count = 100_000
    mean = rng.standard_normal(D) * 0.5; m2 = np.abs(rng.standard_normal(D)) * count + 1.0
    ns = _lib.NormStats(count, ptr(mean), ptr(m2))
    key = derive_seed(3, STREAM_SAMPLE, 1)
    if mode == "indices":
        g = MT64(key)
        idx = np.zeros(B, np.uint64)
        orc().orc_sample_indices_mt(g.handle, n, B, ptr(idx))
        r = _lib.Rng(_lib.RNG_INDICES, 0, 0, ptr(idx))
    else:
        ctr = np.array([77], np.uint64)
        idx = np.zeros(B, np.uint64)
        orc().orc_sample_indices_philox(key, ptr(ctr), n, B, ptr(idx))
        r = _lib.Rng(_lib.RNG_PHILOX, key, 77, None)
    out = [torch.zeros(B, w, device="cuda") for w in (D, A, D)] + [torch.zeros(B, device="cuda")] * 0
    o_obs, o_act, o_boot = out
    o_ret = torch.zeros(B, device="cuda"); o_eff = torch.zeros(B, device="cuda")
    ob = _lib.NStepBatch(o_obs.data_ptr(), o_act.data_ptr(), o_boot.data_ptr(), o_ret.data_ptr(),
                         o_eff.data_ptr(), 0, 0)
    _lib.call("pqlg_replay_sample", h, B, C.byref(r), B, C.byref(ns), C.byref(ob))
    if mode == "philox":
        assert r.counter == int(ctr[0])
    ii = idx.astype(np.int64)
    assert np.array_equal(host(o_obs).view(np.uint32), normalize(count, mean, m2, rows[0][ii]).view(np.uint32))
    assert np.array_equal(host(o_boot).view(np.uint32), normalize(count, mean, m2, rows[2][ii]).view(np.uint32))
    assert np.array_equal(host(o_act), rows[1][ii])
    assert np.array_equal(host(o_ret), rows[3][ii]) and np.array_equal(host(o_eff), rows[4][ii])
    # not ready: min_live above the live count -> empty optional
    with pytest.raises(_lib.NotReady):
        _lib.call("pqlg_replay_sample", h, B, C.byref(r), n + 1, C.byref(ns), C.byref(ob))
    _lib.call("pqlg_replay_destroy", h)


def test_insert_larger_than_capacity_keeps_last_rows_in_order():
    rng = np.random.default_rng(6)
    D, A, cap = 5, 2, 7
    h = new_replay(cap, D, A)
    fill_random(h, rng, 3, D, A)
    rows = fill_random(h, rng, 17, D, A)  # 3 + 17 = 20 -> cursor 6, count 7
    assert state_of(h) == (20 % cap, cap)
    obs, act, boot, ret, eff = read_ring(h, cap, D, A)
    for k in range(17 - cap, 17):
        p = (3 + k) % cap
        assert np.array_equal(obs[p], rows[0][k]) and ret[p] == rows[3][k]
    _lib.call("pqlg_replay_destroy", h)


@pytest.mark.parametrize("mode", ["indices", "philox"])
def test_state_buffer_insert_sample(mode):
    import torch
    rng = np.random.default_rng(8)
    D, cap, B = 60, 1000, 512
    s = C.c_void_p()
    _lib.call("pqlg_states_create", cap, D, None, C.byref(s))
    ost = orc().orc_states_create(cap, D)
    for t in range(5):
        rows = f32(rng.standard_normal((300, D)))
        d = dev(rows)
        _lib.call("pqlg_states_insert", s, d.data_ptr(), 0, 300)
        orc().orc_states_insert(ost, ptr(rows), 300)
    size = C.c_uint64()
    _lib.call("pqlg_states_size", s, C.byref(size))
    assert size.value == cap
    ring = np.ctypeslib.as_array(C.cast(C.cast(ost, C.POINTER(C.c_void_p))[4],
                                        C.POINTER(C.c_float)), (cap * D,)).reshape(cap, D).copy()
    key = derive_seed(0, STREAM_SAMPLE, 2)
    idx = np.zeros(B, np.uint64)
    if mode == "indices":
        g = MT64(key)
        orc().orc_sample_indices_mt(g.handle, cap, B, ptr(idx))
        r = _lib.Rng(_lib.RNG_INDICES, 0, 0, ptr(idx))
    else:
        ctr = np.zeros(1, np.uint64)
        orc().orc_sample_indices_philox(key, ptr(ctr), cap, B, ptr(idx))
        r = _lib.Rng(_lib.RNG_PHILOX, key, 0, None)
    out = torch.zeros(B, D, device="cuda")
    _lib.call("pqlg_states_sample", s, B, C.byref(r), B, None, out.data_ptr(), 0)
    assert np.array_equal(host(out), ring[idx.astype(np.int64)])
    _lib.call("pqlg_states_destroy", s)


@pytest.mark.parametrize("count,B", [(1, 8), (100, 64), (5_000_000, 8192), (30_000, 300),
                                     ((1 << 63) + 1, 512), ((3 << 62) + 12345, 300),
                                     ((1 << 64) - 1, 256)])
def test_device_sampler_indices_match_libstdcxx_over_philox(count, B):
    """The device sampler's index draw (parallel Philox draws + Lemire, and
    the last block's sequential redo when any draw is rejected) equals
    libstdc++'s own uniform_int_distribution<size_t>(0, count-1) driven by
    the same Philox URBG (compiled into the reference harness), including
    counts above 2^63 where about half the draws are rejected, so the redo
    path runs."""
    from oracle_lib import orc, ref
    key = 0x0F1E_2D3C_4B5A_6978 ^ count
    for ctr0 in (0, 11, (1 << 41) + 5):
        got = np.zeros(B, np.uint64)
        ctr = C.c_uint64(ctr0)
        rej = C.c_uint32()
        _lib.call("pqlg_k_sample_indices", key, C.byref(ctr), count, B, got.ctypes.data,
                  C.byref(rej))
        want = np.zeros(B, np.uint64)
        R = ref()
        if R is not None:
            ctr_ref = R.ref_sample_indices_philox(key, ctr0, count, B, want.ctypes.data)
        else:  # the restatement, itself pinned to the reference (test_sampler_cpu.py)
            c = np.array([ctr0], np.uint64)
            orc().orc_sample_indices_philox(key, c.ctypes.data, count, B, want.ctypes.data)
            ctr_ref = int(c[0])
        assert np.array_equal(got, want)
        assert ctr.value == ctr_ref
        if count == (1 << 63) + 1:
            assert rej.value == 1 and ctr.value - ctr0 > B
        if count <= 5_000_000:
            assert rej.value == 0 and ctr.value - ctr0 == B
