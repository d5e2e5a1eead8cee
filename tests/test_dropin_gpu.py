"""The drop-in, proven: the reference's own runtime cores bound to libpqlg.so.

oracle/Makefile `b200` patches the reference's learners.hpp / learners.cpp
at build time (oracle/b200_binding/make_binding.py: PQL_B200 #ifdefs, the
cores' definitions replaced by oracle/b200_binding/b200_cores.inc, which
drives the include/pqlg.hpp shims) and links the result against
libpqlg.so.  The same ref_harness.cpp entry points drive
pql::rt::CriticLearnerCore / PolicyLearnerCore / ActorCore in both builds,
so each test runs the unpatched reference (CPU) and the bound one (B200)
side by side on identical inputs, through the reference's public class
interfaces (learners.hpp:52-139):
  - construction from the reference's RunConfig / TaskDims / init engine
    (the bound cores upload the reference's own initial parameters)
  - ingest of host StepSlices / state batches, ready(), adopt_* (version
    rules), update() / make_snapshot(), accessors
The bound learners use the reference's mt19937_64 sample stream
(PQL_B200_SAMPLER=mt19937), so both sides train on the same rows; the bars
are the precision mode's (test_precision_gpu.py).
"""
import numpy as np
import pytest

from oracle_lib import param_count, ptr, ref, ref_b200
from oracle_model import f32

pytestmark = pytest.mark.gpu

PRECISIONS = {"tf32": 2e-3, "3xtf32": 1e-4}


def libs():
    R, B = ref(), ref_b200()
    if R is None or B is None:
        pytest.skip("oracle/_ref/libpqlref{,_b200}.so not built (make -C oracle ref b200)")
    return R, B


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / (np.linalg.norm(b) + 1e-30))


@pytest.fixture(params=sorted(PRECISIONS))
def prec(request, monkeypatch):
    monkeypatch.setenv("PQL_B200_SAMPLER", "mt19937")
    monkeypatch.setenv("PQL_B200_PRECISION", request.param)
    return request.param


def test_critic_learner_core_bound_vs_reference(prec):
    R, B = libs()
    N, D, A, H, Bt, cap = 64, 11, 3, 64, 256, 5000
    P = param_count([D + A, H, H, 1])
    h = [L.ref_vcore_create(N, Bt, cap, H, D, A, 0, 7, np.float32(1.0), 0) for L in (R, B)]
    # the bound core starts from the reference's CriticPair::create parameters
    for w in range(4):
        a, b = np.zeros(P, np.float32), np.zeros(P, np.float32)
        R.ref_vcore_params(h[0], w, ptr(a))
        B.ref_vcore_params(h[1], w, ptr(b))
        assert np.array_equal(a, b), w
    rng = np.random.default_rng(31)
    for L, hh in zip((R, B), h):
        assert L.ref_vcore_ready(hh, 100) == 0
        loss = np.zeros(1, np.float32)
        assert L.ref_vcore_update(hh, ptr(loss)) == -2  # before warm-up: runtime_error
    for t in range(12):
        obs = f32(rng.standard_normal((N, D)))
        act = f32(rng.uniform(-1, 1, (N, A)))
        boot = f32(rng.standard_normal((N, D)))
        rew = f32(rng.standard_normal(N))
        term = (rng.random(N) < 0.05).astype(np.uint8)
        trunc = ((rng.random(N) < 0.05) & (term == 0)).astype(np.uint8)
        for L, hh in zip((R, B), h):
            L.ref_vcore_ingest(hh, ptr(obs), ptr(act), ptr(boot), ptr(rew), ptr(term), ptr(trunc))
    assert R.ref_vcore_buffer_size(h[0]) == B.ref_vcore_buffer_size(h[1]) > Bt
    assert R.ref_vcore_ready(h[0], 40) == B.ref_vcore_ready(h[1], 40) == 1
    assert R.ref_vcore_ready(h[0], 31) == B.ref_vcore_ready(h[1], 31) == 0  # warm_up 32
    pol = f32(rng.standard_normal(param_count([D, H, H, A])) * 0.1)
    mean, m2 = rng.standard_normal(D) * 0.1, np.abs(rng.standard_normal(D)) * 500 + 100
    for L, hh in zip((R, B), h):
        L.ref_vcore_adopt_policy(hh, ptr(pol), 3)
        L.ref_vcore_adopt_norm(hh, 400, ptr(mean), ptr(m2))
    bar = PRECISIONS[prec]
    for k in range(3):
        la, lb = np.zeros(1, np.float32), np.zeros(1, np.float32)
        assert R.ref_vcore_update(h[0], ptr(la)) == 0
        assert B.ref_vcore_update(h[1], ptr(lb)) == 0
        print(f"\n{prec} update {k}: loss ref={la[0]:.7f} b200={lb[0]:.7f}")
        assert abs(la[0] - lb[0]) <= bar * abs(la[0])
    worst = 0.0
    for w in range(4):
        a, b = np.zeros(P, np.float32), np.zeros(P, np.float32)
        R.ref_vcore_params(h[0], w, ptr(a))
        B.ref_vcore_params(h[1], w, ptr(b))
        worst = max(worst, rel(b, a))
        assert rel(b, a) <= bar, (w, rel(b, a))
    s = [[np.zeros(P, np.float32) for _ in range(2)] for _ in range(2)]
    R.ref_vcore_snapshot(h[0], 9, ptr(s[0][0]), ptr(s[0][1]))
    B.ref_vcore_snapshot(h[1], 9, ptr(s[1][0]), ptr(s[1][1]))
    assert rel(s[1][0], s[0][0]) <= bar and rel(s[1][1], s[0][1]) <= bar
    print(f"  weights worst rel {worst:.2e}")
    for L, hh in zip((R, B), h):
        L.ref_vcore_destroy(hh)


def test_policy_learner_core_bound_vs_reference(prec):
    R, B = libs()
    D, A, H, Bt, cap = 13, 4, 64, 256, 4000
    Pp, Pq = param_count([D, H, H, A]), param_count([D + A, H, H, 1])
    h = [L.ref_pcore_create(Bt, cap, H, D, A, 0, 9, 0) for L in (R, B)]
    a, b = np.zeros(Pp, np.float32), np.zeros(Pp, np.float32)
    R.ref_pcore_snapshot(h[0], 0, ptr(a), None)
    B.ref_pcore_snapshot(h[1], 0, ptr(b), None)
    assert np.array_equal(a, b)  # PolicyHandle::create on both sides
    rng = np.random.default_rng(32)
    states = f32(rng.standard_normal((1000, D)))
    q1, q2 = f32(rng.standard_normal(Pq) * 0.05), f32(rng.standard_normal(Pq) * 0.05)
    junk = f32(np.full(Pq, 7.0))
    mean, m2 = rng.standard_normal(D) * 0.1, np.abs(rng.standard_normal(D)) * 500 + 100
    for L, hh in zip((R, B), h):
        L.ref_pcore_ingest(hh, ptr(states), 1000)
        L.ref_pcore_adopt_critics(hh, ptr(q1), ptr(q2), 4)
        L.ref_pcore_adopt_critics(hh, ptr(junk), ptr(junk), 3)  # older: ignored
        L.ref_pcore_adopt_norm(hh, 1000, ptr(mean), ptr(m2))
    assert R.ref_pcore_buffer_size(h[0]) == B.ref_pcore_buffer_size(h[1]) == 1000
    assert R.ref_pcore_ready(h[0], 32) == B.ref_pcore_ready(h[1], 32) == 1
    bar = PRECISIONS[prec]
    for k in range(3):
        la, lb = np.zeros(1, np.float32), np.zeros(1, np.float32)
        assert R.ref_pcore_update(h[0], ptr(la)) == 0
        assert B.ref_pcore_update(h[1], ptr(lb)) == 0
        print(f"\n{prec} policy update {k}: loss ref={la[0]:.7f} b200={lb[0]:.7f}")
        assert abs(la[0] - lb[0]) <= bar * max(abs(la[0]), 0.05)
    R.ref_pcore_snapshot(h[0], 5, ptr(a), None)
    B.ref_pcore_snapshot(h[1], 5, ptr(b), None)
    print(f"  policy weights rel {rel(b, a):.2e}")
    assert rel(b, a) <= bar
    for L, hh in zip((R, B), h):
        L.ref_pcore_destroy(hh)


def test_actor_core_bound_vs_reference(prec):
    """rt::ActorCore::rollout_step, unpatched (SyntheticEnv through the
    make_env seam, CPU) vs bound (the device actor): StepSlices and the
    normalizer the accessor exposes."""
    R, B = libs()
    N, D, A, H, seed, max_len, T = 256, 32, 8, 256, 5, 50, 4
    h = [L.ref_actor_core_create(N, D, A, H, seed, 0.05, 0.8, -1.0, max_len, 0) for L in (R, B)]
    bar = PRECISIONS[prec]
    for t in range(T):
        out = []
        for L, hh in zip((R, B), h):
            o = dict(obs=np.zeros((N, D), np.float32), act=np.zeros((N, A), np.float32),
                     boot=np.zeros((N, D), np.float32), rew=np.zeros(N, np.float32),
                     term=np.zeros(N, np.uint8), trunc=np.zeros(N, np.uint8))
            assert L.ref_actor_core_step(hh, *(ptr(o[k]) for k in ("obs", "act", "boot", "rew",
                                                                  "term", "trunc"))) == 0
            out.append(o)
        if t == 0:
            assert np.array_equal(out[0]["obs"], out[1]["obs"])
        for key in ("obs", "act", "boot", "rew"):
            assert rel(out[1][key], out[0][key]) <= bar, (t, key)
        assert np.array_equal(out[0]["term"], out[1]["term"])
        assert np.array_equal(out[0]["trunc"], out[1]["trunc"])
    c = [np.zeros(1, np.int64) for _ in range(2)]
    mean = [np.zeros(D) for _ in range(2)]
    m2 = [np.zeros(D) for _ in range(2)]
    for i, (L, hh) in enumerate(zip((R, B), h)):
        L.ref_actor_core_norm(hh, ptr(c[i]), ptr(mean[i]), ptr(m2[i]))
    assert c[0][0] == c[1][0] == N * T
    np.testing.assert_allclose(m2[1], m2[0], rtol=bar)
    for L, hh in zip((R, B), h):
        L.ref_actor_core_destroy(hh)

