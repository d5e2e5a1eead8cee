"""evaluate_policy (learners.cpp:280-325) on the GPU vs the reference's own
rt::evaluate_policy on the synthetic task (tests/golden/evaluate.npz: the
unmodified function, with make_env returning SyntheticEnv -- see
oracle/ref_harness.cpp) and vs the oracle restatement (orc_evaluate):
per-episode returns, mean and standard error.  Actions come from the
TF32 / 3xTF32 policy, so returns are compared with the precision mode's
tolerance; the env and the accumulation are exact."""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import orc, param_count, ptr, sizes_arr
from oracle_model import f32
from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("max_len", [40, 200])
def test_evaluate_matches_oracle(max_len):
    D, A, H, nh, M = 19, 6, 64, 2, 96
    rng = np.random.default_rng(4)
    ps = [D] + [H] * nh + [A]
    pol = f32(rng.standard_normal(param_count(ps)) * 0.1)
    mean = rng.standard_normal(D) * 0.1
    m2 = np.abs(rng.standard_normal(D)) * 50 + 10
    count = 100
    cfg = _lib.default_config(hidden=H, hidden_layers=nh, max_episode_len=max_len)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    ret = np.zeros(M)
    mu, se = C.c_double(), C.c_double()
    ns = _lib.NormStats(count, ptr(mean), ptr(m2))
    _lib.call("pqlg_evaluate", C.byref(cfg), C.byref(dims), ptr(pol), C.byref(ns), M, 77,
              ptr(ret), C.byref(mu), C.byref(se))
    want = np.zeros(M)
    om, ose = np.zeros(1), np.zeros(1)
    assert orc().orc_evaluate(ptr(pol), ptr(sizes_arr(ps)), nh + 1, count, ptr(mean), ptr(m2), M,
                              77, D, A, np.float32(-1), np.float32(1), max_len, ptr(want),
                              ptr(om), ptr(ose)) == 0
    print(f"\nmax_len={max_len}: mean gpu={mu.value:.6f} oracle={om[0]:.6f} "
          f"stderr {se.value:.6f}/{ose[0]:.6f} max|dret|={np.max(np.abs(ret - want)):.2e}")
    assert np.allclose(ret, want, rtol=2e-3, atol=2e-3)
    assert abs(mu.value - om[0]) <= 2e-3 * abs(om[0]) + 1e-6
    # the reported statistics are the reference's formulas over the returns
    assert mu.value == pytest.approx(np.mean(ret), rel=1e-12)
    assert se.value == pytest.approx(np.std(ret, ddof=1) / np.sqrt(M), rel=1e-9)


@pytest.mark.parametrize("prec", [_lib.PREC_TF32, _lib.PREC_3XTF32])
@pytest.mark.parametrize("k", [0, 1, 2, 3])
def test_evaluate_vs_reference_golden(k, prec):
    from pathlib import Path
    G = np.load(Path(__file__).resolve().parent / "golden" / "evaluate.npz")
    D, A, H, nh, M, seed, max_len, sac, count = (int(x) for x in G[f"ev{k}_args"])
    cfg = _lib.default_config(hidden=H, hidden_layers=nh, max_episode_len=max_len,
                              algo=_lib.ALGO_SAC if sac else _lib.ALGO_DDPG, precision=prec)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    mean = np.ascontiguousarray(G[f"ev{k}_mean"])
    m2 = np.ascontiguousarray(G[f"ev{k}_m2"])
    ns = _lib.NormStats(count, ptr(mean), ptr(m2))
    mu, se = C.c_double(), C.c_double()
    _lib.call("pqlg_evaluate", C.byref(cfg), C.byref(dims), ptr(G[f"ev{k}_policy"]), C.byref(ns),
              M, seed, None, C.byref(mu), C.byref(se))
    want_mu, want_se = G[f"ev{k}_result"]
    bar = 2e-3 if prec == _lib.PREC_TF32 else 2e-5
    print(f"\nevaluate case {k} prec {prec}: mean gpu={mu.value:.8f} ref={want_mu:.8f} "
          f"stderr {se.value:.8f}/{want_se:.8f}")
    assert abs(mu.value - want_mu) <= bar * abs(want_mu) + 1e-6
    assert abs(se.value - want_se) <= 10 * bar * abs(want_se) + 1e-6


@pytest.mark.parametrize("algo", [_lib.ALGO_DDPG, _lib.ALGO_SAC])
def test_evaluator_reuse_equals_fresh(algo):
    """The metrics loops keep one Evaluator (env, policy and buffers allocated
    once) and run it per row: each run must equal a fresh pqlg_evaluate of the
    same policy, bit for bit (env streams restored, episodes restarted)."""
    D, A, H, nh, M = 13, 5, 64, 2, 80
    rng = np.random.default_rng(9)
    hout = 2 * A if algo == _lib.ALGO_SAC else A
    ps = [D] + [H] * nh + [hout]
    P = param_count(ps)
    pols = f32(rng.standard_normal((3, P)) * 0.1)
    pols[2] = pols[0]  # a policy seen before returns the same episodes
    mean = rng.standard_normal(D) * 0.1
    m2 = np.abs(rng.standard_normal(D)) * 50 + 10
    cfg = _lib.default_config(hidden=H, hidden_layers=nh, max_episode_len=60, algo=algo)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    ns = _lib.NormStats(100, ptr(mean), ptr(m2))
    ret = np.zeros((3, M))
    mu, se = np.zeros(3), np.zeros(3)
    _lib.call("pqlg_k_evaluate_seq", C.byref(cfg), C.byref(dims), ptr(pols), 3, C.byref(ns), M, 31,
              ptr(ret), ptr(mu), ptr(se))
    for k in range(3):
        want = np.zeros(M)
        m1, s1 = C.c_double(), C.c_double()
        _lib.call("pqlg_evaluate", C.byref(cfg), C.byref(dims), ptr(np.ascontiguousarray(pols[k])),
                  C.byref(ns), M, 31, ptr(want), C.byref(m1), C.byref(s1))
        np.testing.assert_array_equal(ret[k], want)
        assert (mu[k], se[k]) == (m1.value, s1.value)
    np.testing.assert_array_equal(ret[2], ret[0])
    assert not np.array_equal(ret[1], ret[0])
