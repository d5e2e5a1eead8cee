"""evaluate_policy (learners.cpp:280-325) on the GPU vs the oracle
restatement (orc_evaluate) on the synthetic task: per-episode returns,
mean and standard error.  Actions come from the TF32 policy, so returns are
compared with a tolerance; the env and the accumulation are exact."""
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
