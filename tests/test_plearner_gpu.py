"""P-learner (PolicyLearnerCore) on the GPU vs the oracle / reference.
Tolerances as in test_vlearner_gpu.py (TF32 GEMMs): losses rel 2e-3,
post-update policy weights norm-wise <= 2e-3 and per element
|dw| <= 2*lr*k + 1e-3*|w|."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import param_count, ptr
from oracle_model import OraclePUpdate, f32
from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def make_pl(D, A, H, nh, B, cap, seed=0, init_seed=12345):
    cfg = _lib.default_config(batch_size=B, buffer_capacity=cap, hidden=H, hidden_layers=nh,
                              seed=seed)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), init_seed, None, C.byref(h))
    return h


def get(h, which, n):
    out = np.zeros(n, np.float32)
    _lib.call("pqlg_plearner_get_params", h, which, ptr(out))
    return out


def put(h, which, arr):
    arr = f32(arr)
    _lib.call("pqlg_plearner_set_params", h, which, ptr(arr))


def ingest(h, rows):
    import torch
    d = torch.from_numpy(f32(rows)).cuda()
    _lib.call("pqlg_plearner_ingest", h, d.data_ptr(), 0, rows.shape[0])
    torch.cuda.synchronize()


def adopt_norm(h, count, mean, m2):
    mean = np.ascontiguousarray(mean, np.float64)
    m2 = np.ascontiguousarray(m2, np.float64)
    ns = _lib.NormStats(count, ptr(mean), ptr(m2))
    _lib.call("pqlg_plearner_adopt_norm", h, C.byref(ns))
    return mean, m2


def rel(a, b):
    return float(np.linalg.norm(np.asarray(a, np.float64) - b) / (np.linalg.norm(b) + 1e-30))


def check_weights(got, want, lr, k, tol=2e-3):
    r = rel(got, want)
    print(f"  policy weights rel={r:.2e} max|dw|={np.max(np.abs(got - want)):.2e}")
    assert r <= tol, r
    assert np.all(np.abs(got - want) <= 2 * lr * k + 1e-3 * np.abs(want) + 1e-7)


def test_init_matches_reference():
    G = np.load(GOLDEN / "mlp.npz")
    h = make_pl(6, 3, 32, 2, 8, 64, seed=0, init_seed=12345)
    P = param_count([9, 32, 32, 1])
    assert np.array_equal(get(h, 0, param_count([6, 32, 32, 3])), G["init_policy_h32"])
    assert np.array_equal(get(h, 1, P), G["init_critics_h32"][:P])
    assert np.array_equal(get(h, 2, P), G["init_critics_h32"][P:])
    _lib.call("pqlg_plearner_destroy", h)


def test_k_step_updates_vs_reference_golden():
    G = np.load(GOLDEN / "vupdate.npz")
    D, A, H, nh, B, cap = (int(v) for v in G["vu_dims"])
    h = make_pl(D, A, H, nh, B, cap)
    put(h, 0, G["vu_pol"]); put(h, 1, G["vu_q1"]); put(h, 2, G["vu_q2"])
    ingest(h, G["vu_obs"])
    adopt_norm(h, int(G["vu_norm"][0]), G["vu_mean"], G["vu_m2"])
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    # the oracle replays the same steps to measure the objective's term scale
    o = OraclePUpdate(D, A, H, nh, B, G["vu_pol"], G["vu_q1"], G["vu_q2"])
    o.states = G["vu_obs"]
    o.norm = (int(G["vu_norm"][0]), G["vu_mean"], G["vu_m2"])
    for k in range(3):
        l = C.c_float()
        _lib.call("pqlg_plearner_update", h, C.byref(l))
        _, info = o.step()
        ref_loss = float(G["pu_losses"][k])
        print(f"\ngolden step {k}: actor loss gpu={l.value:.6f} ref={ref_loss:.6f} "
              f"qscale={info['qscale']:.4f}")
        # loss = -mean min(Q1,Q2): terms of size qscale largely cancel
        assert abs(l.value - ref_loss) <= 2e-3 * info["qscale"]
    check_weights(get(h, 0, param_count([D] + [H] * nh + [A])), G["pu_params"], 5e-4, 3)
    _lib.call("pqlg_plearner_destroy", h)


@pytest.mark.parametrize("cfg", ["odd_act", "c1", "c3"])
def test_updates_vs_oracle(cfg):
    D, A, H, nh, B, n = {"odd_act": (13, 3, 64, 2, 300, 1000), "c1": (32, 8, 256, 2, 1024, 8000),
                         "c3": (211, 20, 512, 3, 8192, 20000)}[cfg]
    rng = np.random.default_rng(4)
    h = make_pl(D, A, H, nh, B, n + 5)
    pol = get(h, 0, param_count([D] + [H] * nh + [A]))
    # trained-looking critics: random small weights so the actor gradient is non-trivial
    P = param_count([D + A] + [H] * nh + [1])
    q1 = f32(rng.standard_normal(P) * 0.05)
    q2 = f32(rng.standard_normal(P) * 0.05)
    put(h, 1, q1); put(h, 2, q2)
    states = f32(rng.standard_normal((n, D)))
    ingest(h, states)
    count = 10 ** 6
    mean, m2 = adopt_norm(h, count, rng.standard_normal(D) * 0.1,
                          np.abs(rng.standard_normal(D)) * count + count * 0.5)
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    o = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, seed=0)
    o.states = states
    o.norm = (count, mean, m2)
    k = 2
    for step in range(k):
        loss_o, info = o.step()
        l = C.c_float()
        _lib.call("pqlg_plearner_update", h, C.byref(l))
        print(f"\n{cfg} step {step}: actor loss gpu={l.value:.6f} oracle={loss_o:.6f} "
              f"qscale={info['qscale']:.4f}")
        assert abs(l.value - loss_o) <= 2e-3 * info["qscale"]
    check_weights(get(h, 0, pol.size), o.pol, 5e-4, k)
    _lib.call("pqlg_plearner_destroy", h)


def test_graph_update_n_philox_vs_oracle():
    D, A, H, nh, B, n = 32, 8, 256, 2, 1024, 5000
    rng = np.random.default_rng(5)
    h = make_pl(D, A, H, nh, B, n)
    pol = get(h, 0, param_count([D] + [H] * nh + [A]))
    P = param_count([D + A] + [H] * nh + [1])
    q1, q2 = f32(rng.standard_normal(P) * 0.05), f32(rng.standard_normal(P) * 0.05)
    put(h, 1, q1); put(h, 2, q2)
    states = f32(rng.standard_normal((n, D)))
    ingest(h, states)
    o = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, seed=0, philox=True)
    o.states = states
    k = 4
    _lib.call("pqlg_plearner_update_n", h, k)
    res = [o.step() for _ in range(k)]
    l = C.c_float()
    _lib.call("pqlg_plearner_last_loss", h, C.byref(l))
    assert abs(l.value - res[-1][0]) <= 2e-3 * res[-1][1]["qscale"]
    check_weights(get(h, 0, pol.size), o.pol, 5e-4, k)
    _lib.call("pqlg_plearner_destroy", h)


def test_version_rule_and_not_ready():
    D, A, H = 5, 2, 32
    h = make_pl(D, A, H, 2, 64, 500)
    with pytest.raises(_lib.NotReady):
        _lib.call("pqlg_plearner_update", h, C.byref(C.c_float()))
    P = param_count([D + A, H, H, 1])
    a = f32(np.ones(P)); b = f32(np.full(P, 2.0))
    _lib.call("pqlg_plearner_adopt_critics", h, ptr(a), ptr(a), 5)
    _lib.call("pqlg_plearner_adopt_critics", h, ptr(b), ptr(b), 4)  # older: ignored
    assert np.all(get(h, 1, P) == 1.0)
    _lib.call("pqlg_plearner_adopt_critics", h, ptr(b), ptr(b), 5)  # equal: replaces
    assert np.all(get(h, 2, P) == 2.0)
    _lib.call("pqlg_plearner_destroy", h)
