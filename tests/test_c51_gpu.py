"""PQL-D (C51 categorical critic, c51.hpp) on the GPU vs the reference and
the oracle: V-learner (c51_critic_loss update) and P-learner (c51_actor_loss
update).  Tolerances as in test_vlearner_gpu.py (TF32 GEMMs): losses rel
2e-3, dLoss/dlogits and gradients norm-wise 1e-2, post-update weights
norm-wise 2e-3 and per element |dw| <= 2*lr*k + 1e-3*|w|."""
import ctypes as C
from pathlib import Path

import numpy as np
import pytest

from oracle_lib import param_count, ptr
from oracle_model import OraclePUpdate, OracleVUpdate, f32
from paper_2307_12983_b200 import _lib
from test_vlearner_gpu import (adopt_norm, check_weights, insert_rows, params, random_rows, rel,
                               set_params)

pytestmark = pytest.mark.gpu
GOLDEN = Path(__file__).resolve().parent / "golden"


def make_vl(D, A, H, nh, B, cap, L=51, seed=0, init_seed=12345, n_envs=4):
    cfg = _lib.default_config(algo=_lib.ALGO_C51, n_atoms=L, vmin=-10.0, vmax=10.0, batch_size=B,
                              buffer_capacity=cap, hidden=H, hidden_layers=nh, n_envs=n_envs,
                              seed=seed)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), init_seed, None, C.byref(h))
    return h


def make_pl(D, A, H, nh, B, cap, L=51, seed=0):
    cfg = _lib.default_config(algo=_lib.ALGO_C51, n_atoms=L, vmin=-10.0, vmax=10.0, batch_size=B,
                              buffer_capacity=cap, hidden=H, hidden_layers=nh, seed=seed)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 12345, None, C.byref(h))
    return h


def pl_get(h, which, n):
    out = np.zeros(n, np.float32)
    _lib.call("pqlg_plearner_get_params", h, which, ptr(out))
    return out


def pl_put(h, which, arr):
    arr = f32(arr)
    _lib.call("pqlg_plearner_set_params", h, which, ptr(arr))


def pl_ingest(h, rows):
    import torch
    d = torch.from_numpy(f32(rows)).cuda()
    _lib.call("pqlg_plearner_ingest", h, d.data_ptr(), 0, rows.shape[0])
    torch.cuda.synchronize()


def test_c51_vlearner_k_steps_vs_reference_golden():
    G = np.load(GOLDEN / "c51update.npz")
    D, A, H, nh, B, cap, L = (int(v) for v in G["cu_dims"])
    h = make_vl(D, A, H, nh, B, cap, L)
    set_params(h, 0, G["cu_q1"]); set_params(h, 1, G["cu_q2"])
    set_params(h, 2, G["cu_q1"]); set_params(h, 3, G["cu_q2"])
    set_params(h, 4, G["cu_pol"])
    insert_rows(h, G["cu_obs"], G["cu_act"], G["cu_boot"], G["cu_ret"], G["cu_eff"])
    adopt_norm(h, int(G["cu_norm"][0]), G["cu_mean"], G["cu_m2"])
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)
    losses = []
    for _ in range(3):
        l = C.c_float()
        _lib.call("pqlg_vlearner_update", h, C.byref(l))
        losses.append(l.value)
    print("losses gpu", losses, "ref", G["cu_losses"])
    np.testing.assert_allclose(losses, G["cu_losses"], rtol=2e-3)
    P = param_count([D + A] + [H] * nh + [L])
    for w in range(4):
        check_weights(params(h, w, P), G["cu_params"][w], 5e-4, 3)
    _lib.call("pqlg_vlearner_destroy", h)


def test_c51_plearner_k_steps_vs_reference_golden():
    G = np.load(GOLDEN / "c51update.npz")
    D, A, H, nh, B, cap, L = (int(v) for v in G["cu_dims"])
    h = make_pl(D, A, H, nh, B, cap, L)
    pl_put(h, 0, G["cu_pol"]); pl_put(h, 1, G["cu_q1"]); pl_put(h, 2, G["cu_q2"])
    pl_ingest(h, G["cu_obs"])
    mean = np.ascontiguousarray(G["cu_mean"], np.float64)
    m2 = np.ascontiguousarray(G["cu_m2"], np.float64)
    ns = _lib.NormStats(int(G["cu_norm"][0]), ptr(mean), ptr(m2))
    _lib.call("pqlg_plearner_adopt_norm", h, C.byref(ns))
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    losses = []
    for _ in range(3):
        l = C.c_float()
        _lib.call("pqlg_plearner_update", h, C.byref(l))
        losses.append(l.value)
    print("actor losses gpu", losses, "ref", G["cpu_losses"])
    # the actor loss is a mean of -min E terms: compare on the scale of the atoms
    assert np.max(np.abs(np.array(losses) - G["cpu_losses"])) <= 2e-3 * 10.0
    check_weights(pl_get(h, 0, param_count([D] + [H] * nh + [A])), G["cpu_params"], 5e-4, 3)
    _lib.call("pqlg_plearner_destroy", h)


@pytest.mark.parametrize("cfg", ["small", "c4"])
def test_c51_update_intermediates_and_weights_vs_oracle(cfg):
    dims = {"small": (32, 8, 256, 2, 1024, 20000), "c4": (211, 20, 512, 3, 8192, 30000)}[cfg]
    D, A, H, nh, B, n = dims
    L = 51
    rng = np.random.default_rng(11)
    h = make_vl(D, A, H, nh, B, n + 10, L)
    P = param_count([D + A] + [H] * nh + [L])
    q1, q2 = params(h, 0, P), params(h, 1, P)
    pol = params(h, 4, param_count([D] + [H] * nh + [A]))
    obs, act, boot, ret, eff = random_rows(rng, n, D, A)
    ret = f32(ret * 20.0)  # spread the targets over the support
    insert_rows(h, obs, act, boot, ret, eff)
    count = 10**6
    mean, m2 = adopt_norm(h, count, rng.standard_normal(D) * 0.1,
                          np.abs(rng.standard_normal(D)) * count + count * 0.5)
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)
    o = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, distributional=True, n_atoms=L)
    o.set_rows(obs, act, boot, ret, eff)
    o.norm = (count, mean, m2)
    k = 2
    for step in range(k):
        loss_o, info = o.step()
        l = C.c_float()
        _lib.call("pqlg_vlearner_update", h, C.byref(l))
        g = np.zeros(2 * P, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 2, ptr(g))
        sc = np.zeros(2, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 3, ptr(sc))
        r = [rel(g[kk * P:(kk + 1) * P] * sc[kk], info["dq"][kk]) for kk in range(2)]
        print(f"\n{cfg} step {step}: loss gpu={l.value:.6f} oracle={loss_o:.6f} g_rel={r}")
        assert abs(l.value - loss_o) <= 2e-3 * abs(loss_o)
        for kk in range(2):
            assert r[kk] <= 1e-2, r
    for w, want in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        check_weights(params(h, w, P), want, 5e-4, k)
    _lib.call("pqlg_vlearner_destroy", h)


def test_c51_graph_update_n_philox_vs_oracle():
    D, A, H, nh, B, n, L = 32, 8, 256, 2, 1024, 5000, 51
    rng = np.random.default_rng(12)
    h = make_vl(D, A, H, nh, B, n, L)
    P = param_count([D + A] + [H] * nh + [L])
    q1, q2 = params(h, 0, P), params(h, 1, P)
    pol = params(h, 4, param_count([D] + [H] * nh + [A]))
    rows = list(random_rows(rng, n, D, A))
    rows[3] = f32(rows[3] * 20.0)
    insert_rows(h, *rows)
    o = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, philox=True, distributional=True,
                      n_atoms=L)
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


@pytest.mark.parametrize("cfg", ["small", "c4"])
def test_c51_plearner_vs_oracle(cfg):
    D, A, H, nh, B, n = {"small": (31, 7, 256, 2, 1024, 5000),
                         "c4": (211, 20, 512, 3, 8192, 20000)}[cfg]
    L = 51
    rng = np.random.default_rng(13)
    h = make_pl(D, A, H, nh, B, n, L)
    Pp = param_count([D] + [H] * nh + [A])
    Pq = param_count([D + A] + [H] * nh + [L])
    pol, q1, q2 = pl_get(h, 0, Pp), pl_get(h, 1, Pq), pl_get(h, 2, Pq)
    states = f32(rng.standard_normal((n, D)))
    pl_ingest(h, states)
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    o = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, distributional=True, n_atoms=L)
    o.states = states
    k = 2
    for _ in range(k):
        lo, info = o.step()
        l = C.c_float()
        _lib.call("pqlg_plearner_update", h, C.byref(l))
        print(f"\n{cfg}: actor loss gpu={l.value:.6f} oracle={lo:.6f}")
        assert abs(l.value - lo) <= 2e-3 * 10.0
    check_weights(pl_get(h, 0, Pp), o.pol, 5e-4, k)
    _lib.call("pqlg_plearner_destroy", h)


def test_c51_rejects_bad_support():
    with pytest.raises(ValueError):
        make_vl(8, 2, 32, 2, 16, 100, L=65)
    cfg = _lib.default_config(algo=_lib.ALGO_C51, vmin=1.0, vmax=-1.0, batch_size=16,
                              buffer_capacity=100, hidden=32)
    dims = _lib.TaskDims(8, 2, -1.0, 1.0)
    h = C.c_void_p()
    with pytest.raises(ValueError):
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, None, C.byref(h))


@pytest.mark.parametrize("L", [2, 33, 64])
def test_c51_atom_count_edges_vs_oracle(L):
    """The categorical head at the smallest support (2 atoms), a ragged one
    (33: two 32-column chunks, the second nearly empty) and the largest the
    kernels take (64): one critic update vs the oracle."""
    D, A, H, nh, B, n = 12, 3, 64, 2, 256, 3000
    rng = np.random.default_rng(40 + L)
    h = make_vl(D, A, H, nh, B, n, L)
    P = param_count([D + A] + [H] * nh + [L])
    q1, q2 = params(h, 0, P), params(h, 1, P)
    pol = params(h, 4, param_count([D] + [H] * nh + [A]))
    obs, act, boot, ret, eff = random_rows(rng, n, D, A)
    ret = f32(ret * 20.0)
    insert_rows(h, obs, act, boot, ret, eff)
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)
    o = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, distributional=True, n_atoms=L)
    o.set_rows(obs, act, boot, ret, eff)
    loss_o, info = o.step()
    l = C.c_float()
    _lib.call("pqlg_vlearner_update", h, C.byref(l))
    g = np.zeros(2 * P, np.float32)
    _lib.call("pqlg_vlearner_debug_read", h, 2, ptr(g))
    sc = np.zeros(2, np.float32)
    _lib.call("pqlg_vlearner_debug_read", h, 3, ptr(sc))
    r = [rel(g[k * P:(k + 1) * P] * sc[k], info["dq"][k]) for k in range(2)]
    print(f"\nL={L}: loss gpu={l.value:.6f} oracle={loss_o:.6f} g_rel={r}")
    assert abs(l.value - loss_o) <= 2e-3 * abs(loss_o)
    assert max(r) <= 1e-2
    for w, want in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]]):
        check_weights(params(h, w, P), want, 5e-4, 1)
    _lib.call("pqlg_vlearner_destroy", h)
