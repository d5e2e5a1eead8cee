"""GEMM precision modes vs the fp32 oracle, at every config.

The reference computes every affine op in fp32 (scalar.hpp:12-55,
avx2.cpp:37-300).  `pqlg_config.precision` selects
  - TF32    (speed mode): operands rounded to tf32, one tcgen05 MMA per K step
  - 3XTF32  (parity mode): hi/lo tf32 split in shared memory, three MMAs
            accumulated in fp32 (gemm_tf32.cuh, k3x)

Two oracle runs per test: a free-running one (the k-step comparison of the
post-update weights) and a synchronised one whose parameters are reset to the
device's before every update, so each update's TD targets, loss and
gradients are compared on identical inputs (otherwise Adam's sign-like first
steps amplify any last-bit difference into the next update's weights; the
compiled reference's own AVX2 and scalar backends drift apart by 8e-5 in
weights after 3 updates at c3 for the same reason).

Bars written here (norm-wise relative error unless stated):
                           TF32     3XTF32
  TD targets y, loss       2e-3     1e-3    every update, synchronised
  pre-clip gradients       1e-2     1e-3    every update, synchronised
  post-update weights      2e-3     1e-3    free-running, after k = 3 updates
  per-element weights      |dw_i| <= 2 lr k + 1e-3 |w_i|  (both)

3XTF32 is not bit-for-bit fp32: the tcgen05 fp32 accumulator rounds every
MMA's sum toward zero (tools/prec_probe.py: a mean bias of about -1e-8 x K/8
MMA steps on same-sign data, 3x that with three MMAs per step), so a K = 512
layer sits near 1e-6 relative where a CPU fp32 loop sits near 1e-7.

The actor loss is a mean of largely cancelling terms: its bar is stated on
the scale of those terms (mean |min(Q1, Q2)|, or the support width 10 for
C51), as in test_plearner_gpu.py.

Also here: the clip + Adam + Polyak step on the device is bit-exact against
the compiled reference's own fa::clip_global_norm / fa::adam_step /
fa::soft_update (optim.hpp:28-79) fed the learner's own pre-clip gradients.

Observed magnitudes are appended to $PQLG_ERRLOG (JSON lines) when set;
profiles/r2_precision_errors.jsonl is that log from the B200.
"""
import ctypes as C
import json
import os

import numpy as np
import pytest

from oracle_lib import param_count, ptr, ref
from oracle_model import OraclePUpdate, OracleVUpdate, f32
from paper_2307_12983_b200 import _lib
from test_vlearner_gpu import adopt_norm, insert_rows, params, random_rows, rel

pytestmark = pytest.mark.gpu

CFGS = {  # D, A, H, hidden layers, B, live rows
    "c1": (32, 8, 256, 2, 1024, 20000),
    "c2": (60, 8, 512, 3, 8192, 30000),
    "c3": (211, 20, 512, 3, 8192, 30000),
    "c4": (211, 20, 512, 3, 8192, 30000),
}
BARS = {  # y/loss, gradients, weights
    _lib.PREC_TF32: (2e-3, 1e-2, 2e-3),
    _lib.PREC_3XTF32: (1e-3, 1e-3, 1e-3),
}
PREC_NAME = {_lib.PREC_TF32: "tf32", _lib.PREC_3XTF32: "3xtf32"}
K_STEPS = 3
LR = 5e-4


def log_errors(rec):
    path = os.environ.get("PQLG_ERRLOG")
    print("\n" + json.dumps(rec))
    if path:
        with open(path, "a") as f:
            f.write(json.dumps(rec) + "\n")


def weight_errors(got, want, lr, k):
    r = rel(got, want)
    elem_ok = bool(np.all(np.abs(got - want) <= 2 * lr * k + 1e-3 * np.abs(want) + 1e-7))
    return r, float(np.max(np.abs(got - want))), elem_ok


def make_vl(cfg, prec, algo=_lib.ALGO_DDPG):
    D, A, H, nh, B, n = CFGS[cfg]
    c = _lib.default_config(batch_size=B, buffer_capacity=n + 10, hidden=H, hidden_layers=nh,
                            n_envs=4, seed=0, lr_critic=LR, precision=prec, algo=algo,
                            n_atoms=51, vmin=-10.0, vmax=10.0)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(c), C.byref(dims), 12345, None, C.byref(h))
    return h


def make_pl(cfg, prec, algo=_lib.ALGO_DDPG):
    D, A, H, nh, B, n = CFGS[cfg]
    c = _lib.default_config(batch_size=B, buffer_capacity=n + 10, hidden=H, hidden_layers=nh,
                            seed=0, lr_actor=LR, precision=prec, algo=algo, n_atoms=51,
                            vmin=-10.0, vmax=10.0)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(c), C.byref(dims), 12345, None, C.byref(h))
    return h


def run_vlearner(cfg, prec):
    D, A, H, nh, B, n = CFGS[cfg]
    c51 = cfg == "c4"
    L = 51 if c51 else 1
    h = make_vl(cfg, prec, _lib.ALGO_C51 if c51 else _lib.ALGO_DDPG)
    P = param_count([D + A] + [H] * nh + [L])
    q1, q2 = params(h, 0, P), params(h, 1, P)
    pol = params(h, 4, param_count([D] + [H] * nh + [A]))
    rng = np.random.default_rng(21)
    rows = list(random_rows(rng, n, D, A))
    if c51:
        rows[3] = f32(rows[3] * 20.0)  # spread the targets over the support
    insert_rows(h, *rows)
    count = 10**6
    mean, m2 = adopt_norm(h, count, rng.standard_normal(D) * 0.1,
                          np.abs(rng.standard_normal(D)) * count + count * 0.5)
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)
    o = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, distributional=c51, n_atoms=51)
    o.set_rows(*rows)
    o.norm = (count, mean, m2)
    osync = OracleVUpdate(D, A, H, nh, B, q1, q2, pol, seed=0, distributional=c51, n_atoms=51)
    osync.set_rows(*rows)
    osync.norm = (count, mean, m2)
    bar_y, bar_g, bar_w = BARS[prec]
    rec = dict(test="vlearner", cfg=cfg, precision=PREC_NAME[prec], k=K_STEPS, steps=[])
    for step in range(K_STEPS):
        o.step()
        osync.q = [params(h, 0, P), params(h, 1, P)]
        osync.qt = [params(h, 2, P), params(h, 3, P)]
        loss_o, info = osync.step()
        l = C.c_float()
        _lib.call("pqlg_vlearner_update", h, C.byref(l))
        g = np.zeros(2 * P, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 2, ptr(g))
        sc = np.zeros(2, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 3, ptr(sc))
        g_rel = [rel(g[kk * P:(kk + 1) * P] * sc[kk], info["dq"][kk]) for kk in range(2)]
        s = dict(loss_gpu=l.value, loss_oracle=loss_o,
                 loss_rel=abs(l.value - loss_o) / abs(loss_o), g_rel=g_rel)
        if not c51:
            y = np.zeros(B, np.float32)
            _lib.call("pqlg_vlearner_debug_read", h, 0, ptr(y))
            s["y_rel"] = rel(y, info["y"])
        rec["steps"].append(s)
    w = [weight_errors(params(h, i, P), want, LR, K_STEPS)
         for i, want in enumerate([o.q[0], o.q[1], o.qt[0], o.qt[1]])]
    rec["w_rel"] = [x[0] for x in w]
    rec["w_max_abs"] = [x[1] for x in w]
    log_errors(rec)
    _lib.call("pqlg_vlearner_destroy", h)
    for s in rec["steps"]:
        assert s["loss_rel"] <= bar_y, s
        assert s.get("y_rel", 0.0) <= bar_y, s
        assert max(s["g_rel"]) <= bar_g, s
    for r, _, elem_ok in w:
        assert r <= bar_w, w
        assert elem_ok, w


def run_plearner(cfg, prec):
    D, A, H, nh, B, n = CFGS[cfg]
    c51 = cfg == "c4"
    L = 51 if c51 else 1
    h = make_pl(cfg, prec, _lib.ALGO_C51 if c51 else _lib.ALGO_DDPG)
    Pp = param_count([D] + [H] * nh + [A])
    Pq = param_count([D + A] + [H] * nh + [L])
    pol = np.zeros(Pp, np.float32)
    _lib.call("pqlg_plearner_get_params", h, 0, ptr(pol))
    rng = np.random.default_rng(22)
    if c51:  # the P-learner's own (initial) critic replicas
        q1, q2 = np.zeros(Pq, np.float32), np.zeros(Pq, np.float32)
        _lib.call("pqlg_plearner_get_params", h, 1, ptr(q1))
        _lib.call("pqlg_plearner_get_params", h, 2, ptr(q2))
    else:  # trained-looking critics: a non-trivial actor gradient
        q1 = f32(rng.standard_normal(Pq) * 0.05)
        q2 = f32(rng.standard_normal(Pq) * 0.05)
        _lib.call("pqlg_plearner_set_params", h, 1, ptr(q1))
        _lib.call("pqlg_plearner_set_params", h, 2, ptr(q2))
    import torch
    states = f32(rng.standard_normal((n, D)))
    d = torch.from_numpy(states).cuda()
    _lib.call("pqlg_plearner_ingest", h, d.data_ptr(), 0, n)
    torch.cuda.synchronize()
    count = 10**6
    mean = np.ascontiguousarray(rng.standard_normal(D) * 0.1)
    m2 = np.ascontiguousarray(np.abs(rng.standard_normal(D)) * count + count * 0.5)
    ns = _lib.NormStats(count, ptr(mean), ptr(m2))
    _lib.call("pqlg_plearner_adopt_norm", h, C.byref(ns))
    _lib.call("pqlg_plearner_set_sampler", h, _lib.RNG_INDICES)
    o = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, seed=0, distributional=c51, n_atoms=51)
    o.states = states
    o.norm = (count, mean, m2)
    osync = OraclePUpdate(D, A, H, nh, B, pol, q1, q2, seed=0, distributional=c51, n_atoms=51)
    osync.states = states
    osync.norm = (count, mean, m2)
    bar_y, _, bar_w = BARS[prec]
    rec = dict(test="plearner", cfg=cfg, precision=PREC_NAME[prec], k=K_STEPS, steps=[])
    for _ in range(K_STEPS):
        o.step()
        cur = np.zeros(Pp, np.float32)
        _lib.call("pqlg_plearner_get_params", h, 0, ptr(cur))
        osync.pol = cur
        loss_o, info = osync.step()
        l = C.c_float()
        _lib.call("pqlg_plearner_update", h, C.byref(l))
        scale = 10.0 if c51 else info["qscale"]
        rec["steps"].append(dict(loss_gpu=l.value, loss_oracle=loss_o, term_scale=scale,
                                 loss_err_over_scale=abs(l.value - loss_o) / scale))
    got = np.zeros(Pp, np.float32)
    _lib.call("pqlg_plearner_get_params", h, 0, ptr(got))
    r, mx, elem_ok = weight_errors(got, o.pol, LR, K_STEPS)
    rec["w_rel"], rec["w_max_abs"] = r, mx
    log_errors(rec)
    _lib.call("pqlg_plearner_destroy", h)
    for s in rec["steps"]:
        assert s["loss_err_over_scale"] <= bar_y, s
    assert r <= bar_w, rec
    assert elem_ok, rec


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_vlearner_3xtf32_vs_oracle(cfg):
    run_vlearner(cfg, _lib.PREC_3XTF32)


@pytest.mark.parametrize("cfg", ["c1", "c2", "c3", "c4"])
def test_plearner_3xtf32_vs_oracle(cfg):
    run_plearner(cfg, _lib.PREC_3XTF32)


@pytest.mark.parametrize("cfg", ["c2", "c4"])
def test_vlearner_tf32_vs_oracle(cfg):
    # c1 / c3 in TF32 are covered by test_vlearner_gpu.py (k = 2)
    run_vlearner(cfg, _lib.PREC_TF32)


@pytest.mark.parametrize("cfg", ["c2"])
def test_plearner_tf32_vs_oracle(cfg):
    run_plearner(cfg, _lib.PREC_TF32)


# ------------------------------------------------------------- the GEMM itself

GEMM_CASES = [
    # M, N, K, a_mn, b_mn, splits
    (256, 256, 256, 0, 1, 1),      # forward, CTA pair
    (384, 256, 200, 0, 1, 1),      # forward, odd m-tile count (single CTA)
    (300, 20, 40, 0, 1, 1),        # narrow head
    (1024, 512, 512, 0, 0, 1),     # dgrad
    (512, 512, 4096, 1, 1, 8),     # wgrad, split-K
    (231, 512, 1024, 1, 1, 4),     # wgrad of layer 0 (M ragged)
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,splits", GEMM_CASES)
def test_gemm_3xtf32_matches_fp64(M, N, K, a_mn, b_mn, splits):
    from test_gemm_gpu import run_gemm
    rng = np.random.default_rng(M + 5 * N + K)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    D1 = run_gemm(a, b, a_mn, b_mn, splits=splits, round_mode=1)
    D3 = run_gemm(a, b, a_mn, b_mn, splits=splits, round_mode=2)
    R = a.astype(np.float64) @ b.astype(np.float64)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64)
    e1 = float(np.max(np.abs(D1 - R) / scale))
    e3 = float(np.max(np.abs(D3 - R) / scale))
    # fp32 itself: the exactly rounded products summed in fp32
    f32_ref = (a @ b).astype(np.float64)
    ef = float(np.max(np.abs(f32_ref - R) / scale))
    log_errors(dict(test="gemm", shape=[M, N, K, a_mn, b_mn, splits], err_tf32=e1,
                    err_3xtf32=e3, err_fp32_matmul=ef))
    assert e3 < 2e-6, (e1, e3, ef)
    assert e3 < e1 / 50


# -------------------------------------- clip + Adam + Polyak bit-exact (device)

@pytest.mark.parametrize("prec", [_lib.PREC_TF32, _lib.PREC_3XTF32])
def test_clip_adam_polyak_bit_exact_vs_reference(prec):
    """The learner's own pre-clip gradients (debug_read 2) through the
    compiled reference's fa::clip_global_norm, fa::adam_step and
    fa::soft_update reproduce the device's post-update online and target
    weights bit for bit, over 3 consecutive updates (Adam state carried by
    the reference side)."""
    R = ref()
    if R is None:
        pytest.skip("oracle/_ref not built")
    D, A, H, nh, B, n = 32, 8, 256, 2, 1024, 20000
    c = _lib.default_config(batch_size=B, buffer_capacity=n + 10, hidden=H, hidden_layers=nh,
                            n_envs=4, seed=0, lr_critic=LR, precision=prec)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(c), C.byref(dims), 12345, None, C.byref(h))
    P = param_count([D + A] + [H] * nh + [1])
    rng = np.random.default_rng(23)
    insert_rows(h, *random_rows(rng, n, D, A))
    _lib.call("pqlg_vlearner_set_sampler", h, _lib.RNG_INDICES)
    m = [np.zeros(P, np.float32) for _ in range(2)]
    v = [np.zeros(P, np.float32) for _ in range(2)]
    clipped_any = False
    for t in range(3):
        online = [params(h, 0, P), params(h, 1, P)]
        target = [params(h, 2, P), params(h, 3, P)]
        l = C.c_float()
        _lib.call("pqlg_vlearner_update", h, C.byref(l))
        g = np.zeros(2 * P, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 2, ptr(g))
        sc = np.zeros(2, np.float32)
        _lib.call("pqlg_vlearner_debug_read", h, 3, ptr(sc))
        for k in range(2):
            gk = g[k * P:(k + 1) * P].copy()
            R.ref_clip_global_norm(ptr(gk), P, np.float32(0.5))  # learners.cpp:182-183
            # the device's fp64 norm (a different summation order) gives the
            # same fp32 clip scale
            assert np.array_equal(gk, g[k * P:(k + 1) * P] * sc[k]) or sc[k] == 1.0
            clipped_any |= bool(sc[k] != 1.0)
            p = online[k].copy()
            assert R.ref_adam_step(ptr(p), ptr(gk), ptr(m[k]), ptr(v[k]), P, t,
                                   np.float32(LR)) == 0
            assert np.array_equal(p, params(h, k, P)), (t, k)
            tg = target[k].copy()
            R.ref_soft_update(ptr(tg), ptr(p), P, np.float32(0.05))
            assert np.array_equal(tg, params(h, 2 + k, P)), (t, k)
    print(f"\nclip active in at least one update: {clipped_any}")
    _lib.call("pqlg_vlearner_destroy", h)


def test_precision_rejects_unknown_mode():
    c = _lib.default_config(batch_size=16, buffer_capacity=100, hidden=32, precision=7)
    dims = _lib.TaskDims(8, 2, -1.0, 1.0)
    h = C.c_void_p()
    with pytest.raises(ValueError):
        _lib.call("pqlg_vlearner_create", C.byref(c), C.byref(dims), 1, None, C.byref(h))
