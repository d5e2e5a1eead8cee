"""Data-parallel learners (config 5) on one B200.

The round-end box has one GPU, so the multi-rank exchange itself is covered
by the gloo tests in test_dp_cpu.py; here a world-1 NCCL communicator runs
the data-parallel update path (per-layer buckets on a communication branch:
reduction-only finalize + NCCL all-reduce as each layer's gradient completes
-> norm/clip pass -> Adam, dp_buckets.h) and must equal the plain learner bit
for bit, and a rank-1 learner must sample with its own Philox stream.
"""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import param_count, ptr
from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu


def comm_world1():
    ident = (C.c_uint8 * _lib.COMM_ID_BYTES)()
    _lib.call("pqlg_comm_unique_id", ident)
    comm = C.c_void_p()
    _lib.call("pqlg_comm_init", 0, 1, ident, C.byref(comm))
    return comm


def fill(rp, n, seed):
    _lib.call("pqlg_replay_fill_synthetic", rp, n, seed, np.float32(0.970299), 200)


@pytest.mark.parametrize("D,A,H,nh,B,algo", [(17, 6, 64, 2, 256, _lib.ALGO_DDPG),
                                             (211, 20, 512, 3, 1024, _lib.ALGO_DDPG),
                                             (17, 6, 64, 2, 256, _lib.ALGO_SAC)])
def test_vlearner_dp_world1_bit_identical(D, A, H, nh, B, algo):
    import torch
    torch.cuda.set_device(0)
    comm = comm_world1()
    r, w = C.c_int(), C.c_int()
    _lib.call("pqlg_comm_rank", comm, C.byref(r), C.byref(w))
    assert (r.value, w.value) == (0, 1)
    cfg = _lib.default_config(algo=algo, batch_size=B, buffer_capacity=20000, hidden=H,
                              hidden_layers=nh, n_envs=8)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    plain, dp = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 7, None, C.byref(plain))
    _lib.call("pqlg_vlearner_create_dp", C.byref(cfg), C.byref(dims), 7, comm, None, C.byref(dp))
    mean = np.zeros(D)
    m2 = np.full(D, 1e6)
    for h in (plain, dp):
        rp = C.c_void_p()
        _lib.call("pqlg_vlearner_replay", h, C.byref(rp))
        fill(rp, 20000, 3)
        ns = _lib.NormStats(10 ** 6, ptr(mean), ptr(m2))
        _lib.call("pqlg_vlearner_adopt_norm", h, C.byref(ns))
    l_plain, l_dp = C.c_float(), C.c_float()
    for _ in range(3):
        _lib.call("pqlg_vlearner_update", plain, C.byref(l_plain))
        _lib.call("pqlg_vlearner_update", dp, C.byref(l_dp))
        assert l_plain.value == l_dp.value
    # graph replay path too
    _lib.call("pqlg_vlearner_update_n", plain, 4)
    _lib.call("pqlg_vlearner_update_n", dp, 4)
    P = param_count([D + A] + [H] * nh + [1])
    for which in range(4):
        a = np.zeros(P, np.float32)
        b = np.zeros(P, np.float32)
        _lib.call("pqlg_vlearner_get_params", plain, which, ptr(a))
        _lib.call("pqlg_vlearner_get_params", dp, which, ptr(b))
        assert np.array_equal(a, b), which
    kp, kd = C.c_int(), C.c_int()
    _lib.call("pqlg_vlearner_kernels_per_update", plain, C.byref(kp))
    _lib.call("pqlg_vlearner_kernels_per_update", dp, C.byref(kd))
    # one reduce + all-reduce bucket per layer (head + nh hidden layers) on
    # the communication branch; the norm pass replaces the single finalize
    assert kd.value == kp.value + nh + 1
    for h in (plain, dp):
        _lib.call("pqlg_vlearner_destroy", h)
    _lib.call("pqlg_comm_destroy", comm)


@pytest.mark.parametrize("algo", [_lib.ALGO_DDPG, _lib.ALGO_SAC])
def test_plearner_dp_world1_bit_identical(algo):
    import torch
    torch.cuda.set_device(0)
    D, A, H, nh, B = 31, 7, 64, 2, 512
    comm = comm_world1()
    cfg = _lib.default_config(algo=algo, batch_size=B, buffer_capacity=10000, hidden=H,
                              hidden_layers=nh, n_envs=8)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    plain, dp = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 5, None, C.byref(plain))
    _lib.call("pqlg_plearner_create_dp", C.byref(cfg), C.byref(dims), 5, comm, None, C.byref(dp))
    states = torch.randn(5000, D, device="cuda")
    for h in (plain, dp):
        _lib.call("pqlg_plearner_ingest", h, states.data_ptr(), D, 5000)
    la, lb = C.c_float(), C.c_float()
    for _ in range(3):
        _lib.call("pqlg_plearner_update", plain, C.byref(la))
        _lib.call("pqlg_plearner_update", dp, C.byref(lb))
        assert la.value == lb.value
    P = param_count([D] + [H] * nh + [2 * A if algo == _lib.ALGO_SAC else A])
    a = np.zeros(P, np.float32)
    b = np.zeros(P, np.float32)
    _lib.call("pqlg_plearner_get_params", plain, 0, ptr(a))
    _lib.call("pqlg_plearner_get_params", dp, 0, ptr(b))
    assert np.array_equal(a, b)
    if algo == _lib.ALGO_SAC:  # the alpha step sees the all-reduced mean log-prob
        xa, xb = C.c_float(), C.c_float()
        _lib.call("pqlg_plearner_log_alpha", plain, C.byref(xa))
        _lib.call("pqlg_plearner_log_alpha", dp, C.byref(xb))
        assert xa.value == xb.value != 0.0
    for h in (plain, dp):
        _lib.call("pqlg_plearner_destroy", h)
    _lib.call("pqlg_comm_destroy", comm)


def test_comm_allreduce_world1_identity():
    import torch
    torch.cuda.set_device(0)
    comm = comm_world1()
    x = torch.randn(1000, device="cuda")
    y = x.clone()
    _lib.call("pqlg_comm_allreduce_f32", comm, y.data_ptr(), 1000, None)
    torch.cuda.synchronize()
    assert torch.equal(x, y)
    _lib.call("pqlg_comm_destroy", comm)


def test_sharded_actor_world1_bit_identical():
    """pqlg_actor_create_sharded over a world-1 NCCL communicator (batch
    statistics -> all-gather -> rank-order merge) reproduces the plain actor
    bit for bit: observations, actions, normalizer stats; eager steps and
    graph replays (the all-gather is captured with the step)."""
    import torch
    torch.cuda.set_device(0)
    comm = comm_world1()
    N, D, A = 512, 37, 6
    cfg = _lib.default_config(n_envs=N, hidden=64, hidden_layers=2, seed=4, max_episode_len=9)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    plain, sh = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), None, C.byref(plain))
    _lib.call("pqlg_actor_create_sharded", C.byref(cfg), C.byref(dims), comm, None, C.byref(sh))
    sl = _lib.StepSlice()

    def state(h):
        obs = np.zeros((N, D), np.float32)
        act = np.zeros((N, A), np.float32)
        _lib.call("pqlg_actor_read", h, 0, ptr(obs))
        _lib.call("pqlg_actor_read", h, 1, ptr(act))
        cnt = C.c_int64()
        mean = np.zeros(D)
        m2 = np.zeros(D)
        _lib.call("pqlg_actor_norm", h, C.byref(cnt), ptr(mean), ptr(m2))
        return obs, act, cnt.value, mean, m2

    for _ in range(5):
        for h in (plain, sh):
            _lib.call("pqlg_actor_rollout_step", h, C.byref(sl))
        a, b = state(plain), state(sh)
        assert a[2] == b[2] == a[2]
        for x, y in zip(a[:2] + a[3:], b[:2] + b[3:]):
            assert np.array_equal(x, y)
    for h in (plain, sh):
        _lib.call("pqlg_actor_rollout_n", h, 6)
    a, b = state(plain), state(sh)
    assert a[2] == b[2]
    for x, y in zip(a[:2] + a[3:], b[:2] + b[3:]):
        assert np.array_equal(x, y)
    kp, ks = C.c_int(), C.c_int()
    _lib.call("pqlg_actor_kernels_per_step", plain, C.byref(kp))
    _lib.call("pqlg_actor_kernels_per_step", sh, C.byref(ks))
    assert ks.value == kp.value + 1  # the merge kernel
    for h in (plain, sh):
        _lib.call("pqlg_actor_destroy", h)
    _lib.call("pqlg_comm_destroy", comm)
