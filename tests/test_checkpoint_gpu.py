"""Learner / actor checkpoints (pqlg_*_save / _load) in the reference's
format: a save -> load round trip restores every net and the normalizer
exactly, and the file is what fa::load_checkpoint reads."""
import ctypes as C

import numpy as np
import pytest

from oracle_lib import param_count, ptr
from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu
D, A, H, nh = 13, 5, 64, 2


def vl(seed):
    cfg = _lib.default_config(batch_size=64, buffer_capacity=2000, hidden=H, hidden_layers=nh,
                              n_envs=8)
    h = C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(_lib.TaskDims(D, A, -1.0, 1.0)),
              seed, None, C.byref(h))
    return h


def test_vlearner_save_load_round_trip(tmp_path):
    a, b = vl(1), vl(2)
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", a, C.byref(rp))
    _lib.call("pqlg_replay_fill_synthetic", rp, 2000, 5, np.float32(0.97), 50)
    mean = np.linspace(-1, 1, D)
    m2 = np.linspace(10, 20, D)
    _lib.call("pqlg_vlearner_adopt_norm", a, C.byref(_lib.NormStats(500, ptr(mean), ptr(m2))))
    _lib.call("pqlg_vlearner_update_n", a, 3)
    path = str(tmp_path / "v.ckpt").encode()
    _lib.call("pqlg_vlearner_save", a, path)
    _lib.call("pqlg_vlearner_load", b, path)
    for w in range(5):
        n = param_count([D] + [H] * nh + [A]) if w == 4 else param_count([D + A] + [H] * nh + [1])
        x, y = np.zeros(n, np.float32), np.zeros(n, np.float32)
        _lib.call("pqlg_vlearner_get_params", a, w, ptr(x))
        _lib.call("pqlg_vlearner_get_params", b, w, ptr(y))
        assert np.array_equal(x, y), w
    # the file is the reference's format: fa::load_checkpoint reads it
    from oracle_lib import ref
    R = ref()
    if R is not None:
        npar, cnt, dim = C.c_size_t(), C.c_int64(), C.c_size_t()
        assert R.ref_checkpoint_load(path, None, C.byref(npar), C.byref(cnt), None, None,
                                     C.byref(dim)) == 5
        assert cnt.value == 500 and dim.value == D
    for h in (a, b):
        _lib.call("pqlg_vlearner_destroy", h)


def test_actor_save_load_round_trip(tmp_path):
    cfg = _lib.default_config(n_envs=256, hidden=H, hidden_layers=nh)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    a, b = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), None, C.byref(a))
    cfg2 = _lib.default_config(n_envs=256, hidden=H, hidden_layers=nh, seed=7)
    _lib.call("pqlg_actor_create", C.byref(cfg2), C.byref(dims), None, C.byref(b))
    _lib.call("pqlg_actor_rollout_n", a, 5)
    path = str(tmp_path / "a.ckpt").encode()
    _lib.call("pqlg_actor_save", a, path)
    _lib.call("pqlg_actor_load", b, path)
    P = param_count([D] + [H] * nh + [A])
    x, y = np.zeros(P, np.float32), np.zeros(P, np.float32)
    _lib.call("pqlg_actor_read", a, 5, ptr(x))
    _lib.call("pqlg_actor_read", b, 5, ptr(y))
    assert np.array_equal(x, y)
    ca, cb = C.c_int64(), C.c_int64()
    ma, mb, sa, sb = (np.zeros(D) for _ in range(4))
    _lib.call("pqlg_actor_norm", a, C.byref(ca), ptr(ma), ptr(sa))
    _lib.call("pqlg_actor_norm", b, C.byref(cb), ptr(mb), ptr(sb))
    assert ca.value == cb.value == 5 * 256
    assert np.array_equal(ma, mb) and np.array_equal(sa, sb)
    for h in (a, b):
        _lib.call("pqlg_actor_destroy", h)


def test_plearner_save_load_round_trip(tmp_path):
    import torch
    cfg = _lib.default_config(batch_size=64, buffer_capacity=2000, hidden=H, hidden_layers=nh)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    a, b = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, None, C.byref(a))
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 2, None, C.byref(b))
    s = torch.randn(500, D, device="cuda")
    _lib.call("pqlg_plearner_ingest", a, s.data_ptr(), D, 500)
    _lib.call("pqlg_plearner_update_n", a, 2)
    path = str(tmp_path / "p.ckpt").encode()
    _lib.call("pqlg_plearner_save", a, path)
    _lib.call("pqlg_plearner_load", b, path)
    for w in range(3):
        n = param_count([D] + [H] * nh + [A]) if w == 0 else param_count([D + A] + [H] * nh + [1])
        x, y = np.zeros(n, np.float32), np.zeros(n, np.float32)
        _lib.call("pqlg_plearner_get_params", a, w, ptr(x))
        _lib.call("pqlg_plearner_get_params", b, w, ptr(y))
        assert np.array_equal(x, y), w
    # a shape mismatch is rejected
    cfg3 = _lib.default_config(batch_size=64, buffer_capacity=2000, hidden=32, hidden_layers=nh)
    c = C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg3), C.byref(dims), 1, None, C.byref(c))
    with pytest.raises(ValueError):
        _lib.call("pqlg_plearner_load", c, path)
    for h in (a, b, c):
        _lib.call("pqlg_plearner_destroy", h)


def test_sac_learners_and_actor_round_trip(tmp_path):
    """pql_sac cores checkpoint their GaussianPolicy nets (2 x act_dim
    outputs) in the same format; log alpha is not part of the reference's
    checkpoint (checkpoint.hpp:11-21) and is left untouched."""
    cfg = _lib.default_config(algo=_lib.ALGO_SAC, batch_size=64, buffer_capacity=2000, hidden=H,
                              hidden_layers=nh, n_envs=16)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    Pp = param_count([D] + [H] * nh + [2 * A])
    pa, pb = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 3, None, C.byref(pa))
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 4, None, C.byref(pb))
    import torch
    s = torch.randn(500, D, device="cuda")
    _lib.call("pqlg_plearner_ingest", pa, s.data_ptr(), D, 500)
    _lib.call("pqlg_plearner_update_n", pa, 2)
    path = str(tmp_path / "p.ckpt").encode()
    _lib.call("pqlg_plearner_save", pa, path)
    _lib.call("pqlg_plearner_load", pb, path)
    x, y = np.zeros(Pp, np.float32), np.zeros(Pp, np.float32)
    _lib.call("pqlg_plearner_get_params", pa, 0, ptr(x))
    _lib.call("pqlg_plearner_get_params", pb, 0, ptr(y))
    assert np.array_equal(x, y)
    la, lb = C.c_float(), C.c_float()
    _lib.call("pqlg_plearner_log_alpha", pa, C.byref(la))
    _lib.call("pqlg_plearner_log_alpha", pb, C.byref(lb))
    assert la.value != 0.0 and lb.value == 0.0
    # the actor loads the policy net of the P-learner's file
    act = C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), None, C.byref(act))
    _lib.call("pqlg_actor_load", act, path)
    z = np.zeros(Pp, np.float32)
    _lib.call("pqlg_actor_read", act, 5, ptr(z))
    assert np.array_equal(z, x)
    for h, fn in ((pa, "pqlg_plearner_destroy"), (pb, "pqlg_plearner_destroy"),
                  (act, "pqlg_actor_destroy")):
        _lib.call(fn, h)
