"""Profiling driver (run under ncu on the GPU box): a few hidden-layer GEMMs
via the repeat hook, then a handful of c3 critic updates."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "both"
st = torch.cuda.Stream()
if which == "gemm4":  # the update's dominant launch: 4-group hidden layer
    M, N, K = 8192, 512, 512
    a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
    d = torch.empty(M, N, device="cuda"); bias = torch.zeros(N, device="cuda")
    _lib.call("pqlg_k_gemm_tf32_repeat_groups", a.data_ptr(), b.data_ptr(), d.data_ptr(),
              bias.data_ptr(), M, N, K, K, N, N, 4, 3, C.c_void_p(st.cuda_stream))
    st.synchronize()
if which in ("gemm", "both"):
    M, N, K = 8192, 512, 512
    a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
    d = torch.empty(M, N, device="cuda"); bias = torch.zeros(N, device="cuda")
    _lib.call("pqlg_k_gemm_tf32_repeat", a.data_ptr(), b.data_ptr(), d.data_ptr(),
              bias.data_ptr(), M, N, K, K, N, N, 1, 3, C.c_void_p(st.cuda_stream))
    st.synchronize()
if which in ("critic", "both", "c51"):
    D, A, H, nh, B, cap = 211, 20, 512, 3, 8192, 200_000
    extra = dict(algo=_lib.ALGO_C51, n_atoms=51) if which == "c51" else {}
    cfg = _lib.default_config(batch_size=B, buffer_capacity=cap, hidden=H, hidden_layers=nh,
                              n_envs=16384, **extra)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    h = C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, C.c_void_p(st.cuda_stream),
              C.byref(h))
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", h, C.byref(rp))
    _lib.call("pqlg_replay_fill_synthetic", rp, cap, 7, np.float32(0.970299), 200)
    loss = C.c_float()
    for _ in range(3):
        _lib.call("pqlg_vlearner_update", h, C.byref(loss))
    st.synchronize()
if which == "policy":
    D, A, H, nh, B = 211, 20, 512, 3, 8192
    cfg = _lib.default_config(batch_size=B, buffer_capacity=200_000, hidden=H, hidden_layers=nh,
                              n_envs=16384)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    pl = C.c_void_p()
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, C.c_void_p(st.cuda_stream),
              C.byref(pl))
    states = torch.randn(200_000, D, device="cuda")
    _lib.call("pqlg_plearner_ingest", pl, states.data_ptr(), D, 200_000)
    loss = C.c_float()
    for _ in range(3):
        _lib.call("pqlg_plearner_update", pl, C.byref(loss))
    st.synchronize()
print("done")
