"""A/B of the critic / policy update time (graph replay, CUDA events) at c3;
run twice with PQLG_BRANCHES=0/1 to compare the forked-branch graph."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh, B = 211, 20, 512, 3, 8192
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
res = {}
for algo, name in ((_lib.ALGO_DDPG, "ddpg"), (_lib.ALGO_C51, "c51"), (_lib.ALGO_SAC, "sac")):
    cfg = _lib.default_config(algo=algo, batch_size=B, buffer_capacity=1_000_000, hidden=H,
                              hidden_layers=nh, n_envs=16384, precision=int(os.environ.get("PREC", "0")))
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    vl, pl = C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(pl))
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", vl, C.byref(rp))
    _lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 3, np.float32(0.970299), 200)
    states = torch.randn(1_000_000, D, device="cuda")
    _lib.call("pqlg_plearner_ingest", pl, states.data_ptr(), D, 1_000_000)
    for key, h, fn in (("critic", vl, "pqlg_vlearner_update_n"), ("policy", pl, "pqlg_plearner_update_n")):
        _lib.call(fn, h, 20)
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        best = 1e9
        for rep in range(3):
            e0.record(st)
            _lib.call(fn, h, 100)
            e1.record(st)
            e1.synchronize()
            best = min(best, e0.elapsed_time(e1) / 100 * 1e3)
        res[f"{name}_{key}_us"] = round(best, 1)
    loss = C.c_float()
    _lib.call("pqlg_vlearner_last_loss", vl, C.byref(loss))
    res[f"{name}_loss"] = loss.value
    _lib.call("pqlg_vlearner_destroy", vl)
    _lib.call("pqlg_plearner_destroy", pl)
print(os.environ.get("PQLG_BRANCHES", "1"), res)
