"""Profiling driver: c3 pql_sac critic and policy updates (eager launches)
for ncu (tools/ncu_sac.sh)."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np
import torch

os.environ["PQLG_EAGER"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh, B, N = 211, 20, 512, 3, 8192, 16384
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
cfg = _lib.default_config(algo=_lib.ALGO_SAC, batch_size=B, buffer_capacity=1_000_000, hidden=H,
                          hidden_layers=nh, n_envs=N)
dims = _lib.TaskDims(D, A, -1.0, 1.0)
vl, pl = C.c_void_p(), C.c_void_p()
_lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
_lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(pl))
rp = C.c_void_p()
_lib.call("pqlg_vlearner_replay", vl, C.byref(rp))
_lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 7, np.float32(0.970299), 200)
s = torch.randn(1_000_000, D, device="cuda")
_lib.call("pqlg_plearner_ingest", pl, s.data_ptr(), D, 1_000_000)
for _ in range(2):
    _lib.call("pqlg_vlearner_update", vl, None)
    _lib.call("pqlg_plearner_update", pl, None)
st.synchronize()
print("done")
