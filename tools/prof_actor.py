"""Profiling driver: a few config-3 actor steps (+ ingest) for ncu."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh, N = 211, 20, 512, 3, 16384
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
cfg = _lib.default_config(batch_size=8192, buffer_capacity=1_000_000, hidden=H, hidden_layers=nh,
                          n_envs=N)
dims = _lib.TaskDims(D, A, -1.0, 1.0)
act, vl, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
_lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
_lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
_lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(pl))
s = _lib.StepSlice()
for _ in range(3):
    _lib.call("pqlg_actor_rollout_step", act, C.byref(s))
    _lib.call("pqlg_vlearner_ingest", vl, C.byref(s))
    _lib.call("pqlg_plearner_ingest", pl, s.obs, s.ld_obs, N)
st.synchronize()
print("done")
