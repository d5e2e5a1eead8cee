"""Profiling driver for tools/ncu_all.sh: set-up kernels, then exactly one
c3 critic update / policy update / actor step + ingest issued eagerly (so
ncu sees the individual launches)."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

what = sys.argv[1]
D, A, H, nh, B, N = 211, 20, 512, 3, 8192, 16384
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H, hidden_layers=nh,
                          n_envs=N)
dims = _lib.TaskDims(D, A, -1.0, 1.0)
h = C.c_void_p()
if what == "critic":
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(h))
    rp = C.c_void_p()
    _lib.call("pqlg_vlearner_replay", h, C.byref(rp))  # 2 set-up launches (fill, advance)
    _lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 7, np.float32(0.970299), 200)
    _lib.call("pqlg_vlearner_update", h, None)
elif what == "policy":
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(h))
    s = torch.randn(1_000_000, D, device="cuda")  # torch launch(es) first
    _lib.call("pqlg_plearner_ingest", h, s.data_ptr(), D, 1_000_000)
    _lib.call("pqlg_plearner_update", h, None)
else:
    act, vl, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(pl))
    s = _lib.StepSlice()
    for _ in range(2):
        _lib.call("pqlg_actor_rollout_step", act, C.byref(s))
        _lib.call("pqlg_vlearner_ingest", vl, C.byref(s))
        _lib.call("pqlg_plearner_ingest", pl, s.obs, s.ld_obs, N)
st.synchronize()
print("done")
