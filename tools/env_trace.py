"""Phase timeline of the TMA env step (GPU box): per-CTA %globaltimer stamps
from a library variant built with -DPQLG_ENV_TRACE
(tools/build_variant.sh envtrace -DPQLG_ENV_TRACE), run as
PQLG_LIB_VARIANT=envtrace python tools/env_trace.py"""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh, N = 211, 20, 512, 3, 16384
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
cfg = _lib.default_config(n_envs=N, hidden=H, hidden_layers=nh)
dims = _lib.TaskDims(D, A, -1.0, 1.0)
act = C.c_void_p()
_lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
tr = torch.zeros(148 * 32, dtype=torch.int64, device="cuda")
_lib.call("pqlg_actor_rollout_n", act, 5)
st.synchronize()
_lib.call("pqlg_env_trace_set", C.c_void_p(tr.data_ptr()))
for rep in range(3):
    tr.zero_()
    _lib.call("pqlg_actor_rollout_n", act, 1)
    st.synchronize()
t = tr.view(148, 32).cpu().numpy().astype(np.int64)
t0 = t[:, 0].min()
rel = lambda x: (x - t0) / 1e3
names = {0: "entry", 1: "prologue done", 2: "exit", 12: "step warps done", 13: "chains done",
         14: "writers done", 15: "producer done"}
for k in range(4):
    names[4 + k] = f"tile{k} full"
    names[8 + k] = f"tile{k} ready"
    names[20 + k] = f"tile{k} writer0 done"
    names[24 + k] = f"tile{k} chain done"
    names[16] = "tile0 writer0 ready"
    names[17], names[18], names[19] = "tile0 step0 actions", "tile0 step0 M a", "tile0 step0 s'"
    names[28 + k] = f"tile{k} stores issued"
for slot in sorted(names):
    v = t[:, slot]
    ok = v > 0
    if ok.any():
        print(f"{names[slot]:>22}: us after first entry p10/p50/p90/max "
              f"{np.percentile(rel(v[ok]), 10):6.2f} {np.median(rel(v[ok])):6.2f} "
              f"{np.percentile(rel(v[ok]), 90):6.2f} {rel(v[ok]).max():6.2f}  (n={ok.sum()})")
