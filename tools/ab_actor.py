"""Actor step timing at c3 (16384 envs) and c5 (65536 envs): graph replay
(CUDA events) plus the in-graph per-kernel breakdown."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh = 211, 20, 512, 3
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
for N in (16384, 65536):
    for algo in (_lib.ALGO_DDPG, _lib.ALGO_SAC):
        cfg = _lib.default_config(n_envs=N, hidden=H, hidden_layers=nh, algo=algo)
        dims = _lib.TaskDims(D, A, -1.0, 1.0)
        act = C.c_void_p()
        _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
        _lib.call("pqlg_actor_rollout_n", act, 10)
        st.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        _lib.call("pqlg_actor_rollout_n", act, 60)
        e1.record(st)
        e1.synchronize()
        us = e0.elapsed_time(e1) / 60 * 1e3
        rows, g = _lib.time_graph("pqlg_actor_time_steps", act, 10)
        per = {}
        for name, t, shape in rows:
            k = name.split("(")[0][-40:] + (" " + shape.split(" splits")[0] if shape else "")
            per[k] = per.get(k, 0.0) + t / 3 * 1e3
        print(f"N={N} algo={algo}: step {us:.1f} us ({N / us:.1f} M transitions/s); instrumented "
              f"{g / 3 * 1e3:.1f} us: " + "; ".join(f"{k} {v:.1f}" for k, v in per.items()))
        _lib.call("pqlg_actor_destroy", act)
