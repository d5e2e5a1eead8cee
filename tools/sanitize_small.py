"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck):
one V, P update (DDPG, C51, SAC), a few actor steps + ingest, eager launches."""
import ctypes as C
import os
import sys
from pathlib import Path

import numpy as np

os.environ["PQLG_EAGER"] = "1"
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh, B, N = 19, 5, 64, 2, 256, 128
for algo in (_lib.ALGO_DDPG, _lib.ALGO_C51, _lib.ALGO_SAC):
    cfg = _lib.default_config(algo=algo, batch_size=B, buffer_capacity=5000, hidden=H,
                              hidden_layers=nh, n_envs=N, max_episode_len=7)
    dims = _lib.TaskDims(D, A, -1.0, 1.0)
    act, vl, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
    _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), None, C.byref(act))
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, None, C.byref(vl))
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, None, C.byref(pl))
    s = _lib.StepSlice()
    for _ in range(8):
        _lib.call("pqlg_actor_rollout_step", act, C.byref(s))
        ev = C.c_void_p()
        _lib.call("pqlg_actor_step_event", act, C.byref(ev))
        _lib.call("pqlg_vlearner_wait_event", vl, ev)
        _lib.call("pqlg_plearner_wait_event", pl, ev)
        _lib.call("pqlg_vlearner_ingest", vl, C.byref(s))
        _lib.call("pqlg_plearner_ingest", pl, s.obs, s.ld_obs, N)
    loss = C.c_float()
    _lib.call("pqlg_vlearner_update", vl, C.byref(loss))
    _lib.call("pqlg_plearner_update", pl, C.byref(loss))
    for h, fn in ((act, "pqlg_actor_destroy"), (vl, "pqlg_vlearner_destroy"),
                  (pl, "pqlg_plearner_destroy")):
        _lib.call(fn, h)
    print("algo", algo, "ok", loss.value)
