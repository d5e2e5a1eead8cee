"""Warm per-kernel device times of one update / step (GPU box).

Uses the library's launch profiler (pqlg_profile_begin/end: events around
every launch, eager path, no PDL overlap) after warm-up, and prints each
launch of the last profiled step in order with its time, plus the graph-
replayed time of the same step for comparison.

  python tools/kprof.py [critic|policy|actor|c51 ...]
"""
import ctypes as C
import os
import sys
from collections import defaultdict
from pathlib import Path

import numpy as np
import torch

os.environ["PQLG_EAGER"] = "1"  # update(): per-kernel launches the profiler can bracket
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, H, nh, B, N = 211, 20, 512, 3, 8192, 16384
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)


def prof(step, reps=3):
    for _ in range(3):
        step()
    st.synchronize()
    _lib.call("pqlg_profile_begin")
    for _ in range(reps):
        step()
    buf = C.create_string_buffer(1 << 20)
    _lib.call("pqlg_profile_end", buf, len(buf))
    lines = [ln.split("\t") for ln in buf.value.decode().strip().splitlines()]
    per = len(lines) // reps
    last = lines[-per:]
    agg = defaultdict(float)
    for name, ms in lines:
        agg[name] += float(ms) / reps
    tot = sum(float(ms) for _, ms in last)
    print(f"  {per} launches/step, sum of kernel times {tot * 1e3:.1f} us")
    for name, ms in last:
        short = name.split("(")[0].replace("void ", "")[:90]
        print(f"    {float(ms) * 1e3:8.2f} us  {short}")


def graph_time(fn, h, n=50):
    _lib.call(fn, h, 5)
    st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    _lib.call(fn, h, n)
    e1.record(st)
    e1.synchronize()
    return e0.elapsed_time(e1) / n * 1e3


what = sys.argv[1:] or ["critic", "policy", "actor", "c51"]
for w in what:
    if w in ("critic", "c51", "sac"):
        extra = {"c51": dict(algo=_lib.ALGO_C51, n_atoms=51),
                 "sac": dict(algo=_lib.ALGO_SAC)}.get(w, {})
        cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H,
                                  hidden_layers=nh, n_envs=N, **extra)
        dims = _lib.TaskDims(D, A, -1.0, 1.0)
        h = C.c_void_p()
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(h))
        rp = C.c_void_p()
        _lib.call("pqlg_vlearner_replay", h, C.byref(rp))
        _lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 7, np.float32(0.970299), 200)
        mean = np.zeros(D); m2 = np.full(D, 1e6)
        ns = _lib.NormStats(10 ** 6, mean.ctypes.data, m2.ctypes.data)
        _lib.call("pqlg_vlearner_adopt_norm", h, C.byref(ns))
        print(f"{w}: graph-replayed update {graph_time('pqlg_vlearner_update_n', h):.1f} us")
        prof(lambda: _lib.call("pqlg_vlearner_update", h, None))
        _lib.call("pqlg_vlearner_destroy", h)
    elif w in ("policy", "sac_policy"):
        extra = dict(algo=_lib.ALGO_SAC) if w == "sac_policy" else {}
        cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H,
                                  hidden_layers=nh, n_envs=N, **extra)
        dims = _lib.TaskDims(D, A, -1.0, 1.0)
        h = C.c_void_p()
        _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(h))
        states = torch.randn(1_000_000, D, device="cuda")
        _lib.call("pqlg_plearner_ingest", h, states.data_ptr(), D, 1_000_000)
        print(f"policy: graph-replayed update {graph_time('pqlg_plearner_update_n', h):.1f} us")
        prof(lambda: _lib.call("pqlg_plearner_update", h, None))
        _lib.call("pqlg_plearner_destroy", h)
    elif w in ("actor", "sac_actor"):
        extra = dict(algo=_lib.ALGO_SAC) if w == "sac_actor" else {}
        cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H,
                                  hidden_layers=nh, n_envs=N, **extra)
        dims = _lib.TaskDims(D, A, -1.0, 1.0)
        act, vl, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
        _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(act))
        _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(vl))
        _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(pl))
        s = _lib.StepSlice()

        def step():
            _lib.call("pqlg_actor_rollout_step", act, C.byref(s))
            _lib.call("pqlg_vlearner_ingest", vl, C.byref(s))
            _lib.call("pqlg_plearner_ingest", pl, s.obs, s.ld_obs, N)
        print(f"actor: graph-replayed step (no ingest) {graph_time('pqlg_actor_rollout_n', act):.1f} us")
        prof(step)
        for hh, fn in ((act, "pqlg_actor_destroy"), (vl, "pqlg_vlearner_destroy"),
                       (pl, "pqlg_plearner_destroy")):
            _lib.call(fn, hh)
