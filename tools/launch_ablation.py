"""Critic update time (c3, B = 8192) under three launch regimes (GPU box):
graph replay with PDL (default), graph replay without PDL (PQLG_PDL=0), and
eager per-kernel launches (PQLG_EAGER=1, update() each step)."""
import ctypes as C
import os
import subprocess
import sys

CHILD = r'''
import ctypes as C, sys, time, numpy as np, torch
sys.path.insert(0, "@ROOT@")
from paper_2307_12983_b200 import _lib
D, A, H, nh, B, N = 211, 20, 512, 3, 8192, 16384
st = torch.cuda.Stream(); sp = C.c_void_p(st.cuda_stream)
cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H, hidden_layers=nh, n_envs=N)
h = C.c_void_p()
_lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(_lib.TaskDims(D, A, -1.0, 1.0)), 1, sp, C.byref(h))
rp = C.c_void_p(); _lib.call("pqlg_vlearner_replay", h, C.byref(rp))
_lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 7, np.float32(0.970299), 200)
mode = sys.argv[1]
n = 200
if mode == "eager":
    for _ in range(10): _lib.call("pqlg_vlearner_update", h, None)
    st.synchronize(); t0 = time.perf_counter()
    for _ in range(n): _lib.call("pqlg_vlearner_update", h, None)
    st.synchronize(); us = (time.perf_counter() - t0) / n * 1e6
else:
    _lib.call("pqlg_vlearner_update_n", h, 10); st.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); _lib.call("pqlg_vlearner_update_n", h, n); e1.record(st); e1.synchronize()
    us = e0.elapsed_time(e1) / n * 1e3
print(f"{us:.1f}")
'''
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for label, env, mode in (("graph + PDL", {}, "graph"), ("graph, no PDL", {"PQLG_PDL": "0"}, "graph"),
                         ("eager update() (host timer, synced per update)", {"PQLG_EAGER": "1"}, "eager")):
    e = dict(os.environ, **env)
    out = subprocess.run([sys.executable, "-c", CHILD.replace("@ROOT@", root), mode], env=e,
                         capture_output=True, text=True, timeout=600)
    print(f"{label:50s} {out.stdout.strip().splitlines()[-1] if out.stdout.strip() else out.stderr[-300:]} us/update")
