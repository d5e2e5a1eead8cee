"""In-situ marginal cost of every step of the critic / policy update (GPU
box): the update graph is rebuilt with PQLG_SKIP_STEP=i (one process per i)
and replayed; cost(i) = t(full) - t(without step i).  Results of the skipped
runs are meaningless -- only their time is used.

  python tools/skip_probe.py critic|policy|actor [n_steps]
"""
import os
import subprocess
import sys

WHAT = sys.argv[1] if len(sys.argv) > 1 else "critic"
CHILD = r'''
import ctypes as C, sys, numpy as np, torch
sys.path.insert(0, "@ROOT@")
from paper_2307_12983_b200 import _lib
D, A, H, nh, B, N = 211, 20, 512, 3, 8192, 16384
st = torch.cuda.Stream(); sp = C.c_void_p(st.cuda_stream)
cfg = _lib.default_config(batch_size=B, buffer_capacity=1_000_000, hidden=H, hidden_layers=nh, n_envs=N)
dims = _lib.TaskDims(D, A, -1.0, 1.0)
h = C.c_void_p()
if "@WHAT@" == "critic":
    _lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(h))
    rp = C.c_void_p(); _lib.call("pqlg_vlearner_replay", h, C.byref(rp))
    _lib.call("pqlg_replay_fill_synthetic", rp, 1_000_000, 7, np.float32(0.970299), 200)
    fn = "pqlg_vlearner_update_n"; kfn = "pqlg_vlearner_kernels_per_update"
elif "@WHAT@" == "actor":
    _lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), sp, C.byref(h))
    fn = "pqlg_actor_rollout_n"; kfn = None
else:
    _lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, sp, C.byref(h))
    s = torch.randn(1_000_000, D, device="cuda")
    _lib.call("pqlg_plearner_ingest", h, s.data_ptr(), D, 1_000_000)
    fn = "pqlg_plearner_update_n"; kfn = "pqlg_plearner_kernels_per_update"
k = C.c_int(6)
if kfn: _lib.call(kfn, h, C.byref(k))
_lib.lib()[fn](h, 10); st.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
best = 1e9
for _ in range(3):
    e0.record(st); _lib.lib()[fn](h, 100); e1.record(st); e1.synchronize()
    best = min(best, e0.elapsed_time(e1) / 100 * 1e3)
print(k.value, best)
'''


def run(skip):
    env = dict(os.environ)
    if skip is not None:
        env["PQLG_SKIP_STEP"] = str(skip)
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = CHILD.replace("@ROOT@", root).replace("@WHAT@", WHAT)
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True,
                         timeout=300)
    k, t = out.stdout.strip().split()[-2:]
    return int(k), float(t)


k, full = run(None)
print(f"{WHAT}: {k} launches, full update {full:.1f} us")
n = int(sys.argv[2]) if len(sys.argv) > 2 else 24
for i in range(n):
    try:
        _, t = run(i)
    except Exception as ex:  # a skipped step may break a later one (e.g. NaN status)
        print(f"  step {i:2d}: failed ({type(ex).__name__})")
        continue
    print(f"  step {i:2d}: marginal {full - t:7.1f} us", flush=True)
