"""Checksums of the actor, V-learner and P-learner state after a few eager
steps (GPU box): run once plainly and once under `compute-sanitizer --tool
racecheck` and diff the outputs (the tools must not change the results)."""
import ctypes as C, os, sys, numpy as np
os.environ["PQLG_EAGER"] = "1"
sys.path.insert(0, os.getcwd())
from paper_2307_12983_b200 import _lib
D, A, H, nh, B, N = 19, 5, 64, 2, 256, 128
cfg = _lib.default_config(batch_size=B, buffer_capacity=5000, hidden=H, hidden_layers=nh, n_envs=N, max_episode_len=7)
dims = _lib.TaskDims(D, A, -1.0, 1.0)
act, vl, pl = C.c_void_p(), C.c_void_p(), C.c_void_p()
_lib.call("pqlg_actor_create", C.byref(cfg), C.byref(dims), None, C.byref(act))
_lib.call("pqlg_vlearner_create", C.byref(cfg), C.byref(dims), 1, None, C.byref(vl))
s = _lib.StepSlice()
def h(x): return float(np.sum(x.astype(np.float64) * np.arange(1, x.size + 1).reshape(x.shape)))
for t in range(8):
    _lib.call("pqlg_actor_rollout_step", act, C.byref(s))
    o = np.zeros((N, D), np.float32); a = np.zeros((N, A), np.float32)
    _lib.call("pqlg_actor_read", act, 0, o.ctypes.data); _lib.call("pqlg_actor_read", act, 1, a.ctypes.data)
    _lib.call("pqlg_vlearner_ingest", vl, C.byref(s))
    print("step", t, h(o), h(a))
P = 0
n = C.c_int64(); _lib.call("pqlg_vlearner_param_count", vl, 0, C.byref(n))
loss = C.c_float(); _lib.call("pqlg_vlearner_update", vl, C.byref(loss))
X = np.zeros((B, D + A), np.float32); _lib.call("pqlg_vlearner_debug_read", vl, 4, X.ctypes.data)
y = np.zeros(B, np.float32); _lib.call("pqlg_vlearner_debug_read", vl, 0, y.ctypes.data)
q = np.zeros(n.value, np.float32); _lib.call("pqlg_vlearner_get_params", vl, 0, q.ctypes.data)
print("X", h(X), "y", h(y), "q1", h(q), "loss", loss.value)
pl = C.c_void_p()
_lib.call("pqlg_plearner_create", C.byref(cfg), C.byref(dims), 1, None, C.byref(pl))
rows = (np.arange(600 * D, dtype=np.float32).reshape(600, D) % 7.0 - 3.0) * 0.3
import torch
d = torch.from_numpy(rows).cuda()
_lib.call("pqlg_plearner_ingest", pl, d.data_ptr(), D, 600)
torch.cuda.synchronize()
for k in range(2):
    _lib.call("pqlg_plearner_update", pl, C.byref(loss))
    n2 = C.c_int64(); _lib.call("pqlg_plearner_param_count", pl, 0, C.byref(n2))
    pp = np.zeros(n2.value, np.float32); _lib.call("pqlg_plearner_get_params", pl, 0, pp.ctypes.data)
    print("P", k, loss.value, h(pp))
