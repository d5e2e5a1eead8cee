"""Replay gather probe (GPU box): pqlg_replay_sample time vs ring size, and a
torch index_select gather of the same bytes for reference."""
import ctypes as C
import sys
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

D, A, B = 211, 20, 8192
st = torch.cuda.Stream()
sp = C.c_void_p(st.cuda_stream)
out = [torch.empty(B, 232, device="cuda"), torch.empty(B, 24, device="cuda"),
       torch.empty(B, 232, device="cuda"), torch.empty(B, device="cuda"),
       torch.empty(B, device="cuda")]
ob = _lib.NStepBatch(out[0].data_ptr(), out[1].data_ptr(), out[2].data_ptr(), out[3].data_ptr(),
                     out[4].data_ptr(), 232, 24)
for cap in (100_000, 1_000_000, 5_000_000):
    h = C.c_void_p()
    _lib.call("pqlg_replay_create", cap, D, A, sp, C.byref(h))
    _lib.call("pqlg_replay_fill_synthetic", h, cap, 3, np.float32(0.97), 200)
    rng = _lib.Rng(0, 12345, 0, None)
    for _ in range(3):
        _lib.call("pqlg_replay_sample", h, B, C.byref(rng), B, None, C.byref(ob))
    st.synchronize()
    _lib.call("pqlg_profile_begin")
    for _ in range(10):
        _lib.call("pqlg_replay_sample", h, B, C.byref(rng), B, None, C.byref(ob))
    buf = C.create_string_buffer(1 << 16)
    _lib.call("pqlg_profile_end", buf, len(buf))
    ts = [float(l.split("\t")[1]) * 1e3 for l in buf.value.decode().strip().splitlines()
          if "replay_sample" in l]
    print(f"cap {cap}: replay_sample_kernel median {np.median(ts):.1f} us (event-bracketed)",
          flush=True)
    _lib.call("pqlg_replay_destroy", h)
    # torch gather of the same rows from a same-size 2-array ring for comparison
    ring = torch.randn(cap, 212, device="cuda")
    idx = torch.randint(0, cap, (B,), device="cuda")
    with torch.cuda.stream(st):
        for _ in range(3):
            torch.index_select(ring, 0, idx)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(20):
            idx = torch.randint(0, cap, (B,), device="cuda")
            torch.index_select(ring, 0, idx)
            torch.index_select(ring, 0, idx)
        e1.record(st)
    e1.synchronize()
    print(f"cap {cap}: torch 2x index_select + randint {e0.elapsed_time(e1) / 20 * 1e3:.1f} us",
          flush=True)
    del ring
