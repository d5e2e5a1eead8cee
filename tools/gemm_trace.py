"""Per-CTA phase timing of the forward-layer tcgen05 GEMM (GPU box).

Builds tools/_build/libgemmtrace.so (the library's GEMM with
-DPQLG_GEMM_TRACE), runs M x 512 x K with 1 or 2 groups, and prints the
median prologue->first-stage, mainloop and epilogue cycles plus the launch
span from %globaltimer."""
import ctypes as C
import subprocess
import sys
from pathlib import Path

import numpy as np
import torch

ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT))
from paper_2307_12983_b200 import build as b  # noqa: E402

import os
DEFS = os.environ.get("TRACE_DEFS", "").split()
out = ROOT / "tools" / "_build" / ("libgemmtrace%s.so" % "".join(d.replace("-D", "_").replace("=", "") for d in DEFS))
out.parent.mkdir(exist_ok=True)
src = ROOT / "tools" / "gemm_trace.cu"
subprocess.run([b.nvcc(), *b.ARCH, *b.NVCC_FLAGS, *DEFS, "-shared", str(src),
                str(ROOT / "paper_2307_12983_b200" / "csrc" / "common.cu"), "-o", str(out),
                "-lcuda"], check=True)
lib = C.CDLL(str(out))
st = torch.cuda.Stream()
import os
STORE = int(os.environ.get("TRACE_STORE", "1"))
KIND = int(os.environ.get("TRACE_KIND", "0"))
shapes = ([(8192, 512, 512, 1), (8192, 512, 512, 2), (8192, 512, 512, 4), (8192, 512, 232, 4),
           (16384, 512, 512, 1), (8192, 512, 4096, 1)] if KIND == 0
          else [(8192, 20, 512, 1), (16384, 20, 512, 1)])
if KIND == 2:
    shapes = [(8192, 20, 512, 1), (16384, 20, 512, 1)]
for (M, N, K, groups) in shapes:
    a = torch.randn(M, K, device="cuda")
    w = torch.randn(K, max(K, (N + 3) // 4 * 4), device="cuda")  # kind 2: hidden W [K x K]
    d = torch.randn(M, max(N, K), device="cuda"); bias = torch.zeros(max(N, K), device="cuda")
    bn = 256 if KIND == 0 else 32
    ctas = min((M // 128) * ((N + bn - 1) // bn) * groups, 148)
    tr = torch.zeros(ctas * 16, dtype=torch.int64, device="cuda")
    for it in range(3):
        tr.zero_()
        rc = lib.trace_gemm(C.c_void_p(a.data_ptr()), C.c_void_p(w.data_ptr()),
                            C.c_void_p(d.data_ptr()), C.c_void_p(bias.data_ptr()), M, N, K, groups,
                            C.c_void_p(tr.data_ptr()), 1, STORE, KIND, C.c_void_p(st.cuda_stream))
        assert rc == 0
        st.synchronize()
    t = tr.view(ctas, 16).cpu().numpy().astype(np.int64)
    span = (t[:, 6].max() - t[:, 0].min()) / 1e3
    med = lambda x: float(np.median(x))
    first_acc = t[:, 4] - t[:, 1]
    chunks = [t[:, 8 + c] - t[:, 4] for c in range(4)]
    rel = t[:, 12] - t[:, 4]
    lead = t[:, 14] > 0
    commit0 = t[lead, 14] - t[lead, 1]
    second = t[:, 13] > 0
    gap = t[second, 13] - t[second, 12]
    print(f"store={STORE} M={M} N={N} K={K} groups={groups} ctas={ctas}: span {span:.1f} us; "
          f"cycles p50: entry->first acc {med(first_acc):.0f} (leader: entry->tile0 commit issued "
          f"{med(commit0) if lead.any() else -1:.0f}); first-tile epilogue chunk ends "
          f"{[round(med(c)) for c in chunks]} release {med(rel):.0f}; "
          f"tile0 release->tile1 acc {med(gap) if second.any() else -1:.0f}; "
          f"epilogue end - entry {med(t[:, 5] - t[:, 1]):.0f}; SMs {len(set(t[:, 7]))}", flush=True)
