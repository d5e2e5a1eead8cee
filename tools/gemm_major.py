"""GEMM layout probe (GPU box): the tcgen05 TF32 GEMM (Linear epilogue, TMA
store) in all four operand-major combinations at the learners' shapes and at
long K (mainloop-dominated), hot (operands L2-resident, back to back) and
cold (a 256 MB L2 flush between launches), beside cuBLAS TF32.

  python tools/gemm_major.py            (PQLG_PAIR=0 for single-CTA tiles)
"""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

st = torch.cuda.Stream()
torch.backends.cuda.matmul.allow_tf32 = True
flush = torch.empty(64 << 20, device="cuda")  # 256 MB > L2


def timed(fn, it, cold):
    ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True))
          for _ in range(it)]
    with torch.cuda.stream(st):
        for i in range(it):
            if cold:
                flush.fill_(float(i))
            ev[i][0].record(st)
            fn()
            ev[i][1].record(st)
    st.synchronize()
    t = sorted(s.elapsed_time(e) for s, e in ev)
    return t[len(t) // 2]


for (M, N, K) in [(8192, 512, 512), (32768, 512, 512), (8192, 512, 4096), (16384, 512, 512)]:
    fl = 2 * M * N * K
    line = [f"M={M} N={N} K={K}:"]
    for a_mn in (0, 1):
        for b_mn in (0, 1):
            a = torch.randn((K, M) if a_mn else (M, K), device="cuda")
            b = torch.randn((K, N) if b_mn else (N, K), device="cuda")
            d = torch.empty(M, N, device="cuda")
            bias = torch.zeros(N, device="cuda")
            lda = M if a_mn else K
            ldb = N if b_mn else K

            def ours():
                _lib.call("pqlg_k_gemm_tf32", a.data_ptr(), b.data_ptr(), d.data_ptr(),
                          bias.data_ptr(), M, N, K, a_mn, b_mn, lda, ldb, N, 1, 1, 1,
                          C.c_void_p(st.cuda_stream))
            for _ in range(3):
                ours()
            hot = timed(ours, 30, False)
            cold = timed(ours, 30, True)
            line.append(f"A{'MN' if a_mn else 'K'}/B{'MN' if b_mn else 'K'} hot {fl/hot/1e9:.0f} "
                        f"cold {fl/cold/1e9:.0f}")
    a = torch.randn(M, K, device="cuda")
    b = torch.randn(K, N, device="cuda")
    with torch.cuda.stream(st):
        for _ in range(3):
            a @ b
    hot = timed(lambda: a @ b, 30, False)
    cold = timed(lambda: a @ b, 30, True)
    line.append(f"cuBLAS hot {fl/hot/1e9:.0f} cold {fl/cold/1e9:.0f} TF/s")
    print("  ".join(line), flush=True)
