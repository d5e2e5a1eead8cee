"""GEMM micro-benchmark (GPU box): our tcgen05 TF32 GEMM (forward layout,
Linear epilogue) vs cuBLAS TF32 at the learners' shapes and at long K."""
import ctypes as C
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
from paper_2307_12983_b200 import _lib  # noqa: E402

st = torch.cuda.Stream()
torch.backends.cuda.matmul.allow_tf32 = True
for (M, N, K) in [(8192, 512, 512), (16384, 512, 512), (8192, 512, 8192), (32768, 512, 512),
                  (8192, 256, 512), (8192, 512, 231), (16384, 1024, 1024)]:
    a = torch.randn(M, K, device="cuda"); b = torch.randn(K, N, device="cuda")
    d = torch.empty(M, N, device="cuda"); bias = torch.zeros(N, device="cuda")
    lda = (K + 3) // 4 * 4
    if lda != K:
        a = torch.zeros(M, lda, device="cuda")
    def ours(n):
        _lib.call("pqlg_k_gemm_tf32_repeat", a.data_ptr(), b.data_ptr(), d.data_ptr(),
                  bias.data_ptr(), M, N, K, lda, N, N, 1, n, C.c_void_p(st.cuda_stream))
    ours(3); st.synchronize()
    it = 50
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st); ours(it); e.record(st); e.synchronize()
    t_ours = s.elapsed_time(e) / it
    with torch.cuda.stream(st):
        aa = a[:, :K]
        for _ in range(3): aa @ b
        s.record(st)
        for _ in range(it): aa @ b
        e.record(st)
    e.synchronize()
    t_cub = s.elapsed_time(e) / it
    fl = 2 * M * N * K
    print(f"M={M} N={N} K={K}: ours {t_ours*1e3:.1f} us {fl/t_ours/1e9:.0f} TF/s | "
          f"cuBLAS {t_cub*1e3:.1f} us {fl/t_cub/1e9:.0f} TF/s", flush=True)
