"""Probe: 3xTF32 GEMM error vs fp64 as a function of K (accumulation
behaviour of the tcgen05 fp32 accumulator), beside numpy's fp32 matmul."""
import sys
from pathlib import Path
import numpy as np
ROOT = Path(__file__).resolve().parents[1]
sys.path.insert(0, str(ROOT)); sys.path.insert(0, str(ROOT / "tests"))
from test_gemm_gpu import run_gemm

for K in (8, 32, 64, 256, 512, 2048, 8192):
    rng = np.random.default_rng(K)
    M, N = 256, 256
    for dist in ("normal", "positive"):
        a = rng.standard_normal((M, K)).astype(np.float32)
        b = rng.standard_normal((K, N)).astype(np.float32)
        if dist == "positive":
            a, b = np.abs(a), np.abs(b)
        R = a.astype(np.float64) @ b.astype(np.float64)
        scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64)
        out = {}
        for mode in (1, 2):
            D = run_gemm(a, b, 0, 1, round_mode=mode)
            err = (D - R) / scale
            out[mode] = (np.max(np.abs(err)), np.mean(err))
        f = ((a @ b).astype(np.float64) - R) / scale
        print(f"K={K:5d} {dist:8s} tf32 max={out[1][0]:.2e} mean={out[1][1]:+.2e} | "
              f"3x max={out[2][0]:.2e} mean={out[2][1]:+.2e} | np32 max={np.max(np.abs(f)):.2e} "
              f"mean={np.mean(f):+.2e}", flush=True)
