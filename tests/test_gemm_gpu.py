"""tcgen05 TF32 GEMM vs an fp64 matmul of tf32-rounded operands.

Covers the three operand-major combinations the MLP layers use
(fwd: A K-major / B N-major; dgrad: K/K; wgrad: M-major / N-major, split-K)
plus the fourth for completeness, ragged edges (K=231, N=20/51, M not a
multiple of 128) and the TFLOAT32-typed tensor-map mode.
"""
import ctypes as C

import numpy as np
import pytest

from paper_2307_12983_b200 import _lib

pytestmark = pytest.mark.gpu


def tf32_trunc(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return (b & np.uint32(0xFFFFE000)).view(np.float32)


def tf32_rne(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32).astype(np.uint64)
    b = (b + 0xFFF + ((b >> 13) & 1)) & 0xFFFFE000
    return b.astype(np.uint32).view(np.float32)


def tf32_rna(x):
    b = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
    return ((b + np.uint32(0x1000)) & np.uint32(0xFFFFE000)).view(np.float32)


def run_gemm(a_log, b_log, a_mn, b_mn, splits=1, relu=0, bias=None, round_mode=0, pad=0):
    """a_log: logical A [M,K]; b_log: logical B [K,N]. Returns D [M,N] (numpy)."""
    import torch
    M, K = a_log.shape
    N = b_log.shape[1]
    # storage layouts
    a_st = a_log.T if a_mn else a_log            # [K,M] or [M,K]
    b_st = b_log if b_mn else b_log.T            # [K,N] or [N,K]
    lda = a_st.shape[1] + pad
    ldb = b_st.shape[1] + pad
    lda = (lda + 3) // 4 * 4
    ldb = (ldb + 3) // 4 * 4
    A = torch.zeros(a_st.shape[0], lda, dtype=torch.float32, device="cuda")
    A[:, : a_st.shape[1]] = torch.from_numpy(np.ascontiguousarray(a_st))
    B = torch.zeros(b_st.shape[0], ldb, dtype=torch.float32, device="cuda")
    B[:, : b_st.shape[1]] = torch.from_numpy(np.ascontiguousarray(b_st))
    ldd = (N + 3) // 4 * 4  # TMA-stored output rows need 16-byte strides
    D = torch.full((M, ldd), float("nan"), dtype=torch.float32, device="cuda")
    bias_t = torch.from_numpy(bias).cuda() if bias is not None else None
    _lib.call("pqlg_k_gemm_tf32", A.data_ptr(), B.data_ptr(), D.data_ptr(),
              bias_t.data_ptr() if bias_t is not None else None,
              M, N, K, a_mn, b_mn, lda, ldb, ldd, relu, splits, round_mode, None)
    torch.cuda.synchronize()
    return D.cpu().numpy()[:, :N]


def rel_err(D, a, b, rnd, bias=None, relu=0):
    R = rnd(a).astype(np.float64) @ rnd(b).astype(np.float64)
    if bias is not None:
        R = R + bias.astype(np.float64)
    if relu:
        R = np.maximum(R, 0)
    scale = np.abs(a).astype(np.float64) @ np.abs(b).astype(np.float64) + 1e-30
    return float(np.max(np.abs(D - R) / scale))


CASES = [
    # M, N, K, a_mn, b_mn, splits
    (256, 256, 256, 0, 0, 1),
    (256, 256, 256, 0, 1, 1),
    (256, 256, 256, 1, 0, 1),
    (256, 256, 256, 1, 1, 1),
    (300, 20, 40, 0, 1, 1),
    (300, 51, 72, 0, 0, 1),
    (1024, 512, 231, 0, 1, 1),      # critic layer 0 forward (K ragged)
    (1024, 512, 512, 0, 0, 1),      # dgrad
    (512, 512, 4096, 1, 1, 8),      # wgrad, split-K
    (231, 512, 1024, 1, 1, 4),      # wgrad of layer 0 (M ragged)
]


@pytest.mark.parametrize("M,N,K,a_mn,b_mn,splits", CASES)
def test_gemm_matches_rounded_fp64(M, N, K, a_mn, b_mn, splits):
    rng = np.random.default_rng(M * 7 + N * 3 + K + a_mn * 2 + b_mn)
    a = rng.standard_normal((M, K)).astype(np.float32)
    b = rng.standard_normal((K, N)).astype(np.float32)
    D = run_gemm(a, b, a_mn, b_mn, splits=splits)
    assert np.isfinite(D).all()
    e_tr = rel_err(D, a, b, tf32_trunc)
    e_rn = rel_err(D, a, b, tf32_rna)
    print(f"\nM={M} N={N} K={K} a_mn={a_mn} b_mn={b_mn} splits={splits}: "
          f"err_vs_trunc={e_tr:.3e} err_vs_rna={e_rn:.3e}")
    assert min(e_tr, e_rn) < 2e-5


def test_gemm_bias_relu_and_tf32_tma_mode():
    rng = np.random.default_rng(5)
    a = rng.standard_normal((384, 200)).astype(np.float32)
    b = rng.standard_normal((200, 256)).astype(np.float32)
    bias = rng.standard_normal(256).astype(np.float32)
    for mode in (0, 1):
        D = run_gemm(a, b, 0, 1, relu=1, bias=bias, round_mode=mode)
        e_tr = rel_err(D, a, b, tf32_trunc, bias, 1)
        e_rn = rel_err(D, a, b, tf32_rna, bias, 1)
        e_re = rel_err(D, a, b, tf32_rne, bias, 1)
        print(f"\nround_mode={mode}: err_vs_trunc={e_tr:.3e} err_vs_rna={e_rn:.3e} "
              f"err_vs_rne={e_re:.3e}")
        # plain fp32 maps: the tensor core truncates; TFLOAT32 maps: TMA
        # rounds to nearest-even on the way into shared memory
        assert (e_tr if mode == 0 else e_re) < 2e-5
