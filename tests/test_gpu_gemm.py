# SPDX-License-Identifier: Apache-2.0
"""The library's GEMM engines through sort_op_gemm against float64 products of the same rounded
operands: the streaming tcgen05 GEMM (csrc/gemm_stream.cuh: SORT-large projections,
attention.cpp:93-95,125,131; SwishGLU FFN SPEC.md:291-299; every training product) with
K-major and MN-major operands (the four transpose combinations), tails in M / K, several
n-tiles, split-K for long-K weight gradients; the TF32 variant (fp32 ranking head and
tokenizer) and the SIMT kernel for shapes TMA cannot tile (N = 3 logits)."""
import numpy as np
import pytest

from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200 import synth

pytestmark = pytest.mark.gpu


def _tf32(a):
    u = np.ascontiguousarray(a, np.float32).view(np.uint32)
    return ((u + 0x1000) & 0xFFFFE000).view(np.float32)  # round to 10 mantissa bits


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1, 32, 8), (300, 1024, 1024), (1000, 2080, 56), (5000, 64, 2560)])
@pytest.mark.parametrize("ta,tb", [(False, True), (False, False), (True, False), (True, True)])
def test_bf16_stream_gemm_vs_fp64(M, N, K, ta, tb):
    lda, ldb = (M if ta else K), (K if tb else N)
    if lda % 8 or ldb % 8:
        pytest.skip("TMA row pitch must be a multiple of 8 bf16")
    rng = np.random.default_rng(M + N + K + 2 * ta + tb)
    A = synth.bf16_round(rng.normal(size=(K, M) if ta else (M, K)).astype(np.float32))
    B = synth.bf16_round(rng.normal(size=(N, K) if tb else (K, N)).astype(np.float32))
    C = R.op_gemm(A, B, ta, tb)
    ref = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
    err = np.max(np.abs(C - ref)) / max(1.0, np.max(np.abs(ref)))
    assert err < 1e-5, err


@pytest.mark.parametrize("M,N,K,ta,tb", [(256, 256, 16384, True, False), (56, 256, 262144 // 4, True, False),
                                         (2048, 256, 256, False, False), (2048, 3, 256, False, False),
                                         (2048, 256, 3, False, True), (777, 56, 256, False, True)])
def test_tf32_and_simt_gemm_vs_fp64(M, N, K, ta, tb):
    rng = np.random.default_rng(M + N + K)
    A = _tf32(rng.normal(size=(K, M) if ta else (M, K)).astype(np.float32))
    B = _tf32(rng.normal(size=(N, K) if tb else (K, N)).astype(np.float32))
    C = R.op_gemm(A, B, ta, tb, tf32=True)
    ref = (A.T if ta else A).astype(np.float64) @ (B.T if tb else B).astype(np.float64)
    err = np.max(np.abs(C - ref)) / max(1.0, np.max(np.abs(ref)))
    assert err < 2e-3, err
