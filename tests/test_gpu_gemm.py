# SPDX-License-Identifier: Apache-2.0
"""The streaming tcgen05 GEMM (csrc/gemm_stream.cuh; SORT-large projections, attention.cpp:93-95,
125,131 and the SwishGLU FFN SPEC.md:291-299) against a float64 product of the same
bf16-rounded operands: tails in M, K not a multiple of 64, several n-tiles."""
import numpy as np
import pytest

from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200 import synth

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("M,N,K", [(128, 256, 64), (1, 32, 8), (300, 1024, 1024), (1000, 2080, 56), (5000, 64, 2560)])
def test_stream_gemm_vs_fp64(M, N, K):
    rng = np.random.default_rng(M + N + K)
    A = synth.bf16_round(rng.normal(size=(M, K)).astype(np.float32))
    B = synth.bf16_round(rng.normal(size=(N, K)).astype(np.float32))
    C = R.op_gemm(A, B)
    ref = A.astype(np.float64) @ B.astype(np.float64).T
    err = np.max(np.abs(C - ref)) / max(1.0, np.max(np.abs(ref)))
    assert err < 1e-5, err
