# SPDX-License-Identifier: Apache-2.0
"""The tensor-core ranking head (misc.cuh k_head_wsplit / GsHead) multiplies the bf16 candidate
rows by g . W1 split into three bf16 pieces, hi = bf16(w), mid = bf16(w - hi),
lo = bf16(w - hi - mid). Its fp32 claim rests on hi + mid + lo == w exactly (then every
product x . piece is exact in the fp32 accumulator). This restates the device split in numpy
(round-to-nearest-even bf16, fp32 differences as on the device) and checks the identity over
the whole range a head weight can take (|w| >= 2^-100); below ~2^-110 the lo piece becomes a
bf16 subnormal (irrelevant for weights: the error is then below 2^-130 absolute)."""
import numpy as np

from paper_2603_03988_b200.synth import bf16_round


def split3(w):
    w = np.asarray(w, np.float32)
    hi = bf16_round(w)
    r1 = (w - hi).astype(np.float32)  # exact (Sterbenz)
    mid = bf16_round(r1)
    lo = bf16_round((r1 - mid).astype(np.float32))
    return hi, mid, lo


def test_three_bf16_pieces_reconstruct_fp32_exactly():
    rng = np.random.default_rng(0)
    mant = rng.standard_normal(1_000_000).astype(np.float32)
    scale = np.float32(2.0) ** rng.integers(-100, 100, mant.size).astype(np.float32)
    w = mant * scale
    w = w[np.abs(w) >= np.float32(2.0) ** -100]
    w = np.concatenate([w, np.array([1.0, -1.0, 1.0 / 3.0, 0.0, -0.0, 65504.0, 2.0 ** -100,
                                                 np.nextafter(np.float32(1), np.float32(2))], np.float32)])
    hi, mid, lo = split3(w)
    recon = hi.astype(np.float64) + mid.astype(np.float64) + lo.astype(np.float64)
    assert np.array_equal(recon, w.astype(np.float64))


def test_split_of_typical_head_weights_is_exact_and_pieces_shrink():
    rng = np.random.default_rng(1)
    g = (1.0 + 0.1 * rng.standard_normal(256)).astype(np.float32)
    w1 = (rng.standard_normal((256, 256)) / 16.0).astype(np.float32)
    wg = (g[:, None] * w1).astype(np.float32)  # g[k] * W1[k][n] in fp32, as k_head_wsplit
    hi, mid, lo = split3(wg)
    assert np.array_equal(hi.astype(np.float64) + mid + lo, wg.astype(np.float64))
    nz = hi != 0
    assert np.all(np.abs(mid[nz]) <= np.abs(hi[nz]) * 2.0 ** -8)
    assert np.all(np.abs(lo[nz]) <= np.abs(hi[nz]) * 2.0 ** -16)
