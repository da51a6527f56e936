# SPDX-License-Identifier: Apache-2.0
"""GPU training step (sort_train_step: forward + backward of the whole scoring path) against
the fp64 oracle backward (tests/test_oracle_backward.py pins that by finite differences).

The GPU forward is bf16 (the inference kernels), the backward bf16 tcgen05 GEMMs and attention
core with fp32 accumulation and gradients (the ranking head and tokenizer in fp32); the
oracle is fed the same bf16-rounded weights. The bar is self-calibrated, because these
gradients are intrinsically sensitive at bf16 resolution (ReLU / softmax decisions flip):
the oracle's own gradients move by `noise[n]` (relative L2, the larger of NOISE_SAMPLES
draws) when every trainable weight is perturbed by a relative N(0, 2^-8) -- one bf16 ulp,
the resolution the GPU forward computes its activations at. Each GPU gradient must be
within NOISE_FACTOR * noise[n] (floor GRAD_FLOOR) of the oracle's and point the same way
(cosine > COS_MIN, or above 1 - NOISE_FACTOR^2 (1 - the oracle's own noise cosine) for
gradients whose direction the perturbation already turns, e.g. a profile table with one
contributing row per request); dtokens likewise. Measured on B200: GPU error ~= 0.5-1.5x
noise."""
import numpy as np
import pytest

import oracle as O
from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200 import synth
from paper_2603_03988_b200.config import base_config, tiny_config

pytestmark = pytest.mark.gpu

NOISE_FACTOR = 3.0
NOISE_SAMPLES = 2
GRAD_FLOOR = 2e-2
COS_MIN = 0.99


def rel_l2(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-30))


def cosine(a, b):
    return float((a * b).sum() / max(np.linalg.norm(a) * np.linalg.norm(b), 1e-30))


def _oracle_grads(cfg, P, b, dz, names, B):
    om = O.OracleModel(cfg, P)
    ref = {n: np.zeros_like(P[n], dtype=np.float64) for n in names}
    dtok, logits = [], []
    for i in range(B):
        logits.append(om.forward(b, i)[1])
        g, dt = om.backward(b, i, dz[i].astype(np.float64), names)
        for n in names:
            ref[n] += g[n]
        dtok.append(dt)
    return ref, np.stack(dtok), np.stack(logits)


def _check_step(cfg, seed, B):
    P = synth.make_params(cfg, seed=seed)
    Pr = {k: synth.bf16_round(v).astype(np.float64) for k, v in P.items()}
    gm = R.SortModel(cfg, P, max_batch=B)
    b = synth.make_batch(cfg, B, seed=seed + 1)
    dz = np.random.default_rng(seed).normal(size=(B, cfg.n_cand, 3)).astype(np.float32)
    logits = gm.train_step(b, dz)
    names = [n for n in P if n != "tok.item_table"]  # the item table is frozen
    ref, dtok_ref, zref = _oracle_grads(cfg, Pr, b, dz, names, B)
    assert np.max(np.abs(logits - zref)) < 5e-2
    rng = np.random.default_rng(seed + 2)
    noise = {n: 0.0 for n in names}
    noise_cos = {n: 1.0 for n in names}
    dtok_noise = 0.0
    for _ in range(NOISE_SAMPLES):
        Pn = {k: (v * (1 + rng.normal(size=v.shape) * 2.0 ** -8) if k != "tok.item_table" else v)
              for k, v in Pr.items()}
        refn, dtokn, _ = _oracle_grads(cfg, Pn, b, dz, names, B)
        for n in names:
            noise[n] = max(noise[n], rel_l2(refn[n], ref[n]))
            noise_cos[n] = min(noise_cos[n], cosine(refn[n], ref[n]))
        dtok_noise = max(dtok_noise, rel_l2(dtokn, dtok_ref))
    report = {}
    for n in names:
        g = gm.grad(n).astype(np.float64)
        err = rel_l2(g, ref[n])
        cos = cosine(g, ref[n])
        # the direction bar is calibrated like the magnitude bar: a gradient with few
        # contributing rows (a profile table row per request) turns by bf16 noise alone
        # (1 - cos) grows with the square of the angle, so a NOISE_FACTOR x larger angle than
        # the perturbation's own is NOISE_FACTOR^2 x its (1 - cos))
        cos_min = min(COS_MIN, 1.0 - NOISE_FACTOR ** 2 * (1.0 - noise_cos[n]))
        report[n] = (err, noise[n], cos, cos_min)
    bad = {n: r for n, r in report.items()
           if r[0] > max(NOISE_FACTOR * r[1], GRAD_FLOOR) or r[2] < r[3]}
    assert not bad, bad
    dtok = gm.dtokens(B)
    assert rel_l2(dtok, dtok_ref) < max(NOISE_FACTOR * dtok_noise, GRAD_FLOOR)
    return report


def test_train_step_tiny_vs_oracle():
    _check_step(tiny_config(keep=[262, 128]), 7, 2)


def test_train_step_base_shape_vs_oracle():
    """SORT-base widths (d=256, 8 heads, m=640, W=256, F=128) with a shorter history so the
    fp64 dense oracle stays fast; pruning after layer 2 as in SORT-base."""
    cfg = base_config(n_hist=300, n_cand=16, n_items=20000)
    cfg.keep = [cfg.prefix_len, cfg.prefix_len, 128, 128]
    _check_step(cfg, 11, 2)


def test_train_step_is_deterministic_in_loss_scale():
    """Gradients are linear in dL/dlogits: doubling dz doubles every gradient."""
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=5)
    gm = R.SortModel(cfg, P, max_batch=1)
    b = synth.make_batch(cfg, 1, seed=6)
    dz = np.random.default_rng(1).normal(size=(1, cfg.n_cand, 3)).astype(np.float32)
    gm.train_step(b, dz)
    g1 = gm.grads_flat()
    gm.train_step(b, 2 * dz)
    g2 = gm.grads_flat()
    assert rel_l2(g2, 2 * g1) < 1e-3


def test_bce_adamw_step_and_weight_repack():
    """Full optimizer step on the device: ranking loss (vs the numpy restatement of
    SPEC.md:381-389), AdamW on the fp32 masters (vs numpy adamw), then the
    bf16 inference weights rebuilt on the device must equal those a fresh handle builds on the
    host from the updated parameters: the next forward is bit-identical."""
    cfg = tiny_config(keep=[262, 128])
    P = synth.make_params(cfg, seed=9)
    gm = R.SortModel(cfg, P, max_batch=2)
    b = synth.make_batch(cfg, 2, seed=10)
    labels = (np.random.default_rng(3).random((2, cfg.n_cand, 3)) < 0.3).astype(np.float32)
    # the training forward keeps Q unscaled (the backward recomputes S from it); the inference
    # forward's pre-scaled Q (attn_prescale) rounds differently in bf16, so the loss reference
    # comes from an inference forward with the same unscaled Q
    gm.set_option("attn_prescale", 0)
    _, z0 = gm.forward_logits(b)
    gm.set_option("attn_prescale", 1)
    loss = gm.train_step_bce(b, labels)
    ref_loss, _ = O.bce_loss(z0, labels)
    assert abs(loss - ref_loss) < 1e-4 * max(1.0, abs(ref_loss))
    names = [n for n in P if n != "tok.item_table"]
    before = {n: gm.get_param(n).astype(np.float64) for n in names}
    grads = {n: gm.grad(n).astype(np.float64) for n in names}
    gm.adamw_step(lr=1e-2)
    for n in names:
        exp, _, _ = O.adamw(before[n], grads[n], 0.0, 0.0, 1, lr=1e-2)
        got = gm.get_param(n)
        assert np.allclose(got, exp, rtol=1e-5, atol=1e-6), n
    moved = sum(float(np.abs(gm.get_param(n) - before[n]).max()) for n in names)
    assert moved > 0
    P2 = {n: gm.get_param(n) for n in names}
    P2["tok.item_table"] = P["tok.item_table"]
    fresh = R.SortModel(cfg, P2, max_batch=2)
    p_dev = gm.forward(b)
    p_host = fresh.forward(b)
    assert np.array_equal(p_dev, p_host)


@pytest.mark.parametrize("mk", ["tiny", "base_shape"])
def test_attention_backward_variants_agree(mk):
    """The tcgen05 attention backward (k_attn_bwd_tc: dK/dV and dQ passes, default), the
    mma.sync kernel (attn_bwd_tc = 0) and the fp32 SIMT kernels (attn_bwd_tc = attn_bwd_mma = 0)
    on the same saved activations: every gradient within bf16 resolution. The tcgen05 passes
    use no atomics: the weight-matrix gradients of two runs are bit-identical."""
    if mk == "tiny":
        cfg = tiny_config(keep=[262, 128])
        B = 2
    else:
        cfg = base_config(n_hist=300, n_cand=16, n_items=20000)
        cfg.keep = [cfg.prefix_len, cfg.prefix_len, 128, 128]
        B = 4
    P = synth.make_params(cfg, seed=12)
    gm = R.SortModel(cfg, P, max_batch=B)
    b = synth.make_batch(cfg, B, seed=13)
    dz = np.random.default_rng(4).normal(size=(B, cfg.n_cand, 3)).astype(np.float32)
    gm.train_step(b, dz)
    g_tc = gm.grads_flat()
    det = [n for n in P if n.split(".")[-1] in ("wq", "wk", "wv", "wo", "wg", "w_gate", "w_up", "w_down")]
    g_det = {n: gm.grad(n) for n in det}
    gm.train_step(b, dz)
    # every weight-matrix gradient (GEMMs over the attention-core adjoints) is bit-identical
    # across runs; gain / bias / feature-table sums use float atomics across CTAs
    for n in det:
        assert np.array_equal(gm.grad(n), g_det[n]), n
    try:
        gm.set_option("attn_bwd_tc", 0)
        gm.train_step(b, dz)
        g_mma = gm.grads_flat()
        gm.set_option("attn_bwd_mma", 0)
        gm.train_step(b, dz)
        g_simt = gm.grads_flat()
    finally:
        gm.set_option("attn_bwd_tc", 1)
        gm.set_option("attn_bwd_mma", 1)
    assert rel_l2(g_mma, g_simt) < 1e-2
    assert rel_l2(g_tc, g_simt) < 1e-2
