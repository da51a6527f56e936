# SPDX-License-Identifier: Apache-2.0
"""The pre-training oracle (tokenize_click_sequence, tokenizer.cpp:240-284)
against the spec's examples and independent numpy restatements: [BOS; clicks] layout, gap
time buckets (first click at INT64_MAX / 4), vocab = 2 uniform logits -> CE = ln 2, tied
logits (target = h . item_table[click]), causality (a later click never moves an earlier
position's log-sum-exp)."""
import numpy as np

import oracle as O
from paper_2603_03988_b200.config import pretrain_config
from paper_2603_03988_b200.synth import make_batch, make_params


def tiny_pre(**kw):
    c = dict(model_dim=64, heads=4, layers=2, ffn_dim=160, n_hist=24, batch=2, n_items=300)
    c.update(kw)
    return pretrain_config(**c)


def _bucket(delta, nb):
    d = max(int(delta), 0)
    return min((d + 1).bit_length() - 1, nb - 1)


def test_tokenize_clicks_layout_and_gap_buckets():
    cfg = tiny_pre()
    P = make_params(cfg, seed=1)
    batch = make_batch(cfg, 2, seed=2)
    om = O.OracleModel(cfg, P)
    tok, ht = om.tokenize_clicks(batch, 1)
    ts = batch["hist_ts"][1]
    expect = [cfg.n_time_buckets - 1] + [_bucket(ts[i] - ts[i - 1], cfg.n_time_buckets) for i in range(1, cfg.n_hist)]
    assert ht.tolist() == expect
    np.testing.assert_array_equal(tok[0], P["tok.special"][0])
    # history projection restated in numpy
    cat = np.concatenate([P["tok.item_table"][batch["hist_item"][1]], P["tok.action_table"][batch["hist_action"][1]],
                          P["tok.scene_table"][batch["hist_scene"][1]], P["tok.time_table"][ht]], axis=1)
    y = cat.astype(np.float64) @ P["tok.w_hist"] + P["tok.b_hist"]
    y = y / np.sqrt(np.mean(y * y, axis=1, keepdims=True) + 1e-6) * P["tok.g_hist"]
    np.testing.assert_allclose(tok[1:], y, rtol=1e-12, atol=1e-12)


def test_vocab2_uniform_logits_ce_is_ln2():
    cfg = tiny_pre(n_items=2)
    P = make_params(cfg, seed=3)
    P["tok.item_table"][1] = P["tok.item_table"][0]  # identical rows -> uniform logits
    batch = make_batch(cfg, 1, seed=4)
    lse, tgt, _ = O.OracleModel(cfg, P).pretrain_forward(batch, 0)
    np.testing.assert_allclose(lse - tgt, np.log(2.0), rtol=1e-12)


def test_tied_logits_and_causality():
    cfg = tiny_pre()
    P = make_params(cfg, seed=5)
    batch = make_batch(cfg, 1, seed=6)
    om = O.OracleModel(cfg, P)
    lse, tgt, h = om.pretrain_forward(batch, 0)
    E = P["tok.item_table"].astype(np.float64)
    z = h[:-1] @ E.T
    np.testing.assert_allclose(tgt, z[np.arange(cfg.n_hist), batch["hist_item"][0]], rtol=1e-12, atol=1e-12)
    m = z.max(1)
    np.testing.assert_allclose(lse, m + np.log(np.exp(z - m[:, None]).sum(1)), rtol=1e-12)
    j = 10
    b2 = {k: v.copy() for k, v in batch.items()}
    b2["hist_item"][0, j] = (b2["hist_item"][0, j] + 1) % cfg.n_items
    lse2, tgt2, _ = om.pretrain_forward(b2, 0)
    np.testing.assert_array_equal(lse2[:j + 1], lse[:j + 1])   # token j+1 = click j
    assert np.abs(lse2[j + 1:] - lse[j + 1:]).max() > 0
