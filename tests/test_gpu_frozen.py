# SPDX-License-Identifier: Apache-2.0
"""Parameter::frozen (params.hpp:15-25) and transfer_item_table (tokenizer.cpp:376-383;
SPEC.md:148, 399-406) on the device:
  * a frozen parameter gets zero gradient and its bytes do not change across optimizer steps;
  * the item table starts frozen; unfrozen, its gradient matches the oracle's
    Tokenizer::backward item rows (tokenizer.cpp:315-317, 346-352) and AdamW moves it;
  * transfer_item_table copies the table between handles and sets the flag.
Tolerance: the item-table gradient is a sum of bf16-backward row gradients, checked like the
other tokenizer gradients of test_gpu_train.py: rel-L2 <= ITEM_REL and cosine >= ITEM_COS
against the fp64 oracle on the same bf16-rounded weights."""
import numpy as np
import pytest

import oracle as O
from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200 import synth
from paper_2603_03988_b200.config import ConfigError, tiny_config

pytestmark = pytest.mark.gpu

ITEM_REL = 5e-2
ITEM_COS = 0.998


def _step(gm, b, B, cfg, seed=0):
    labels = (np.random.default_rng(seed).random((B, cfg.n_cand, 3)) < 0.3).astype(np.float32)
    gm.train_step_bce(b, labels)
    gm.adamw_step(1e-2)


def test_frozen_dense_parameter_is_byte_identical_after_steps():
    cfg = tiny_config(keep=[262, 128])
    P = synth.make_params(cfg, seed=21)
    B = 2
    gm = R.SortModel(cfg, P, max_batch=B)
    b = synth.make_batch(cfg, B, seed=22)
    gm.set_frozen("attn.0.wq")
    gm.set_frozen("tok.action_table")
    before = {n: gm.get_param(n).copy() for n in ("attn.0.wq", "tok.action_table", "attn.0.wk", "tok.item_table")}
    for k in range(3):
        _step(gm, b, B, cfg, k)
        assert not np.any(gm.get_grad("attn.0.wq")) and not np.any(gm.get_grad("tok.action_table"))
    assert np.array_equal(gm.get_param("attn.0.wq"), before["attn.0.wq"])
    assert np.array_equal(gm.get_param("tok.action_table"), before["tok.action_table"])
    assert np.array_equal(gm.get_param("tok.item_table"), before["tok.item_table"])  # frozen by default
    assert not np.array_equal(gm.get_param("attn.0.wk"), before["attn.0.wk"])
    with pytest.raises(ConfigError):
        gm.get_grad("tok.item_table")
    # unfreezing restores training of the dense parameter
    gm.set_frozen("attn.0.wq", False)
    _step(gm, b, B, cfg, 5)
    assert not np.array_equal(gm.get_param("attn.0.wq"), before["attn.0.wq"])
    with pytest.raises(ConfigError):
        gm.set_frozen("no.such.param")


def test_unfrozen_item_table_gradient_vs_oracle_and_drift():
    cfg = tiny_config(keep=[262, 128])
    P = synth.make_params(cfg, seed=31)
    Pr = {k: synth.bf16_round(v).astype(np.float64) for k, v in P.items()}
    B = 2
    gm = R.SortModel(cfg, P, max_batch=B)
    gm.set_frozen("tok.item_table", False)
    b = synth.make_batch(cfg, B, seed=32)
    dz = np.random.default_rng(33).normal(size=(B, cfg.n_cand, 3)).astype(np.float32)
    gm.train_step(b, dz)
    g = gm.get_grad("tok.item_table").astype(np.float64)
    om = O.OracleModel(cfg, Pr)
    om.set_item_trainable(True)
    ref = np.zeros_like(Pr["tok.item_table"])
    for i in range(B):
        gi, _ = om.backward(b, i, dz[i].astype(np.float64), ["tok.item_table"])
        ref += gi["tok.item_table"]
    touched = np.unique(np.concatenate([b["hist_item"].ravel(), b["cand_item"].ravel()]))
    untouched = np.setdiff1d(np.arange(cfg.n_items), touched)
    assert not np.any(g[untouched])
    rel = np.linalg.norm(g - ref) / np.linalg.norm(ref)
    cos = float((g * ref).sum() / (np.linalg.norm(g) * np.linalg.norm(ref)))
    assert rel < ITEM_REL and cos > ITEM_COS, (rel, cos)
    # AdamW moves the (unfrozen) table (freeze=false -> the table drifts)
    t0 = gm.get_param("tok.item_table").copy()
    gm.adamw_step(1e-2)
    assert np.linalg.norm(gm.get_param("tok.item_table") - t0) > 0


def test_transfer_item_table_sets_freeze_flag():
    cfg = tiny_config(keep=[262, 128])
    src = R.SortModel(cfg, synth.make_params(cfg, seed=41), max_batch=2)
    dst = R.SortModel(cfg, synth.make_params(cfg, seed=42), max_batch=2)
    b = synth.make_batch(cfg, 2, seed=43)
    dst.transfer_item_table(src, freeze=True)
    t = src.get_param("tok.item_table")
    assert np.array_equal(dst.get_param("tok.item_table"), t)
    # the forward now reads the transferred rows: same scores as a handle built with that table
    P2 = synth.make_params(cfg, seed=42)
    P2["tok.item_table"] = synth.make_params(cfg, seed=41)["tok.item_table"]
    ref = R.SortModel(cfg, P2, max_batch=2)
    assert np.array_equal(dst.forward(b), ref.forward(b))
    for k in range(2):  # freeze=True: unchanged bytes after optimizer steps
        _step(dst, b, 2, cfg, k)
    assert np.array_equal(dst.get_param("tok.item_table"), t)
    dst.transfer_item_table(src, freeze=False)
    _step(dst, b, 2, cfg, 9)
    assert not np.array_equal(dst.get_param("tok.item_table"), t)
