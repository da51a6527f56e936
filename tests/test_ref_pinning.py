# SPDX-License-Identifier: Apache-2.0
"""Pins the fp64 CPU oracle (oracle/sort_oracle.cpp) AND the product's host planner
(paper_2603_03988_b200/csrc/plan.cpp through the C ABI) to the REFERENCE's own code:
oracle/_ref/libref.so is /root/reference/proj/src/{mask,tokenizer,attention}.cpp compiled
unmodified against oracle/ref_shim/Eigen/Dense (oracle/Makefile). CPU only.

Integer artifacts (time buckets, masks, visible counts, schedules, retained rows, positions,
roles, candidate index) must be bit-identical; fp64 values within 1e-9 relative (the
shim's GEMM accumulation order is the only difference to Eigen's)."""
import numpy as np
import pytest

import oracle as O
import ref as RF
from paper_2603_03988_b200 import runtime as R
from paper_2603_03988_b200 import synth
from paper_2603_03988_b200.config import (ROLE_BOS, ROLE_CAND, ROLE_HIST, ROLE_PROF, ROLE_SEP, base_config,
                                          geometric_schedule, large_config, tiny_config)

pytestmark = pytest.mark.skipif(not RF.available(), reason="oracle/_ref/libref.so not built (needs /root/reference)")

TOL = 1e-9


def _close(a, b, tol=TOL):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    scale = max(1.0, float(np.max(np.abs(b))) if b.size else 1.0)
    return float(np.max(np.abs(a - b))) <= tol * scale if a.size else True


# ------------------------------------------------------------------ integer rules
def test_time_bucket_reference_oracle_product():
    vals = [0, 1, 2, 3, -1, -2**40, 2**62, 2**63 - 1, -(2**63)]
    for k in range(1, 63):
        vals += [2**k - 3, 2**k - 2, 2**k - 1, 2**k, 2**k + 1]
    vals += list(np.random.default_rng(0).integers(-2**40, 2**62, 2000))
    for nb in (2, 8, 32):
        for d in vals:
            d = int(d)
            r = RF.time_bucket(d, nb)
            assert O.time_bucket(d, nb) == r, (d, nb)
            if d > -(2**63):
                assert R.time_bucket(d, nb) == r, (d, nb)


def test_schedules_reference_oracle_product():
    for p in (1, 2, 7, 128, 262, 513, 1030, 4102):
        for dpt in (1, 2, 3, 4, 6, 12):
            for tgt in (1, 64, 128, 300):
                r = RF.geometric_schedule(p, dpt, tgt)
                assert O.geometric_schedule(p, dpt, tgt) == r
                assert R.geometric_schedule(p, dpt, tgt) == r
                assert geometric_schedule(p, dpt, tgt) == r
    assert RF.geometric_schedule(1030, 4, 128) == [1030, 514, 256, 128]
    assert RF.geometric_schedule(4102, 12, 128) == [4102, 2993, 2184, 1593, 1163, 848, 619, 452, 330, 240, 175, 128]
    assert RF.full_schedule(1030, 4) == [1030] * 4


def _random_structure(rng):
    n_hist = int(rng.integers(0, 80))
    n_prof = int(rng.integers(0, 4))
    n_cand = int(rng.integers(0, 9)) if rng.random() < 0.15 else int(rng.integers(1, 9))
    st = bool(rng.integers(0, 2))
    roles = ([ROLE_BOS] if st else []) + [ROLE_HIST] * n_hist + ([ROLE_SEP] if st else []) + \
        [ROLE_PROF] * n_prof + ([ROLE_SEP] if st else []) + [ROLE_CAND] * n_cand
    L = len(roles)
    pos = list(range(L - n_cand)) + [L - n_cand] * n_cand
    return roles, pos


def test_masks_and_retained_rows_reference_oracle_product():
    """build_mask / mask_visible_count / retained_rows (mask.cpp:14-154) over 400 random
    structures with chained pruning: the reference's dense mask equals the oracle's and the
    product planner's compact [lo, hi] + self form, bit for bit."""
    rng = np.random.default_rng(11)
    n_rows = 0
    for trial in range(400):
        roles, pos = _random_structure(rng)
        if not roles:
            continue
        W = int(rng.choice([-1, 1, 2, 5, 16, 64]))
        F = int(rng.integers(0, 40))
        ks = bool(rng.integers(0, 2))
        r, p = list(roles), list(pos)
        for _ in range(int(rng.integers(1, 4))):
            keep = int(rng.integers(1, len(r) + 1))
            qr = RF.retained_rows(r, keep, ks)
            assert O.retained_rows(r, keep, ks) == qr
            assert R.retained_rows(r, keep, ks) == qr
            vis, cnt = RF.build_mask(len(qr), r, p, W, F, qr)
            assert np.array_equal(O.build_mask(len(qr), r, p, W, F, qr), vis)
            assert cnt == int(vis.sum())
            lo, hi, se = R.mask_intervals(r, p, qr, W, F)
            dense = np.zeros_like(vis)
            c = np.arange(len(r))
            for i in range(len(qr)):
                dense[i] = (c >= lo[i]) & (c <= hi[i])
                if se[i] >= 0:
                    dense[i, se[i]] = 1
            assert np.array_equal(dense, vis)
            n_rows += len(qr)
            r = [r[i] for i in qr]
            p = [p[i] for i in qr]
    assert n_rows > 5000
    # suffix overload (query_rows omitted)
    roles, pos = _random_structure(np.random.default_rng(3))
    vis, _ = RF.build_mask(5, roles, pos, 8, 4)
    assert np.array_equal(O.build_mask(5, roles, pos, 8, 4), vis)


@pytest.mark.parametrize("mk", [tiny_config, base_config, large_config])
def test_config_visible_counts_reference(mk):
    """Per-layer visible counts of the bench configs from the reference's build_mask: the
    numbers the FLOP model (flops.py) and the attention tile lists are built from."""
    from paper_2603_03988_b200 import plan as PL
    cfg = mk()
    for lp in PL.layer_plans(cfg):
        if lp.l_q * lp.l_kv > 6_000_000:
            continue  # SORT-large's first layers: covered by the oracle/product test above
        vis, cnt = RF.build_mask(lp.l_q, lp.roles_kv.tolist(), lp.pos_kv.tolist(), cfg.local_window,
                                 cfg.full_suffix, lp.query_rows.tolist())
        assert cnt == lp.visible
        assert np.array_equal(vis, lp.dense())


def test_base_visible_counts_match_survey():
    from paper_2603_03988_b200 import plan as PL
    cfg = base_config()
    counts = []
    for lp in PL.layer_plans(cfg):
        _, cnt = RF.build_mask(lp.l_q, lp.roles_kv.tolist(), lp.pos_kv.tolist(), cfg.local_window,
                               cfg.full_suffix, lp.query_rows.tolist())
        counts.append(cnt)
    assert counts == [387968, 387968, 189696, 16512]


def test_prune_queries():
    x = np.random.default_rng(0).normal(size=(9, 5))
    for n in (1, 4, 9):
        assert np.array_equal(RF.prune_queries(x, n), O.prune_queries(x, n))
    with pytest.raises(RF.RefError):
        RF.prune_queries(x, 0)


# ------------------------------------------------------------------ numeric operators
def test_rmsnorm_and_rope_reference_oracle():
    rng = np.random.default_rng(1)
    for rows, cols in ((1, 4), (7, 32), (33, 256)):
        x = rng.normal(size=(rows, cols)) * rng.uniform(0.01, 10)
        g = 1 + 0.1 * rng.normal(size=cols)
        y, inv = RF.rmsnorm(x, g)
        assert _close(O.rmsnorm(x, g), y)
        dy = rng.normal(size=(rows, cols))
        dx, dg = RF.rmsnorm_backward(dy, x, g)
        # norm.hpp:32-45 against the oracle's restatement
        dg_o = np.zeros(cols)
        dx_o = np.zeros_like(x)
        lib = O.lib()
        xx, gg, dd = (np.ascontiguousarray(a, np.float64) for a in (x, g, dy))
        O._check(lib.oracle_rmsnorm_backward(O._p(dd, O.f64p), O._p(xx, O.f64p), O._p(inv, O.f64p), rows, cols,
                                             O._p(gg, O.f64p), O._p(dg_o, O.f64p), O._p(dx_o, O.f64p)))
        assert _close(dx_o, dx) and _close(dg_o, dg)
    x = rng.normal(size=(40, 32))
    pos = rng.integers(0, 5000, 40)
    for inv_ in (False, True):
        assert _close(O.rope(x, pos, 10000.0, inv_), RF.rope(x, pos, 10000.0, inv_))
    assert _close(RF.rope(RF.rope(x, pos), pos, inverse=True), x, 1e-12)


@pytest.mark.parametrize("dtype,tol", [(np.float64, 1e-10), (np.float32, 2e-5)])
def test_block_attention_reference_oracle(dtype, tol):
    """dense_masked_attention / blockwise_masked_attention (block_attention.hpp): outputs and
    skipped / total block counts equal the oracle's on random structured masks."""
    rng = np.random.default_rng(5)
    for trial in range(12):
        roles, pos = _random_structure(rng)
        if ROLE_CAND not in roles or len(roles) < 4:
            continue
        qr = RF.retained_rows(roles, int(rng.integers(1, len(roles))), False)
        vis, _ = RF.build_mask(len(qr), roles, pos, int(rng.choice([-1, 4, 16])), 8, qr)
        mask = np.where(vis == 1, 0.0, -np.inf)
        dk = int(rng.choice([4, 16, 32]))
        q = rng.normal(size=(len(qr), dk))
        k = rng.normal(size=(len(roles), dk))
        v = rng.normal(size=(len(roles), dk))
        ref_d = RF.dense_attention(q, k, v, mask, dtype)
        assert _close(O.dense_attention(q, k, v, mask, dtype), ref_d, tol)
        for blk in (1, 3, 16, 128):
            ro, rs, rt = RF.blockwise_attention(q, k, v, mask, blk, dtype)
            oo, os_, ot = O.blockwise_attention(q, k, v, mask, blk, dtype)
            assert (rs, rt) == (os_, ot)
            assert _close(oo, ro, tol) and _close(ro, ref_d, tol * 10)


def test_skip_fraction_spec_threshold():
    """SPEC.md:544 ("bench-attn"): at L=4096, W=256, 16x16 tiles the block-skip fraction of
    the local-window mask is >= 0.85. Computed with the reference's own blockwise operator on
    the reference's own mask (dense, l_q = l_kv = 4096 non-candidate history + 0 targets
    beyond F), so the figure is the reference's."""
    L = 4096
    roles = [ROLE_HIST] * L
    pos = list(range(L))
    vis, _ = RF.build_mask(L, roles, pos, 256, 128)
    mask = np.where(vis == 1, 0.0, -np.inf).astype(np.float32)
    z = np.zeros((L, 1), np.float32)
    _, sk, tot = RF.blockwise_attention(z, z, z, mask, 16, np.float32)
    frac = sk / tot
    assert frac >= 0.85, frac
    # the same census from the product planner's compact rows (the GPU uses 128x128 tiles)
    lo, hi, se = R.mask_intervals(roles, pos, list(range(L)), 256, 128)
    nb = L // 16
    tiles = np.zeros((nb, nb), bool)
    for i in range(L):
        tiles[i // 16, lo[i] // 16: hi[i] // 16 + 1] = True
    assert nb * nb - int(tiles.sum()) == sk


# ------------------------------------------------------------------ tokenizer / attention / model
@pytest.fixture(scope="module")
def tiny():
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=3)
    return cfg, P, O.OracleModel(cfg, P), RF.RefModel(cfg, P)


def test_tokenize_sample_reference_oracle(tiny):
    cfg, P, om, rm = tiny
    b = synth.make_batch(cfg, 3, seed=4)
    for i in range(3):
        t_o, t_r = om.tokenize(b, i), rm.tokenize(b, i)
        for k in ("position_ids", "roles", "candidate_index", "hist_time"):
            assert np.array_equal(t_o[k], t_r[k]), k
        assert _close(t_o["tokens"], t_r["tokens"])


def test_tokenizer_errors_match_reference(tiny):
    cfg, P, om, rm = tiny
    b = synth.make_batch(cfg, 1, seed=4)
    b["hist_item"][0, 3] = cfg.n_items  # OOV (tokenizer.cpp:14-19)
    with pytest.raises(RF.RefError) as e_r:
        rm.tokenize(b, 0)
    with pytest.raises(O.OracleError) as e_o:
        om.tokenize(b, 0)
    assert e_r.value.status == e_o.value.status == 1
    assert "outside vocabulary" in str(e_r.value) and "outside vocabulary" in str(e_o.value)


def test_tokenize_click_sequence_reference_oracle(tiny):
    cfg, P, om, rm = tiny
    b = synth.make_batch(cfg, 2, seed=9)
    for i in range(2):
        to, ho = om.tokenize_clicks(b, i)
        tr, hr = rm.tokenize_clicks(b, i)
        assert np.array_equal(ho, hr)
        assert _close(to, tr)


def test_tokenizer_backward_reference_oracle(tiny):
    """Tokenizer::backward (tokenizer.cpp:286-354) with the item table frozen (the SORT
    transfer+freeze setting the oracle and the GPU path use)."""
    cfg, P, om, rm = tiny
    rm.set_frozen("tok.item_table", True)
    b = synth.make_batch(cfg, 1, seed=6)
    L = cfg.seq_len
    dt = np.random.default_rng(2).normal(size=(L, cfg.model_dim))
    names = ["tok.special", "tok.w_hist", "tok.b_hist", "tok.g_hist", "tok.w_prof", "tok.b_prof", "tok.g_prof",
             "tok.w_cand", "tok.b_cand", "tok.g_cand", "tok.action_table", "tok.scene_table", "tok.time_table",
             "tok.profile_table.0", "tok.profile_table.1", "tok.profile_table.2"]
    g_r = rm.tokenizer_backward(b, 0, dt, names + ["tok.item_table"])
    g_o = om.tokenizer_backward(b, 0, dt, names)
    for n in names:
        assert g_o[n] is not None, n
        assert _close(g_o[n], g_r[n]), n
    assert not np.any(g_r["tok.item_table"])  # frozen (tokenizer.cpp:315, 346)
    rm.set_frozen("tok.item_table", False)


def _layer_inputs(cfg, om, b, layer):
    meta = om.layer_meta(b, 0)
    t = om.tokenize(b, 0)
    roles, pos = t["roles"].tolist(), t["position_ids"].tolist()
    for l in range(layer):
        qr = meta["query_rows"][l]
        roles = [roles[i] for i in qr]
        pos = [pos[i] for i in qr]
    qr = meta["query_rows"][layer]
    vis = O.build_mask(len(qr), roles, pos, cfg.local_window, cfg.full_suffix, qr)
    xn = np.random.default_rng(layer).normal(size=(len(roles), cfg.model_dim))
    return xn, qr, vis, pos


@pytest.mark.parametrize("keep", [None, "geo"])
def test_attention_layer_forward_backward_reference_oracle(keep):
    """AttentionLayer::forward (attention.cpp:71-132) and ::backward (:134-202, built with the
    force-included fixups for its undeclared names) against the oracle's restatement, per layer,
    on pruned layers too."""
    cfg = tiny_config(n_hist=60, n_cand=5)
    if keep == "geo":
        cfg.keep = geometric_schedule(cfg.prefix_len, cfg.layers, 20)
    P = synth.make_params(cfg, seed=8)
    om, rm = O.OracleModel(cfg, P), RF.RefModel(cfg, P)
    b = synth.make_batch(cfg, 1, seed=2)
    for layer in range(cfg.layers):
        xn, qr, vis, pos = _layer_inputs(cfg, om, b, layer)
        a_r = rm.attention(layer, xn, qr, vis, pos)
        assert _close(om.attention(layer, xn, qr, vis, pos), a_r)
        dout = np.random.default_rng(10 + layer).normal(size=a_r.shape)
        names = [f"attn.{layer}.{n}" for n in ("wq", "wk", "wv", "wo", "wg", "qk_gain_q", "qk_gain_k")]
        dx_r, g_r = rm.attention_backward(layer, xn, qr, vis, pos, dout, names)
        dx_o, g_o = om.attention_backward(layer, xn, qr, vis, pos, dout, names)
        assert _close(dx_o, dx_r, 1e-8)
        for n in names:
            assert _close(g_o[n], g_r[n], 1e-8), n


def test_reference_attention_backward_finite_differences():
    """The reference backward (with the fixups) is the adjoint of the reference forward:
    central differences of <dout, forward(xn)> along random directions."""
    cfg = tiny_config(n_hist=20, n_cand=3, layers=1)
    P = synth.make_params(cfg, seed=8)
    om, rm = O.OracleModel(cfg, P), RF.RefModel(cfg, P)
    b = synth.make_batch(cfg, 1, seed=2)
    xn, qr, vis, pos = _layer_inputs(cfg, om, b, 0)
    dout = np.random.default_rng(1).normal(size=(len(qr), cfg.model_dim))
    dx, _ = rm.attention_backward(0, xn, qr, vis, pos, dout, ["attn.0.wq"])
    rng = np.random.default_rng(4)
    for _ in range(3):
        u = rng.normal(size=xn.shape)
        eps = 1e-5
        f = lambda x: float(np.sum(dout * rm.attention(0, x, qr, vis, pos)))  # noqa: E731
        fd = (f(xn + eps * u) - f(xn - eps * u)) / (2 * eps)
        assert abs(fd - float(np.sum(dx * u))) <= 1e-6 * max(1.0, abs(fd))


@pytest.mark.parametrize("variant", ["tiny", "tiny_geo", "tiny_keep_specials", "mid_prune2"])
def test_model_forward_reference_composition_vs_oracle(variant):
    """Whole-model logits: the reference's tokenizer / build_mask / retained_rows /
    AttentionLayer::forward / rmsnorm_forward composed with the spec-only FFN, block and head
    (oracle/ref_harness.cpp) equal the oracle's model_forward."""
    if variant == "mid_prune2":
        cfg = base_config(n_hist=200, n_cand=12, n_items=3000, layers=4)
        cfg.keep = [cfg.prefix_len, cfg.prefix_len, 40, 40]
    else:
        cfg = tiny_config()
        if variant == "tiny_geo":
            cfg.keep = geometric_schedule(cfg.prefix_len, cfg.layers, 128)
        if variant == "tiny_keep_specials":
            cfg.keep = [cfg.prefix_len, 50]
            cfg.keep_specials = True
    P = synth.make_params(cfg, seed=12)
    om, rm = O.OracleModel(cfg, P), RF.RefModel(cfg, P)
    b = synth.make_batch(cfg, 2, seed=13)
    for i in range(2):
        po, lo = om.forward(b, i)
        pr, lr = rm.forward(b, i)
        assert _close(lo, lr) and _close(po, pr)
