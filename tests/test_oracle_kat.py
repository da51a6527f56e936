# SPDX-License-Identifier: Apache-2.0
"""Pins the CPU oracle against every known-answer example SPEC.md gives for the
hot path (the reference ships no tests/fixtures -- SURVEY.md section 4) and the
derived counts in SURVEY.md section 8, plus cross-checks against the independent
numpy restatement in np_ref.py. CPU only."""
import json
import math
import os

import numpy as np
import pytest

import oracle as O
import np_ref
from paper_2603_03988_b200.config import (ROLE_BOS, ROLE_CAND, ROLE_HIST, ROLE_PROF, ROLE_SEP,
                                          base_config, tiny_config, large_config)
from paper_2603_03988_b200 import synth

KAT = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_kats.json")))


@pytest.fixture(scope="module")
def tiny():
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=3)
    return cfg, P, O.OracleModel(cfg, P)


def _batch_with(cfg, n_hist, n_prof_vals, n_cand, seed=0):
    rng = np.random.default_rng(seed)
    return {
        "hist_item": rng.integers(0, cfg.n_items, (1, n_hist), dtype=np.int32),
        "hist_action": rng.integers(0, 3, (1, n_hist), dtype=np.int32),
        "hist_scene": rng.integers(0, 4, (1, n_hist), dtype=np.int32),
        "hist_ts": np.sort(rng.integers(0, 1000, (1, n_hist))).astype(np.int64),
        "req_ts": np.array([5000], np.int64),
        "profile": np.array([n_prof_vals], np.int32),
        "cand_item": rng.integers(0, cfg.n_items, (1, n_cand), dtype=np.int32),
    }


# ------------------------------------------------------------------ time buckets
def test_time_bucket_matches_integer_form():
    """tokenizer.cpp:36-40 -- the double-log2 rule equals min(63-clz(1+d), nb-1)."""
    vals = [0, 1, 2, 3, 4, 7, 8, 1023, 1024, 1025, 2**31 - 1, 2**31, 2**40, 2**62, -5]
    for k in range(1, 62):
        vals += [2**k - 3, 2**k - 2, 2**k - 1, 2**k, 2**k + 1]
    for d in vals:
        dd = max(d, 0)
        ref = min((1 + dd).bit_length() - 1, 31)
        assert O.time_bucket(d, 32) == ref, d


# ------------------------------------------------------------------ tokenizer
def test_tokenizer_minimal_sequence():
    k = KAT["tokenizer_minimal"]
    cfg = tiny_config(profile_vocab=[8], n_hist=0, n_cand=1)
    m = O.OracleModel(cfg, synth.make_params(cfg, seed=1))
    t = m.tokenize(_batch_with(cfg, 0, [3], 1))
    assert len(t["roles"]) == k["L"]
    assert t["roles"].tolist() == k["roles"]


def test_tokenizer_candidate_positions():
    k = KAT["tokenizer_cand_positions"]
    cfg = tiny_config(profile_vocab=[8, 8], n_hist=3, n_cand=4)
    m = O.OracleModel(cfg, synth.make_params(cfg, seed=1))
    t = m.tokenize(_batch_with(cfg, 3, [1, 2], 4))
    cand = t["roles"] == ROLE_CAND
    assert set(t["position_ids"][cand].tolist()) == {k["cand_pos"]}
    assert t["position_ids"][~cand].tolist() == list(range(8))
    assert len(t["roles"]) == 1 + 3 + 1 + 2 + 1 + 4


def test_tokenizer_oov_is_config_error(tiny):
    cfg, P, m = tiny
    b = synth.make_batch(cfg, 1, seed=2)
    b["hist_item"][0, 5] = cfg.n_items
    with pytest.raises(O.OracleError) as e:
        m.tokenize(b)
    assert e.value.status == 1


def test_tokenizer_zero_candidates_error():
    cfg = tiny_config(n_cand=0)
    m = O.OracleModel(cfg, synth.make_params(tiny_config(), seed=1))
    with pytest.raises(O.OracleError) as e:
        m.tokenize(_batch_with(cfg, 4, [1, 2, 3], 0))
    assert e.value.status == 1


def test_rmsnorm_zero_vector_eps_guard():
    y = O.rmsnorm(np.zeros((2, 8)), np.ones(8))
    assert np.all(y == 0.0)


def test_tokenizer_matches_numpy(tiny):
    cfg, P, m = tiny
    b = synth.make_batch(cfg, 1, seed=4)
    t = m.tokenize(b)
    x, roles, pos, tb = np_ref.tokenize(P, cfg, b)
    np.testing.assert_allclose(t["tokens"], x, rtol=1e-12, atol=1e-12)
    assert t["roles"].tolist() == roles.tolist()
    assert t["position_ids"].tolist() == pos.tolist()
    assert t["hist_time"].tolist() == tb.tolist()


# ------------------------------------------------------------------ masks / pruning
def test_mask_causal_reduction():
    n = 9
    roles = [ROLE_HIST] * n
    vis = O.build_mask(n, roles, list(range(n)), local_window=-1, full_suffix=0)
    assert np.array_equal(vis, np.tril(np.ones((n, n), np.uint8)))


def test_mask_two_candidates_hand_case():
    k = KAT["mask_two_candidates"]
    vis = O.build_mask(5, k["roles"], k["pos"], local_window=-1, full_suffix=128)
    assert vis.tolist() == k["visible"]


def test_mask_query_row_out_of_range_is_config_error():
    with pytest.raises(O.OracleError) as e:
        O.build_mask(1, [ROLE_HIST] * 3, [0, 1, 2], -1, 0, query_rows=[3])
    assert e.value.status == 1


def test_prune_queries():
    k = KAT["prune_queries"]
    x = np.arange(10 * 3, dtype=np.float64).reshape(10, 3)
    assert np.array_equal(O.prune_queries(x, 10), x)
    assert np.array_equal(O.prune_queries(x, 1), x[-1:])
    assert np.array_equal(O.prune_queries(x, k["n"]), x[k["rows"]])
    with pytest.raises(O.OracleError):
        O.prune_queries(x, 11)


def test_geometric_schedules():
    k = KAT["schedules"]
    assert O.geometric_schedule(1030, 4, 128) == k["geo_1030_4_128"]
    assert O.geometric_schedule(4102, 12, 128) == k["geo_4102_12_128"]
    assert O.geometric_schedule(262, 2, 128) == k["geo_262_2_128"]
    from paper_2603_03988_b200.config import geometric_schedule as py_geo
    for p in (1, 5, 129, 262, 1030, 4102):
        for dpt in (1, 2, 3, 4, 12):
            assert py_geo(p, dpt, 128) == O.geometric_schedule(p, dpt, 128)


def _layer_visible_counts(cfg):
    m = O.OracleModel(cfg, synth.make_params(cfg, seed=1)) if cfg.n_items <= 5000 else None
    return m


def _struct_roles(cfg):
    roles = [ROLE_BOS] + [ROLE_HIST] * cfg.n_hist + [ROLE_SEP] + [ROLE_PROF] * cfg.n_prof + \
        [ROLE_SEP] + [ROLE_CAND] * cfg.n_cand
    L = len(roles)
    pos = list(range(L - cfg.n_cand)) + [L - cfg.n_cand] * cfg.n_cand
    return roles, pos


def test_visible_counts_sort_base_and_tiny():
    k = KAT["visible_counts"]
    cfg = base_config()
    roles, pos = _struct_roles(cfg)
    counts = []
    r, p = np.array(roles), np.array(pos)
    for keep in cfg.keep_schedule():
        qr = O.retained_rows(r.tolist(), keep, False)
        vis = O.build_mask(len(qr), r.tolist(), p.tolist(), cfg.local_window, cfg.full_suffix, qr)
        counts.append(int(vis.sum()))
        r, p = r[qr], p[qr]
    assert counts == [k["base_layer12"], k["base_layer12"], k["base_layer3"], k["base_layer4"]]
    t = tiny_config()
    roles, pos = _struct_roles(t)
    vis = O.build_mask(len(roles), roles, pos, t.local_window, t.full_suffix)
    assert int(vis.sum()) == k["tiny_full"]


def test_mask_rows_are_single_interval_plus_self():
    """visible set = one contiguous non-candidate kv interval (+ self)."""
    rng = np.random.default_rng(0)
    for trial in range(120):
        n_hist = int(rng.integers(0, 40))
        n_cand = int(rng.integers(0, 6))
        roles = [ROLE_BOS] + [ROLE_HIST] * n_hist + [ROLE_SEP, ROLE_PROF, ROLE_SEP] + \
            [ROLE_CAND] * n_cand
        L = len(roles)
        pos = list(range(L - n_cand)) + [L - n_cand] * n_cand
        W = int(rng.choice([-1, 1, 2, 5, 17]))
        F = int(rng.integers(0, 20))
        r, p = np.array(roles), np.array(pos)
        for _ in range(int(rng.integers(1, 4))):
            keep = int(rng.integers(1, L + 1))
            qr = O.retained_rows(r.tolist(), keep, bool(rng.integers(0, 2)))
            vis = O.build_mask(len(qr), r.tolist(), p.tolist(), W, F, qr)
            ref = np_ref.mask_np(r, p, qr, W, F)
            assert np.array_equal(vis, ref)
            for i, qi in enumerate(qr):
                cols = np.nonzero(vis[i])[0]
                noncand = [c for c in cols if r[c] != ROLE_CAND]
                if noncand:
                    assert noncand == list(range(noncand[0], noncand[-1] + 1))
                cands = [c for c in cols if r[c] == ROLE_CAND]
                assert cands in ([], [qi])
            r, p = r[qr], p[qr]


# ------------------------------------------------------------------ rope
def test_rope_position_zero_identity_and_shift_invariance():
    rng = np.random.default_rng(1)
    x = rng.normal(size=(3, 16))
    assert np.allclose(O.rope(x, [0, 0, 0]), x, atol=0, rtol=0)
    q, k = rng.normal(size=(1, 16)), rng.normal(size=(1, 16))
    a = (O.rope(q, [3]) @ O.rope(k, [7]).T).item()
    b = (O.rope(q, [103]) @ O.rope(k, [107]).T).item()
    assert abs(a - b) < 1e-6
    # inverse is the exact adjoint
    assert np.allclose(O.rope(O.rope(x, [5, 9, 1030]), [5, 9, 1030], inverse=True), x, atol=1e-12)
    assert np.allclose(O.rope(x, [4, 5, 6]), np_ref.rope(x, [4, 5, 6]), atol=1e-14)


# ------------------------------------------------------------------ attention layer
def _attn_setup(cfg, P, L, seed=0):
    rng = np.random.default_rng(seed)
    xn = rng.normal(size=(L, cfg.model_dim))
    roles = [ROLE_HIST] * L
    pos = list(range(L))
    qr = list(range(L))
    vis = O.build_mask(L, roles, pos, -1, 0, qr)
    return xn, qr, vis, pos


def test_attention_random_12_tokens_vs_plain(tiny):
    cfg, P, m = tiny
    xn, qr, vis, pos = _attn_setup(cfg, P, 12)
    out = m.attention(0, xn, qr, vis, pos)
    ref = np_ref.attention_layer({k: np.asarray(v, np.float64) for k, v in P.items()}, 0, cfg, xn,
                                 qr, vis, pos)
    assert np.max(np.abs(out - ref)) < 1e-5


def test_attention_zero_gate_weights_halve_output(tiny):
    cfg, P, _ = tiny
    P0 = dict(P)
    P0["attn.0.wg"] = np.zeros_like(P["attn.0.wg"])
    gated = O.OracleModel(cfg, P0)
    import dataclasses
    ungated = O.OracleModel(dataclasses.replace(cfg, gate=False), P0)
    xn, qr, vis, pos = _attn_setup(cfg, P0, 10, seed=1)
    a = gated.attention(0, xn, qr, vis, pos)
    b = ungated.attention(0, xn, qr, vis, pos)
    assert np.allclose(a, 0.5 * b, atol=1e-12)


def test_attention_one_token_is_gated_value_row(tiny):
    cfg, P, m = tiny
    xn, qr, vis, pos = _attn_setup(cfg, P, 1, seed=2)
    out = m.attention(0, xn, qr, vis, pos)
    Pd = {k: np.asarray(v, np.float64) for k, v in P.items()}
    v = xn @ Pd["attn.0.wv"]
    g = np_ref.sigmoid(xn @ Pd["attn.0.wg"])
    assert np.allclose(out, (g * v) @ Pd["attn.0.wo"], atol=1e-12)


def test_pruning_as_restriction(tiny):
    """pruned layer == unpruned layer restricted to the kept rows (W=inf)."""
    cfg, P, m = tiny
    L = 20
    xn, qr_full, vis_full, pos = _attn_setup(cfg, P, L, seed=5)
    full = m.attention(0, xn, qr_full, vis_full, pos)
    keep = list(range(L - 7, L))
    vis = O.build_mask(len(keep), [ROLE_HIST] * L, pos, -1, 0, keep)
    pr = m.attention(0, xn, keep, vis, pos)
    assert np.max(np.abs(pr - full[keep])) < 1e-5


# ------------------------------------------------------------------ block operator
def _qkv(rng, lq, lkv, dk, dtype=np.float64):
    return (rng.normal(size=(lq, dk)).astype(dtype), rng.normal(size=(lkv, dk)).astype(dtype),
            rng.normal(size=(lkv, dk)).astype(dtype))


def _addmask(vis, dtype=np.float64):
    return np.where(vis.astype(bool), 0.0, -np.inf).astype(dtype)


def test_blockwise_all_visible_no_skips():
    rng = np.random.default_rng(0)
    q, k, v = _qkv(rng, 40, 40, 8)
    m = np.zeros((40, 40))
    out, sk, tot = O.blockwise_attention(q, k, v, m, 16)
    assert sk == 0 and tot == 9
    assert np.max(np.abs(out - O.dense_attention(q, k, v, m))) < 1e-6


def test_blockwise_candidate_diagonal_skips():
    """N=64 candidates, B=16: >= (N/B)^2 - N/B candidate-region tiles skipped."""
    N, P = 64, 64
    roles = [ROLE_HIST] * P + [ROLE_CAND] * N
    pos = list(range(P)) + [P] * N
    vis = O.build_mask(P + N, roles, pos, -1, 0)
    rng = np.random.default_rng(2)
    q, k, v = _qkv(rng, P + N, P + N, 8)
    _, sk, _ = O.blockwise_attention(q, k, v, _addmask(vis), 16)
    # count skipped tiles inside the candidate x candidate region
    nb = N // 16
    cand_skipped = sum(1 for i in range(nb) for j in range(nb)
                       if not vis[P + 16 * i:P + 16 * i + 16, P + 16 * j:P + 16 * j + 16].any())
    assert cand_skipped >= nb * nb - nb


def test_blockwise_local_window_skip_fraction_and_equivalence():
    """W=256 local mask on L=4096: skip fraction >= 1-(2W+B)/L per q-block
    row, output equals dense to 1e-5; overall skip fraction >= 0.85."""
    L, W, B = 4096, 256, 16
    roles = [ROLE_HIST] * L
    pos = list(range(L))
    vis = O.build_mask(L, roles, pos, W, 0)
    # per q-block-row skip fraction from the mask itself
    nb = L // B
    tiles = vis.reshape(nb, B, nb, B).any(axis=(1, 3))
    assert np.all(1.0 - tiles.sum(axis=1) / nb >= 1.0 - (2 * W + B) / L - 1e-12)
    rng = np.random.default_rng(3)
    q, k, v = _qkv(rng, L, L, 16)
    out, sk, tot = O.blockwise_attention(q, k, v, _addmask(vis), B)
    assert sk / tot >= 0.85
    dense = O.dense_attention(q, k, v, _addmask(vis))
    assert np.max(np.abs(out - dense)) < 1e-5


def test_blockwise_vs_dense_acceptance_100_cases():
    """SPEC.md:570 acceptance #1: < 1e-9 at fp64 and < 1e-4 at fp32 over 100 random cases."""
    rng = np.random.default_rng(4)
    for case in range(100):
        lq = int(rng.integers(1, 40))
        lkv = lq + int(rng.integers(0, 30))
        dk = int(rng.choice([2, 4, 8, 16]))
        vis = (rng.random((lq, lkv)) < 0.6).astype(np.uint8)
        vis[np.arange(lq), rng.integers(0, lkv, lq)] = 1  # every row has a visible key
        B = int(rng.integers(1, 20))
        q, k, v = _qkv(rng, lq, lkv, dk)
        out, _, _ = O.blockwise_attention(q, k, v, _addmask(vis), B)
        assert np.max(np.abs(out - O.dense_attention(q, k, v, _addmask(vis)))) < 1e-9
        o32, _, _ = O.blockwise_attention(q, k, v, _addmask(vis, np.float32), B, dtype=np.float32)
        d32 = O.dense_attention(q, k, v, _addmask(vis, np.float32), dtype=np.float32)
        assert np.max(np.abs(o32 - d32)) < 1e-4


def test_block_skip_counts_sort_base_layer1():
    k = KAT["block_skip"]
    cfg = base_config()
    roles, pos = _struct_roles(cfg)
    vis = O.build_mask(len(roles), roles, pos, cfg.local_window, cfg.full_suffix)
    L = len(roles)
    for B, sk_ref, tot_ref in ((16, k["base_l1_b16_skipped"], k["base_l1_b16_total"]),
                               (128, k["base_l1_b128_skipped"], k["base_l1_b128_total"])):
        nb = -(-L // B)
        pad = np.zeros((nb * B, nb * B), np.uint8)
        pad[:L, :L] = vis
        any_t = pad.reshape(nb, B, nb, B).any(axis=(1, 3))
        assert nb * nb == tot_ref and int((~any_t).sum()) == sk_ref


# ------------------------------------------------------------------ FFN
def test_swishglu_known_answers():
    k = KAT["swishglu_hand"]
    x = np.array([k["x"]])
    out = O.swishglu(x, np.array([[1.0], [0.0]]), np.array([[0.0], [1.0]]), np.array([[1.0]]))
    assert abs(out[0, 0] - k["value"]) < 1e-4
    z = O.swishglu(np.ones((3, 4)), np.zeros((4, 5)), np.zeros((4, 5)), np.zeros((5, 4)))
    assert np.all(z == 0.0)


# ------------------------------------------------------------------ model
def test_model_matches_numpy(tiny):
    cfg, P, m = tiny
    b = synth.make_batch(cfg, 1, seed=9)
    p, lg = m.forward(b)
    pr, lr = np_ref.model_forward(P, cfg, b)
    assert np.max(np.abs(lg - lr)) < 1e-9


def test_model_pruned_schedule_matches_numpy():
    cfg = tiny_config(keep=[262, 128], keep_specials=False)
    P = synth.make_params(cfg, seed=11)
    m = O.OracleModel(cfg, P)
    b = synth.make_batch(cfg, 1, seed=12)
    _, lg = m.forward(b)
    _, lr = np_ref.model_forward(P, cfg, b)
    assert np.max(np.abs(lg - lr)) < 1e-9
    cfg2 = tiny_config(keep=[200, 100], keep_specials=True)
    m2 = O.OracleModel(cfg2, P)
    _, lg2 = m2.forward(b)
    _, lr2 = np_ref.model_forward(P, cfg2, b)
    assert np.max(np.abs(lg2 - lr2)) < 1e-9


def test_model_zero_params_give_half():
    cfg = tiny_config()
    P = {k: np.zeros_like(v) for k, v in synth.make_params(cfg, seed=1).items()}
    m = O.OracleModel(cfg, P)
    p, _ = m.forward(synth.make_batch(cfg, 1, seed=1))
    assert np.all(p == 0.5)


def test_model_candidate_permutation_and_isolation(tiny):
    cfg, P, m = tiny
    b = synth.make_batch(cfg, 1, seed=21)
    p, _ = m.forward(b)
    perm = np.random.default_rng(0).permutation(cfg.n_cand)
    b2 = {k: v.copy() for k, v in b.items()}
    b2["cand_item"][0] = b["cand_item"][0][perm]
    p2, _ = m.forward(b2)
    assert np.array_equal(p2, p[perm])
    # isolation: changing candidate 3 leaves all others bit-identical
    b3 = {k: v.copy() for k, v in b.items()}
    b3["cand_item"][0, 3] = (b["cand_item"][0, 3] + 1) % cfg.n_items
    p3, _ = m.forward(b3)
    others = [i for i in range(cfg.n_cand) if i != 3]
    assert np.array_equal(p3[others], p[others])


def test_request_centric_equals_impression_centric(tiny):
    """one request-centric pass == N single-candidate passes (1e-4)."""
    cfg, P, m = tiny
    import dataclasses
    b = synth.make_batch(cfg, 1, seed=31)
    p, _ = m.forward(b)
    c1 = dataclasses.replace(cfg, n_cand=1)
    m1 = O.OracleModel(c1, P)
    for j in range(cfg.n_cand):
        bj = {k: v.copy() for k, v in b.items()}
        bj["cand_item"] = b["cand_item"][:, j:j + 1].copy()
        pj, _ = m1.forward(bj)
        assert np.max(np.abs(pj[0] - p[j])) < 1e-4


def test_flops_ratio_band():
    from paper_2603_03988_b200.flops import forward_flops
    cfg = base_config()
    import dataclasses
    geo = dataclasses.replace(cfg, keep=O.geometric_schedule(cfg.prefix_len, 4, 128))
    full = dataclasses.replace(cfg, keep=None)
    k = KAT["flops_ratio_geo_band"]
    ratio = forward_flops(geo)["block"] / forward_flops(full)["block"]
    assert k["lo"] <= ratio <= k["hi"]
    assert abs(ratio - k["derived"]) < 0.005
    # SORT-base "prune after layer 2": 5.456 GFLOP block stack per request
    assert abs(forward_flops(cfg)["block"] / 1e9 - 5.456) < 0.01


def test_oracle_reproduces_golden_fixture():
    """The committed fixture (tests/golden/make_golden.py) is reproduced bit-for-bit."""
    from golden.make_golden import params_digest, PARAM_SEED
    fx = np.load(os.path.join(os.path.dirname(__file__), "golden", "tiny_fixture.npz"))
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=PARAM_SEED)
    assert str(fx["params_sha256"]) == params_digest(P)
    m = O.OracleModel(cfg, P)
    batch = {k[3:]: fx[k] for k in fx.files if k.startswith("in_")}
    for i in range(batch["req_ts"].shape[0]):
        p, lg = m.forward(batch, i)
        assert np.array_equal(lg, fx["logits"][i])
        assert np.array_equal(m.tokenize(batch, i)["hist_time"], fx["hist_time"][i])
