# SPDX-License-Identifier: Apache-2.0
"""The MoE FFN oracle against the spec's examples and an independent numpy
restatement: route_topk (exactly-k, ties -> lower index, bias-free reduction, brute-force sort
oracle, bias-neutral combine), moe_forward (dense reduction bit-for-bit, weighted aggregation),
update_balance (uniform -> no change, monotonicity) and the model-level routing control."""
import dataclasses

import numpy as np
import pytest

import oracle as O
from paper_2603_03988_b200.config import SortConfig
from paper_2603_03988_b200.flops import forward_flops
from paper_2603_03988_b200.synth import make_batch, make_params


def _sig(z):
    return 1.0 / (1.0 + np.exp(-z))


def _np_route(x, router, bias, k):
    s = _sig(x @ router)
    b = s + bias[None, :]
    E = router.shape[1]
    sel = np.zeros((x.shape[0], k), np.int32)
    for i in range(x.shape[0]):
        order = sorted(range(E), key=lambda e: (-b[i, e], e))  # brute-force sort, lower index on ties
        sel[i] = order[:k]
    w = np.take_along_axis(s, sel, 1)
    return sel, w / w.sum(1, keepdims=True)


def _swishglu(x, g, u, d):
    a, b = x @ g, x @ u
    return (a * _sig(a) * b) @ d


def test_route_all_experts_when_k_equals_E():
    rng = np.random.default_rng(1)
    x, r = rng.normal(size=(7, 16)), rng.normal(size=(16, 4))
    sel, w, mg = O.moe_route(x, r, rng.normal(size=4), 4)
    assert all(sorted(row) == [0, 1, 2, 3] for row in sel.tolist())
    np.testing.assert_allclose(w.sum(1), 1.0, rtol=1e-15)
    assert np.all(np.isinf(mg))


def test_route_matches_bruteforce_sort_E8_k2():
    rng = np.random.default_rng(2)
    x, r, b = rng.normal(size=(200, 32)), rng.normal(size=(32, 8)) / 6, 0.05 * rng.normal(size=8)
    sel, w, _ = O.moe_route(x, r, b, 2)
    esel, ew = _np_route(x, r, b, 2)
    np.testing.assert_array_equal(sel, esel)
    np.testing.assert_allclose(w, ew, rtol=1e-13)


def test_route_zero_bias_is_plain_topk():
    rng = np.random.default_rng(3)
    x, r = rng.normal(size=(50, 16)), rng.normal(size=(16, 8))
    sel, _, _ = O.moe_route(x, r, None, 3)
    s = x @ r
    np.testing.assert_array_equal(sel, np.argsort(-s, axis=1, kind="stable")[:, :3])


def test_route_ties_break_to_lower_index():
    rng = np.random.default_rng(4)
    x = rng.normal(size=(6, 8))
    col = rng.normal(size=(8, 1))
    r = np.repeat(col, 5, axis=1)  # all five experts score identically
    sel, w, mg = O.moe_route(x, r, None, 2)
    assert sel.tolist() == [[0, 1]] * 6
    np.testing.assert_allclose(w, 0.5)
    np.testing.assert_array_equal(mg, 0.0)


def test_combine_weights_are_bias_neutral():
    rng = np.random.default_rng(5)
    E, k, d, m = 6, 2, 16, 8
    x, r = rng.normal(size=(40, d)), rng.normal(size=(d, E)) / 4
    wg, wu, wd = (rng.normal(size=s) / 4 for s in ((E, d, m), (E, d, m), (E, m, d)))
    sel, _, _ = O.moe_route(x, r, None, k)
    o1, s1, w1 = O.moe_ffn(x, r, np.zeros(E), k, wg, wu, wd, forced=sel)
    o2, s2, w2 = O.moe_ffn(x, r, rng.normal(size=E), k, wg, wu, wd, forced=sel)
    np.testing.assert_array_equal(s1, s2)
    np.testing.assert_array_equal(w1, w2)
    np.testing.assert_array_equal(o1, o2)


def test_dense_reduction_bit_for_bit():
    rng = np.random.default_rng(6)
    d, m = 16, 12
    x = rng.normal(size=(9, d))
    g, u, dn = rng.normal(size=(d, m)), rng.normal(size=(d, m)), rng.normal(size=(m, d))
    out, sel, w = O.moe_ffn(x, rng.normal(size=(d, 1)), None, 1, g[None], u[None], dn[None])
    assert np.all(sel == 0) and np.all(w == 1.0)
    np.testing.assert_array_equal(out, O.swishglu(x, g, u, dn))


def test_spec_scalar_expert():
    # m = 1, gate = [1, 0], up = [0, 1], down = [1]^T on x = (2, 3): swish(2) * 3 ~ 5.2848
    g = np.array([[[1.0], [0.0]]])
    u = np.array([[[0.0], [1.0]]])
    dn = np.array([[[1.0, 0.0]]])
    out, _, _ = O.moe_ffn(np.array([[2.0, 3.0]]), np.zeros((2, 1)), None, 1, g, u, dn)
    assert out[0, 0] == pytest.approx(2 * _sig(2.0) * 3, rel=1e-15)
    assert out[0, 0] == pytest.approx(5.2848, abs=1e-4)


@pytest.mark.parametrize("shared", [0, 1])
def test_moe_ffn_matches_numpy(shared):
    rng = np.random.default_rng(7 + shared)
    E, k, d, m = 8, 2, 24, 10
    n = E + shared
    x, r, b = rng.normal(size=(64, d)), rng.normal(size=(d, E)) / 5, 0.05 * rng.normal(size=E)
    wg, wu, wd = (rng.normal(size=s) / 4 for s in ((n, d, m), (n, d, m), (n, m, d)))
    out, sel, w = O.moe_ffn(x, r, b, k, wg, wu, wd, shared=shared)
    esel, ew = _np_route(x, r, b, k)
    np.testing.assert_array_equal(sel, esel)
    ref = np.zeros_like(x)
    for i in range(x.shape[0]):
        for j in range(k):
            e = esel[i, j]
            ref[i] += ew[i, j] * _swishglu(x[i:i + 1], wg[e], wu[e], wd[e])[0]
        if shared:
            ref[i] += _swishglu(x[i:i + 1], wg[E], wu[E], wd[E])[0]
    np.testing.assert_allclose(out, ref, rtol=1e-12, atol=1e-12)


def test_update_bias_uniform_and_monotone():
    b0 = np.array([0.1, -0.2, 0.0, 0.3])
    np.testing.assert_array_equal(O.moe_update_bias([5, 5, 5, 5], b0), b0)
    b1 = O.moe_update_bias([100, 0, 0, 0], b0, gamma=1e-3)
    assert b1[0] < b0[0] and np.all(b1[1:] > b0[1:])
    np.testing.assert_allclose(b1 - b0, [-1e-3, 1e-3, 1e-3, 1e-3], rtol=1e-12)


def _moe_cfg(**kw):
    base = dict(model_dim=64, heads=4, layers=2, ffn_dim=160, n_hist=40, n_cand=8, local_window=16,
                full_suffix=16, keep=[46, 12], n_items=500, moe_experts=8, moe_topk=1, moe_shared=1,
                moe_ffn_dim=80)
    base.update(kw)
    return SortConfig(**base)


def test_model_forward_moe_routing_control():
    cfg = _moe_cfg()
    params = make_params(cfg, seed=3)
    batch = make_batch(cfg, 1, seed=4)
    om = O.OracleModel(cfg, params)
    p0, _ = om.forward(batch, 0)
    p1, _, sel, mg = om.forward_moe(batch, 0)
    np.testing.assert_array_equal(p0, p1)
    lq = om.layer_meta(batch, 0)["l_q"]
    assert [s.shape for s in sel] == [(q, 1) for q in lq]
    assert all(np.all(m > 0) for m in mg)
    p2, _, sel2, _ = om.forward_moe(batch, 0, forced=sel)  # own routing forced -> identical
    np.testing.assert_array_equal(p1, p2)
    flipped = [s.copy() for s in sel]
    flipped[0] = (flipped[0] + 1) % cfg.moe_experts
    p3, _, sel3, _ = om.forward_moe(batch, 0, forced=flipped)
    np.testing.assert_array_equal(sel3[0], flipped[0])
    assert np.abs(p3 - p1).max() > 1e-6


def test_flops_invariance_and_dense_match():
    dense = SortConfig(model_dim=64, heads=4, layers=2, ffn_dim=160, n_hist=40, n_cand=8, keep=[46, 12])
    f_dense = forward_flops(dense)["ffn"]
    for E in (2, 4, 8, 16):  # activated FLOPs do not depend on E beyond the router
        moe = dataclasses.replace(dense, moe_experts=E, moe_topk=1, moe_shared=1, moe_ffn_dim=80)
        assert abs(forward_flops(moe)["ffn"] / f_dense - 1.0) < 0.02 + 2 * E / (6 * 160)
    moe8 = dataclasses.replace(dense, moe_experts=8, moe_topk=1, moe_shared=1, moe_ffn_dim=80)
    assert abs(forward_flops(moe8)["ffn"] / f_dense - 1.0) < 0.02
