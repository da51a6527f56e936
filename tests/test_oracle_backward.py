# SPDX-License-Identifier: Apache-2.0
"""The fp64 oracle's training backward (AttentionLayer::backward, attention.cpp:134-202, with
the intended math; rmsnorm_backward, norm.hpp:32-45; the spec's SwishGLU FFN / pre-norm
blocks / ranking head) pinned by central finite differences of the
oracle's own forward, as SPEC.md:411 prescribes. CPU only."""
import numpy as np
import pytest

import oracle as O
from paper_2603_03988_b200 import synth
from paper_2603_03988_b200.config import tiny_config

FD_EPS = 1e-5
FD_REL_TOL = 1e-6   # fp64 central differences on an O(1) loss


@pytest.fixture(scope="module")
def setup():
    # pruning after layer 0, windowed + full-causal rows, specials kept
    cfg = tiny_config(n_hist=40, n_cand=5, keep=[46, 20], local_window=8, full_suffix=6)
    P = {k: v.astype(np.float64) for k, v in synth.make_params(cfg, seed=3).items()}
    b = synth.make_batch(cfg, 1, seed=4)
    W = np.random.default_rng(0).normal(size=(cfg.n_cand, 3))
    return cfg, P, b, W


def _loss(cfg, P, b, W):
    _, z = O.OracleModel(cfg, P).forward(b, 0)
    return float((W * z).sum())


def _fd(cfg, P, b, W, name, idx):
    Pp = dict(P); Pp[name] = P[name].copy(); Pp[name][idx] += FD_EPS
    Pm = dict(P); Pm[name] = P[name].copy(); Pm[name][idx] -= FD_EPS
    return (_loss(cfg, Pp, b, W) - _loss(cfg, Pm, b, W)) / (2 * FD_EPS)


def test_param_grads_match_finite_differences(setup):
    cfg, P, b, W = setup
    names = [n for n in P if not n.startswith("tok.")]
    g, _ = O.OracleModel(cfg, P).backward(b, 0, W, names)
    rng = np.random.default_rng(1)
    for n in names:
        assert g[n] is not None and g[n].shape == P[n].shape, n
        for _ in range(2):
            idx = tuple(int(rng.integers(0, s)) for s in P[n].shape)
            fd = _fd(cfg, P, b, W, n, idx)
            an = g[n][idx]
            assert abs(fd - an) <= FD_REL_TOL * max(1.0, abs(fd)) + 1e-9, (n, idx, fd, an)


def test_tokenizer_grads_match_finite_differences(setup):
    """Tokenizer::backward (tokenizer.cpp:286-352): projections, biases, gains, specials and the
    feature tables (the item table is frozen: no gradient)."""
    cfg, P, b, W = setup
    names = [n for n in P if n.startswith("tok.")]
    g, _ = O.OracleModel(cfg, P).backward(b, 0, W, names)
    assert g["tok.item_table"] is None
    rng = np.random.default_rng(4)
    used = {"tok.action_table": b["hist_action"][0], "tok.scene_table": b["hist_scene"][0]}
    for n in names:
        if n == "tok.item_table":
            continue
        assert g[n] is not None and g[n].shape == P[n].shape, n
        for _ in range(2):
            if n in used:  # probe a row the request actually uses
                idx = (int(rng.choice(used[n])), int(rng.integers(0, P[n].shape[1])))
            else:
                idx = tuple(int(rng.integers(0, s)) for s in P[n].shape)
            fd = _fd(cfg, P, b, W, n, idx)
            assert abs(fd - g[n][idx]) <= FD_REL_TOL * max(1.0, abs(fd)) + 1e-9, (n, idx, fd, g[n][idx])


def test_dtokens_match_finite_differences(setup):
    """Special rows enter the sequence raw (tokenizer.cpp:171-176), so d loss / d special[k]
    equals dtokens at that special token's row (BOS = row 0, first SEP = row 1 + H)."""
    cfg, P, b, W = setup
    _, dt = O.OracleModel(cfg, P).backward(b, 0, W, [])
    for k, row in ((0, 0), (1, 1 + cfg.n_hist)):
        for j in (0, 7, cfg.model_dim - 1):
            fd = _fd(cfg, P, b, W, "tok.special", (k, j))
            assert abs(fd - dt[row, j]) <= FD_REL_TOL * max(1.0, abs(fd)) + 1e-9, (k, j)


# ----------------------------------------------------------------------- loss / optimizer KATs
def test_bce_loss_spec_examples():
    """SPEC.md:386-389."""
    z = np.zeros((4, 3))
    loss, _ = O.bce_loss(z, np.ones((4, 3)), weights=(1.0, 0.0, 0.0))
    assert abs(loss - np.log(2)) < 1e-12                       # p = 0.5 -> ln 2
    z = np.full((1, 3), np.log(0.9 / 0.1))                     # p = 0.9
    loss, dz = O.bce_loss(z, np.ones((1, 3)), weights=(1.0, 0.0, 0.0))
    assert abs(loss - 0.10536051565782628) < 1e-12             # -ln 0.9
    assert abs(dz[0, 0] - (0.9 - 1.0)) < 1e-12 and dz[0, 1] == 0.0


def test_adamw_spec_examples():
    """SPEC.md:453-456."""
    p, m, v = O.adamw(np.array([1.0]), np.array([0.0]), 0.0, 0.0, 1, lr=0.1, wd=0.0)
    assert p[0] == 1.0                                          # zero grad, zero wd
    p, _, _ = O.adamw(np.array([1.0]), np.array([1.0]), 0.0, 0.0, 1, lr=0.1, wd=0.0)
    assert abs(p[0] - (1 - 0.1 / (1 + 1e-8))) < 1e-12          # ~0.9
    p, _, _ = O.adamw(np.array([2.0]), np.array([0.0]), 0.0, 0.0, 1, lr=0.1, wd=0.01)
    assert abs(p[0] - 2.0 * (1 - 0.001)) < 1e-12               # decay only
