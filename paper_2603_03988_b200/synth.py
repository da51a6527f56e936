# SPDX-License-Identifier: Apache-2.0
"""Seeded synthetic requests and random-init weights for the SORT path.

The reference's own generator (data.cpp:71-278) produces ~12-event histories
over 5,000 items (data.hpp:42,59) and cannot make the fixed 1024/4096-event
bench workloads, so this module writes the fixed-shape
workload SURVEY.md section 8(d) specifies:

* history: item ~ U[0, n_items), action ~ U{0,1,2}, scene ~ U[0, 4),
  timestamps non-decreasing and strictly before the request, gaps
  log-uniform over [1, 2^31] s so every one of the 32 recency buckets occurs;
* profile: one U[0, vocab_f) value per field;
* candidates: N distinct items; no side features.

Arrays are structure-of-arrays ``[B, H]`` int32/int64 -- the layout the GPU
tokenizer reads (the reference's AoS ``RequestSample``, data.hpp:13-38, is
what a host binding would pack from).

Weights use the reference parameter names (tokenizer.cpp:45-63,
attention.cpp:37-46) plus the spec-named block/FFN/head tensors. Values are
rounded to bf16-representable fp32 so the fp64 oracle and the bf16 GPU path
are fed identical weights.
"""
from __future__ import annotations

from typing import Dict

import numpy as np

from .config import SortConfig


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round-to-nearest-even to bf16, returned as float32."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    rounded = ((u + 0x7FFF + ((u >> 16) & 1)) >> 16) << 16
    return rounded.astype(np.uint32).view(np.float32)


def make_batch(cfg: SortConfig, batch: int, seed: int = 1) -> Dict[str, np.ndarray]:
    rng = np.random.default_rng(seed)
    H, N, B = cfg.n_hist, cfg.n_cand, batch
    req_ts = np.full((B,), 1_800_000_000, dtype=np.int64) + rng.integers(0, 86400, size=B)
    # log-uniform gaps: delta in [1, 2^31], oldest event first => delta non-increasing
    expo = rng.uniform(0.0, 31.0, size=(B, H))
    delta = np.floor(np.exp2(expo)).astype(np.int64)
    delta = -np.sort(-delta, axis=1)
    hist_ts = req_ts[:, None] - delta
    out = {
        "hist_item": rng.integers(0, cfg.n_items, size=(B, H), dtype=np.int32),
        "hist_action": rng.integers(0, cfg.n_actions, size=(B, H), dtype=np.int32),
        "hist_scene": rng.integers(0, cfg.n_scenes, size=(B, H), dtype=np.int32),
        "hist_ts": np.ascontiguousarray(hist_ts, dtype=np.int64),
        "req_ts": req_ts,
        "profile": np.stack([rng.integers(0, v, size=B, dtype=np.int32) for v in cfg.profile_vocab],
                            axis=1).astype(np.int32) if cfg.n_prof else np.zeros((B, 0), np.int32),
        "cand_item": np.stack([rng.choice(cfg.n_items, size=N, replace=False) for _ in range(B)]
                              ).astype(np.int32),
    }
    return {k: np.ascontiguousarray(v) for k, v in out.items()}


def param_shapes(cfg: SortConfig) -> Dict[str, tuple]:
    d, m = cfg.model_dim, cfg.ffn_dim
    dh = cfg.head_hidden or d
    hw = cfg.item_dim + cfg.action_dim + cfg.scene_dim + cfg.time_dim
    s = {
        "tok.special": (3, d),
        "tok.item_table": (cfg.n_items, cfg.item_dim),
        "tok.action_table": (cfg.n_actions, cfg.action_dim),
        "tok.scene_table": (cfg.n_scenes, cfg.scene_dim),
        "tok.time_table": (cfg.n_time_buckets, cfg.time_dim),
        "tok.w_hist": (hw, d), "tok.b_hist": (1, d), "tok.g_hist": (1, d),
        "tok.w_prof": (cfg.profile_dim, d), "tok.b_prof": (1, d), "tok.g_prof": (1, d),
        "tok.w_cand": (cfg.item_dim, d), "tok.b_cand": (1, d), "tok.g_cand": (1, d),
        "final_norm.gain": (1, d),
        "head.w1": (d, dh), "head.b1": (1, dh), "head.w2": (dh, 3), "head.b2": (1, 3),
    }
    for f, v in enumerate(cfg.profile_vocab):
        s[f"tok.profile_table.{f}"] = (v, cfg.profile_dim)
    if cfg.pretrain:  # tied next-item head: hidden -> item-embedding width
        s["pretrain.proj"] = (d, cfg.item_dim)
    for l in range(cfg.layers):
        for w in ("wq", "wk", "wv", "wo", "wg"):
            s[f"attn.{l}.{w}"] = (d, d)
        s[f"attn.{l}.qk_gain_q"] = (cfg.heads, cfg.head_dim)
        s[f"attn.{l}.qk_gain_k"] = (cfg.heads, cfg.head_dim)
        s[f"block.{l}.attn_norm"] = (1, d)
        s[f"block.{l}.ffn_norm"] = (1, d)
        if cfg.moe_experts > 0:
            E, me = cfg.moe_experts, cfg.moe_ffn_dim
            s[f"ffn.{l}.router"] = (d, E)
            s[f"ffn.{l}.router_bias"] = (1, E)
            names = [f"expert.{e}" for e in range(E)] + (["shared"] if cfg.moe_shared else [])
            for x in names:
                s[f"ffn.{l}.{x}.w_gate"] = (d, me)
                s[f"ffn.{l}.{x}.w_up"] = (d, me)
                s[f"ffn.{l}.{x}.w_down"] = (me, d)
        else:
            s[f"ffn.{l}.w_gate"] = (d, m)
            s[f"ffn.{l}.w_up"] = (d, m)
            s[f"ffn.{l}.w_down"] = (m, d)
    return s


def make_params(cfg: SortConfig, seed: int = 7, init: str = "fanin") -> Dict[str, np.ndarray]:
    """Random-init weights. ``init="spec"`` is SPEC.md's N(0, 0.02) with output
    projections scaled by 1/sqrt(2*depth); ``init="fanin"``
    (default) uses N(0, 1/fan_in) so every layer moves the scores visibly --
    the parity tests want errors in any layer to reach the logits. Gains are
    1 + 0.1*N(0,1) and biases 0.1*N(0,1) so they are non-trivial for parity."""
    rng = np.random.default_rng(seed)
    out = {}
    for name, (r, c) in param_shapes(cfg).items():
        leaf = name.rsplit(".", 1)[-1]
        if name.startswith("tok.") and name.endswith("table") or name == "tok.special" \
                or ".profile_table." in name:
            std = 0.02 if init == "spec" else 1.0
            a = rng.normal(0.0, std, size=(r, c))
        elif leaf.startswith("g_") or leaf in ("attn_norm", "ffn_norm", "gain") \
                or leaf.startswith("qk_gain"):
            a = 1.0 + 0.1 * rng.normal(size=(r, c))
        elif leaf == "router_bias":  # balancing state; small and non-trivial for parity
            a = 0.05 * rng.normal(size=(r, c))
        elif leaf.startswith("b"):
            a = 0.1 * rng.normal(size=(r, c))
        else:
            if init == "spec":
                std = 0.02
                if leaf in ("wo", "w_down"):
                    std /= np.sqrt(2.0 * cfg.layers)
            else:
                std = 1.0 / np.sqrt(r)
            a = rng.normal(0.0, std, size=(r, c))
        out[name] = bf16_round(a.astype(np.float32))
    return out
