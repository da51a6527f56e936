# SPDX-License-Identifier: Apache-2.0
"""Analytic forward FLOPs per request (SPEC.md:233-241 ``flops_estimate``).

Convention: 2 FLOPs per MAC;
attention counts only VISIBLE mask entries (QK^T and PV: 4*dk per entry per
head); norms, RoPE, softmax exp and biases are not counted.
"""
from __future__ import annotations

from .config import SortConfig
from .plan import layer_plans


def forward_flops(cfg: SortConfig) -> dict:
    d, m, h = cfg.model_dim, cfg.ffn_dim, cfg.heads
    dk = d // h
    dh = cfg.head_hidden or d
    hw = cfg.item_dim + cfg.action_dim + cfg.scene_dim + cfg.time_dim
    tok = 2 * (cfg.n_hist * hw * d + cfg.n_prof * cfg.profile_dim * d + cfg.n_cand * cfg.item_dim * d)
    proj = attn = ffn = 0
    layers = []
    for p in layer_plans(cfg):
        lp = 2 * (3 * p.l_q * d * d + 2 * p.l_kv * d * d)   # Q, G, O on queries; K, V on kv rows
        la = 4 * dk * h * p.visible                          # QK^T + PV over visible entries
        if cfg.moe_experts > 0:  # activated experts only (k routed + shared) + fp32 router
            lf = 2 * 3 * p.l_q * d * cfg.moe_ffn_dim * (cfg.moe_topk + cfg.moe_shared) \
                + 2 * p.l_q * d * cfg.moe_experts
        else:
            lf = 2 * 3 * p.l_q * d * m                       # gate, up, down
        layers.append({"proj": lp, "attn": la, "ffn": lf, "visible_per_head": p.visible,
                       "l_q": p.l_q, "l_kv": p.l_kv})
        proj, attn, ffn = proj + lp, attn + la, ffn + lf
    head = 2 * cfg.n_cand * (d * dh + dh * 3)
    block = proj + attn + ffn
    return {"tokenizer": tok, "proj": proj, "attn": attn, "ffn": ffn, "block": block,
            "head": head, "total": tok + block + head, "layers": layers}


def tokenizer_bytes(cfg: SortConfig, elem_bytes: int = 2) -> int:
    """Algorithmic HBM bytes of the tokenizer per request: the gathered embedding rows, the
    index/timestamp inputs and the written token rows (+ one fp32 row statistic)."""
    gathered = cfg.n_hist * (cfg.item_dim + cfg.action_dim + cfg.scene_dim + cfg.time_dim) \
        + cfg.n_prof * cfg.profile_dim + cfg.n_cand * cfg.item_dim
    idx = cfg.n_hist * (4 + 4 + 4 + 8) + cfg.n_prof * 4 + cfg.n_cand * 4 + 8
    out = cfg.seq_len * (cfg.model_dim * elem_bytes + 4)
    return gathered * elem_bytes + idx + out
