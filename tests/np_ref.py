# SPDX-License-Identifier: Apache-2.0
"""Independent numpy fp64 restatement of the SORT forward (second oracle).

Written separately from oracle/sort_oracle.cpp so the two can cross-check each
other ("a torch-fp64 re-implementation as an
independent cross-check"). Vectorised numpy, small cases only.
"""
from __future__ import annotations

import numpy as np

from paper_2603_03988_b200.config import ROLE_BOS, ROLE_CAND, ROLE_HIST, ROLE_PROF, ROLE_SEP


def rmsnorm(x, g, eps=1e-6):
    inv = 1.0 / np.sqrt((x * x).mean(axis=-1, keepdims=True) + eps)
    return x * inv * np.asarray(g).reshape(-1)


def rope(x, pos, theta=10000.0):
    d = x.shape[-1]
    j = np.arange(d // 2)
    freq = theta ** (-2.0 * j / d)
    ang = np.asarray(pos, np.float64)[:, None] * freq[None, :]
    c, s = np.cos(ang), np.sin(ang)
    x0, x1 = x[:, 0::2], x[:, 1::2]
    out = np.empty_like(x)
    out[:, 0::2] = c * x0 - s * x1
    out[:, 1::2] = s * x0 + c * x1
    return out


def sigmoid(x):
    return np.where(x >= 0, 1.0 / (1.0 + np.exp(-np.abs(x))), np.exp(-np.abs(x)) / (1.0 + np.exp(-np.abs(x))))


def mask_np(roles, pos, query_rows, W, F):
    roles = np.asarray(roles)
    pos = np.asarray(pos)
    cand = roles == ROLE_CAND
    prefix = pos[cand][0] if cand.any() else pos.max() + 1
    lq, lkv = len(query_rows), len(roles)
    vis = np.zeros((lq, lkv), np.uint8)
    c = np.arange(lkv)
    for r, qi in enumerate(query_rows):
        causal = c <= qi
        if cand[qi]:
            ok = causal & (~cand | (c == qi))
        else:
            ok = causal & ~cand
            if W != -1 and pos[qi] < prefix - F:
                ok &= (pos >= pos[qi] - W + 1) & (pos <= pos[qi])
        vis[r] = ok
    return vis


def attention_layer(P, l, cfg, xn, query_rows, vis, pos):
    d, h = cfg.model_dim, cfg.heads
    dk = d // h
    xq = xn[query_rows]
    pq = np.asarray(pos)[query_rows]
    q_raw, k_raw, v = xq @ P[f"attn.{l}.wq"], xn @ P[f"attn.{l}.wk"], xn @ P[f"attn.{l}.wv"]
    out = np.zeros((len(query_rows), d))
    for i in range(h):
        sl = slice(i * dk, (i + 1) * dk)
        q, k = q_raw[:, sl], k_raw[:, sl]
        if cfg.qknorm:
            q = rmsnorm(q, P[f"attn.{l}.qk_gain_q"][i])
            k = rmsnorm(k, P[f"attn.{l}.qk_gain_k"][i])
        q, k = rope(q, pq, cfg.rope_theta), rope(k, pos, cfg.rope_theta)
        s = (q @ k.T) / np.sqrt(dk)
        s = np.where(vis.astype(bool), s, -np.inf)
        s = s - s.max(axis=1, keepdims=True)
        e = np.exp(s)
        a = e / e.sum(axis=1, keepdims=True)
        out[:, sl] = a @ v[:, sl]
    if cfg.gate:
        out = sigmoid(xq @ P[f"attn.{l}.wg"]) * out
    return out @ P[f"attn.{l}.wo"]


def tokenize(P, cfg, batch, b=0):
    H, N = cfg.n_hist, cfg.n_cand
    d = cfg.model_dim
    delta = np.maximum(batch["req_ts"][b] - batch["hist_ts"][b], 0)
    tb = np.minimum(np.floor(np.log2(1.0 + delta.astype(np.float64))).astype(np.int64),
                    cfg.n_time_buckets - 1)
    hcat = np.concatenate([P["tok.item_table"][batch["hist_item"][b]],
                           P["tok.action_table"][batch["hist_action"][b]],
                           P["tok.scene_table"][batch["hist_scene"][b]],
                           P["tok.time_table"][tb]], axis=1).astype(np.float64)
    hist = rmsnorm(hcat @ P["tok.w_hist"] + P["tok.b_hist"], P["tok.g_hist"])
    pcat = np.stack([P[f"tok.profile_table.{f}"][batch["profile"][b][f]]
                     for f in range(cfg.n_prof)]).astype(np.float64)
    prof = rmsnorm(pcat @ P["tok.w_prof"] + P["tok.b_prof"], P["tok.g_prof"])
    ccat = P["tok.item_table"][batch["cand_item"][b]].astype(np.float64)
    cand = rmsnorm(ccat @ P["tok.w_cand"] + P["tok.b_cand"], P["tok.g_cand"])
    sp = P["tok.special"].astype(np.float64)
    rows, roles = [], []
    if cfg.special_tokens:
        rows.append(sp[0:1]); roles.append(ROLE_BOS)
    rows.append(hist); roles += [ROLE_HIST] * H
    if cfg.special_tokens:
        rows.append(sp[1:2]); roles.append(ROLE_SEP)
    rows.append(prof); roles += [ROLE_PROF] * cfg.n_prof
    if cfg.special_tokens:
        rows.append(sp[2:3]); roles.append(ROLE_SEP)
    rows.append(cand); roles += [ROLE_CAND] * N
    x = np.concatenate(rows, axis=0)
    L = x.shape[0]
    pos = np.concatenate([np.arange(L - N), np.full(N, L - N)])
    return x, np.asarray(roles), pos, tb


def retained(roles, keep, keep_specials):
    roles = np.asarray(roles)
    nc = int((roles != ROLE_CAND).sum())
    drop = nc - min(keep, nc)
    out, seen = [], 0
    for i, r in enumerate(roles):
        if r == ROLE_CAND:
            out.append(i)
            continue
        ins = seen >= drop
        seen += 1
        if ins or (keep_specials and r in (ROLE_BOS, ROLE_SEP)):
            out.append(i)
    return out


def swish(x):
    return x * sigmoid(x)


def model_forward(P, cfg, batch, b=0):
    P = {k: np.asarray(v, np.float64) for k, v in P.items()}
    x, roles, pos, _ = tokenize(P, cfg, batch, b)
    for l, keep in enumerate(cfg.keep_schedule()):
        qr = retained(roles, keep, cfg.keep_specials)
        vis = mask_np(roles, pos, qr, cfg.local_window, cfg.full_suffix)
        xn = rmsnorm(x, P[f"block.{l}.attn_norm"])
        x = x[qr] + attention_layer(P, l, cfg, xn, qr, vis, pos)
        roles, pos = roles[qr], pos[qr]
        xf = rmsnorm(x, P[f"block.{l}.ffn_norm"])
        x = x + (swish(xf @ P[f"ffn.{l}.w_gate"]) * (xf @ P[f"ffn.{l}.w_up"])) @ P[f"ffn.{l}.w_down"]
    xc = rmsnorm(x[roles == ROLE_CAND], P["final_norm.gain"])
    hid = np.maximum(xc @ P["head.w1"] + P["head.b1"], 0.0)
    logits = hid @ P["head.w2"] + P["head.b2"]
    return sigmoid(logits), logits
