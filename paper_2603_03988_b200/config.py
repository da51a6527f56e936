# SPDX-License-Identifier: Apache-2.0
"""Model/batch configuration for the SORT block path.

Mirrors the reference's plain config structs -- ``TokenizerConfig``
(tokenizer.hpp:31-56), ``AttentionSettings`` (attention.hpp:13-29),
``MaskSpec`` (mask.hpp:15-31), ``PruneSchedule`` (mask.hpp:48-61) -- plus the
spec-only block stack / head sizes and the fixed batch
geometry the batched GPU path is planned for (all requests of one call share
history length and candidate count).
"""
from __future__ import annotations

import dataclasses
import math
from typing import List, Optional

ROLE_BOS, ROLE_HIST, ROLE_SEP, ROLE_PROF, ROLE_CAND = 0, 1, 2, 3, 4


class ConfigError(ValueError):
    """rankformer::ConfigError (common.hpp:17-21) -- CLI exit code 1."""


class RuntimeFailure(RuntimeError):
    """rankformer::RuntimeFailure (common.hpp:23-27) -- CLI exit code 2."""


def geometric_schedule(prefix_len: int, depth: int, target: int) -> List[int]:
    """make_geometric_schedule (mask.cpp:97-117), evaluated in double exactly as
    the reference does (the raw value 256.499 at geo(1030,4,128) is 0.001 from
    the lround boundary -- SURVEY.md Appendix 11)."""
    if depth < 1:
        raise ConfigError("make_geometric_schedule: depth must be >= 1")
    prefix_len = max(prefix_len, 1)
    final_keep = min(target, prefix_len)
    if depth == 1:
        return [final_keep]
    ratio = final_keep / prefix_len
    keep, prev = [], prefix_len
    for l in range(depth):
        t = l / (depth - 1)
        raw = prefix_len * math.pow(ratio, t)
        k = int(raw)  # lround: half away from zero (raw >= 0 here), exact for raw < 2**52
        if raw - k >= 0.5:
            k += 1
        k = min(max(k, final_keep), prev)
        keep.append(k)
        prev = k
    return keep


@dataclasses.dataclass
class SortConfig:
    # tokenizer (tokenizer.hpp:32-44 defaults)
    model_dim: int = 64
    item_dim: int = 32
    action_dim: int = 8
    scene_dim: int = 8
    time_dim: int = 8
    profile_dim: int = 16
    n_items: int = 5000
    n_actions: int = 3
    n_scenes: int = 4
    n_time_buckets: int = 32
    profile_vocab: List[int] = dataclasses.field(default_factory=lambda: [8, 8, 8])
    special_tokens: bool = True
    # block stack
    heads: int = 4
    layers: int = 2
    ffn_dim: int = 160
    head_hidden: int = 0  # 0 -> model_dim (SPEC.md "Head hidden width d_h = d")
    qknorm: bool = True
    gate: bool = True
    rope_theta: float = 10000.0
    # DeepSeek-style MoE FFN; moe_experts = 0 -> dense SwishGLU
    moe_experts: int = 0
    moe_topk: int = 1
    moe_shared: int = 1
    moe_ffn_dim: int = 0
    # generative pre-training model: click sequences [BOS; clicks]
    pretrain: bool = False
    # mask / pruning
    local_window: int = 32
    full_suffix: int = 128
    keep: Optional[List[int]] = None  # None -> full schedule
    keep_specials: bool = False
    # batch geometry
    n_hist: int = 256
    n_cand: int = 16
    batch: int = 1

    @property
    def head_dim(self) -> int:
        return self.model_dim // self.heads

    @property
    def n_prof(self) -> int:
        return len(self.profile_vocab)

    @property
    def seq_len(self) -> int:
        if self.pretrain:  # [BOS; clicks] (tokenizer.cpp:243)
            return 1 + self.n_hist
        # L = 1 + H + 1 + |U| + 1 + N (tokenizer.cpp:158-159)
        return (3 if self.special_tokens else 0) + self.n_hist + self.n_prof + self.n_cand

    @property
    def prefix_len(self) -> int:
        return self.seq_len - self.n_cand

    def keep_schedule(self) -> List[int]:
        if self.keep is None:
            return [max(self.prefix_len, 1)] * self.layers  # make_full_schedule (mask.cpp:119-123)
        return list(self.keep)

    def validate(self) -> None:
        if self.heads < 1 or self.model_dim % self.heads:
            raise ConfigError("attention: model_dim must be a positive multiple of heads")
        if self.head_dim % 2:
            raise ConfigError("attention: head dim must be even for the rotary transform")
        ks = self.keep_schedule()
        if len(ks) != self.layers:
            raise ConfigError("PruneSchedule: one keep count per layer")
        if any(b > a for a, b in zip(ks, ks[1:])):
            raise ConfigError("PruneSchedule: keep counts must be non-increasing")
        if any(k < 1 for k in ks):
            raise ConfigError("PruneSchedule: keep counts must be >= 1")
        if self.local_window != -1 and self.local_window < 1:
            raise ConfigError("MaskSpec: local_window must be >= 1 or -1 (unbounded)")


def tiny_config(**kw) -> SortConfig:
    """BASELINE.json configs[0]: 2 layers, d=64, 4 heads, 1 request x 256 history + 16 targets,
    local window 32 (the reference defaults: attention.hpp:14-15)."""
    c = SortConfig(model_dim=64, heads=4, layers=2, ffn_dim=160, local_window=32, full_suffix=128,
                   n_hist=256, n_cand=16, batch=1, n_items=5000, keep=None)
    return dataclasses.replace(c, **kw)


def base_config(**kw) -> SortConfig:
    """BASELINE.json configs[1]: SORT-base, 4 layers, d=256, 8 heads, 256 requests x 1024
    history + 64 targets, query pruning after layer 2 (keep = [1030, 1030, 128, 128])."""
    c = SortConfig(model_dim=256, heads=8, layers=4, ffn_dim=640, local_window=256,
                   full_suffix=128, n_hist=1024, n_cand=64, batch=256, n_items=1_000_000)
    c.keep = [c.prefix_len, c.prefix_len, 128, 128]
    return dataclasses.replace(c, **kw)


def base_moe_config(**kw) -> SortConfig:
    """SURVEY.md section 8(f) "next 1": SORT-base with the DeepSeek-style MoE FFN at the paper's
    best sparsity 1/8: 8 routed experts, top-1, one shared expert, expert width
    ffn_dim / 2 = 320 so the activated FFN width (shared + routed) equals the dense 640 (the
    spec's sizing rule)."""
    c = base_config(moe_experts=8, moe_topk=1, moe_shared=1, moe_ffn_dim=320)
    return dataclasses.replace(c, **kw)


def pretrain_config(**kw) -> SortConfig:
    """SURVEY.md section 8(f) "next 4": the SORT-base block stack as a causal next-item model
    over click sequences (no candidates, no local window, no pruning),
    1024 clicks per sequence, 64 sequences, a 65,536-item vocabulary with the full softmax."""
    c = SortConfig(model_dim=256, heads=8, layers=4, ffn_dim=640, local_window=-1, full_suffix=0,
                   n_hist=1024, n_cand=0, profile_vocab=[], batch=64, n_items=65536, pretrain=True)
    return dataclasses.replace(c, **kw)


def large_config(**kw) -> SortConfig:
    """BASELINE.json configs[3]: SORT-large, 12 layers, d=1024, 16 heads, 4096 history,
    W=256, 128 targets, geometric schedule (mask.cpp:97-117)."""
    c = SortConfig(model_dim=1024, heads=16, layers=12, ffn_dim=2560, local_window=256,
                   full_suffix=128, n_hist=4096, n_cand=128, batch=8, n_items=1_000_000)
    c.keep = geometric_schedule(c.prefix_len, c.layers, 128)
    return dataclasses.replace(c, **kw)
