# SPDX-License-Identifier: Apache-2.0
"""Host-side structural plan of a SORT forward: token roles/positions, per-layer
retained rows and the compact mask form, in Python.

This is the Python mirror of the C++ planner inside libsort_b200.so
(csrc/plan.cpp); both restate the reference's integer rules:

* sequence layout / positions: Tokenizer::tokenize_sample (tokenizer.cpp:170-237)
* retained rows: retained_rows (mask.cpp:132-154)
* mask: build_mask (mask.cpp:14-76), stored per query row as one contiguous
  non-candidate kv interval [lo, hi] plus an optional ``self`` column for
  candidate rows. Because retained rows keep their
  order and ORIGINAL positions, positions are strictly increasing over the
  non-candidate kv rows, so the window test on positions becomes a
  lower_bound on the kv index.
"""
from __future__ import annotations

import bisect
import dataclasses
from typing import List

import numpy as np

from .config import ROLE_BOS, ROLE_CAND, ROLE_HIST, ROLE_PROF, ROLE_SEP, SortConfig


def sequence_structure(cfg: SortConfig):
    if cfg.pretrain:  # [BOS; clicks] (tokenize_click_sequence, tokenizer.cpp:243-256)
        return [ROLE_BOS] + [ROLE_HIST] * cfg.n_hist, list(range(1 + cfg.n_hist))
    roles: List[int] = []
    if cfg.special_tokens:
        roles.append(ROLE_BOS)
    roles += [ROLE_HIST] * cfg.n_hist
    if cfg.special_tokens:
        roles.append(ROLE_SEP)
    roles += [ROLE_PROF] * cfg.n_prof
    if cfg.special_tokens:
        roles.append(ROLE_SEP)
    roles += [ROLE_CAND] * cfg.n_cand
    L = len(roles)
    prefix = L - cfg.n_cand
    pos = list(range(prefix)) + [prefix] * cfg.n_cand
    return roles, pos


def retained_rows(roles: List[int], keep: int, keep_specials: bool) -> List[int]:
    non_cand = sum(1 for r in roles if r != ROLE_CAND)
    drop = non_cand - min(keep, non_cand)
    out, seen = [], 0
    for i, r in enumerate(roles):
        if r == ROLE_CAND:
            out.append(i)
            continue
        in_suffix = seen >= drop
        seen += 1
        if in_suffix or (keep_specials and r in (ROLE_BOS, ROLE_SEP)):
            out.append(i)
    return out


def mask_intervals(roles, pos, query_rows, window: int, full_suffix: int):
    """Per query row: (lo, hi, self) in kv-index space; self = -1 for non-candidates."""
    cands = [i for i, r in enumerate(roles) if r == ROLE_CAND]
    prefix_positions = pos[cands[0]] if cands else max(p + 1 for p in pos)
    nc_idx = [i for i, r in enumerate(roles) if r != ROLE_CAND]
    nc_pos = [pos[i] for i in nc_idx]
    lo, hi, self_ = [], [], []
    for qi in query_rows:
        q_pos = pos[qi]
        if roles[qi] == ROLE_CAND:
            # all non-candidate kv rows before it (candidates form the suffix) + itself
            k = bisect.bisect_right(nc_idx, qi)
            lo.append(nc_idx[0] if k else 0)
            hi.append(nc_idx[k - 1] if k else -1)
            self_.append(qi)
            continue
        k = bisect.bisect_right(nc_idx, qi)  # non-candidates with kv index <= qi
        windowed = window != -1 and q_pos < prefix_positions - full_suffix
        first = 0
        if windowed:
            first = bisect.bisect_left(nc_pos, q_pos - window + 1, 0, k)
        lo.append(nc_idx[first])
        hi.append(nc_idx[k - 1])
        self_.append(-1)
    return np.array(lo, np.int32), np.array(hi, np.int32), np.array(self_, np.int32)


@dataclasses.dataclass
class LayerPlan:
    l_q: int
    l_kv: int
    query_rows: np.ndarray
    lo: np.ndarray
    hi: np.ndarray
    self_idx: np.ndarray
    roles_kv: np.ndarray
    pos_kv: np.ndarray

    @property
    def visible(self) -> int:
        n = np.maximum(self.hi - self.lo + 1, 0).sum()
        return int(n + (self.self_idx >= 0).sum())

    def dense(self) -> np.ndarray:
        vis = np.zeros((self.l_q, self.l_kv), np.uint8)
        c = np.arange(self.l_kv)
        for r in range(self.l_q):
            vis[r] = (c >= self.lo[r]) & (c <= self.hi[r])
            if self.self_idx[r] >= 0:
                vis[r, self.self_idx[r]] = 1
        return vis


def layer_plans(cfg: SortConfig) -> List[LayerPlan]:
    roles, pos = sequence_structure(cfg)
    out = []
    for keep in cfg.keep_schedule():
        qr = retained_rows(roles, keep, cfg.keep_specials)
        lo, hi, se = mask_intervals(roles, pos, qr, cfg.local_window, cfg.full_suffix)
        out.append(LayerPlan(len(qr), len(roles), np.array(qr, np.int32), lo, hi, se,
                             np.array(roles, np.int32), np.array(pos, np.int32)))
        roles = [roles[i] for i in qr]
        pos = [pos[i] for i in qr]
    return out
