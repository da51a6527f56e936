# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY -- ctypes binding of the CPU oracle (liboracle.so).

The oracle is the fp64 restatement of the reference hot path (see
sort_oracle.h). Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / --impl reference legs may import this module, and only as the
checker / the timed CPU reference -- never as the product path.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from typing import Dict, List, Optional, Sequence

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")
_lib = None

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f64p = C.POINTER(C.c_double)
f32p = C.POINTER(C.c_float)
u8p = C.POINTER(C.c_uint8)


class OrModelCfg(C.Structure):
    _fields_ = [
        ("model_dim", C.c_int), ("item_dim", C.c_int), ("action_dim", C.c_int),
        ("scene_dim", C.c_int), ("time_dim", C.c_int), ("profile_dim", C.c_int),
        ("n_items", C.c_int), ("n_actions", C.c_int), ("n_scenes", C.c_int),
        ("n_time_buckets", C.c_int), ("n_profile_fields", C.c_int),
        ("profile_vocab", C.c_int * 16), ("special_tokens", C.c_int),
        ("layers", C.c_int), ("heads", C.c_int), ("ffn_dim", C.c_int),
        ("qknorm", C.c_int), ("gate", C.c_int), ("rope_theta", C.c_double),
        ("local_window", C.c_int), ("full_suffix", C.c_int), ("keep", C.c_int * 64),
        ("keep_specials", C.c_int), ("head_hidden", C.c_int),
        ("moe_experts", C.c_int), ("moe_topk", C.c_int), ("moe_shared", C.c_int),
        ("moe_ffn_dim", C.c_int),
    ]


class OrSample(C.Structure):
    _fields_ = [
        ("timestamp", C.c_int64), ("n_hist", C.c_int), ("hist_item", i32p),
        ("hist_action", i32p), ("hist_scene", i32p), ("hist_ts", i64p), ("n_prof", C.c_int),
        ("profile", i32p), ("n_cand", C.c_int), ("cand_item", i32p),
    ]


class OracleError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


def build() -> str:
    src = os.path.join(_HERE, "sort_oracle.cpp")
    if (not os.path.exists(_LIB_PATH)) or os.path.getmtime(_LIB_PATH) < os.path.getmtime(src):
        subprocess.check_call(["make", "-s", "-C", _HERE])
    return _LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            build()
        L = C.CDLL(_LIB_PATH)
        L.oracle_last_error.restype = C.c_char_p
        L.oracle_mask_visible_count.restype = C.c_int64
        L.oracle_model_create.argtypes = [C.POINTER(OrModelCfg), C.POINTER(C.c_void_p)]
        L.oracle_model_destroy.argtypes = [C.c_void_p]
        L.oracle_model_set_param.argtypes = [C.c_void_p, C.c_char_p, f64p, C.c_int, C.c_int]
        L.oracle_tokenize.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, i32p, i32p, i32p,
                                      i32p, i32p]
        L.oracle_model_forward.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, f64p]
        L.oracle_model_forward_batch.argtypes = [C.c_void_p, C.POINTER(OrSample), C.c_int,
                                                 C.c_int, f64p]
        L.oracle_model_layer_meta.argtypes = [C.c_void_p, C.POINTER(OrSample), i32p, i64p, i32p,
                                              i32p]
        L.oracle_attention_forward.argtypes = [C.c_void_p, C.c_int, f64p, C.c_int, i32p, C.c_int,
                                               u8p, i32p, f64p]
        L.oracle_time_bucket.argtypes = [C.c_int64, C.c_int]
        L.oracle_model_backward.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, f64p,
                                            C.POINTER(C.c_void_p)]
        L.oracle_grads_get.argtypes = [C.c_void_p, C.c_char_p, f64p, i32p, i32p]
        L.oracle_grads_destroy.argtypes = [C.c_void_p]
        L.oracle_model_forward_moe.argtypes = [C.c_void_p, C.POINTER(OrSample), i32p, f64p, f64p,
                                               i32p, f64p]
        L.oracle_moe_route.argtypes = [f64p, C.c_int, C.c_int, C.c_int, C.c_int, f64p, f64p, i32p,
                                       f64p, f64p]
        L.oracle_moe_ffn.argtypes = [f64p, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int,
                                     f64p, f64p, f64p, f64p, f64p, i32p, f64p, i32p, f64p]
        L.oracle_moe_update_bias.argtypes = [i64p, C.c_int, C.c_double, f64p]
        L.oracle_pretrain_forward.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, f64p, f64p]
        L.oracle_tokenize_clicks.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, i32p]
        L.oracle_attention_backward.argtypes = [C.c_void_p, C.c_int, f64p, C.c_int, i32p, C.c_int, u8p, i32p,
                                                f64p, f64p, C.POINTER(C.c_void_p)]
        L.oracle_tokenizer_backward.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, C.POINTER(C.c_void_p)]
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise OracleError(status, lib().oracle_last_error().decode())


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


# ------------------------------------------------------------------ free functions
def time_bucket(delta: int, n_buckets: int) -> int:
    return lib().oracle_time_bucket(int(delta), int(n_buckets))


def build_mask(l_q: int, roles: Sequence[int], pos: Sequence[int], local_window: int,
               full_suffix: int, query_rows: Optional[Sequence[int]] = None) -> np.ndarray:
    roles = np.ascontiguousarray(roles, dtype=np.int32)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    l_kv = len(roles)
    out = np.zeros((l_q, l_kv), dtype=np.uint8)
    qr = None if query_rows is None else np.ascontiguousarray(query_rows, dtype=np.int32)
    _check(lib().oracle_build_mask(l_q, l_kv, local_window, full_suffix, _p(roles, i32p),
                                   _p(pos, i32p), None if qr is None else _p(qr, i32p),
                                   _p(out, u8p)))
    return out


def geometric_schedule(prefix_len: int, depth: int, target: int) -> List[int]:
    out = np.zeros(max(depth, 1), dtype=np.int32)
    _check(lib().oracle_geometric_schedule(prefix_len, depth, target, _p(out, i32p)))
    return out.tolist()


def retained_rows(roles: Sequence[int], keep: int, keep_specials: bool) -> List[int]:
    roles = np.ascontiguousarray(roles, dtype=np.int32)
    out = np.zeros(len(roles), dtype=np.int32)
    n = C.c_int(0)
    _check(lib().oracle_retained_rows(_p(roles, i32p), len(roles), keep, int(keep_specials),
                                      _p(out, i32p), C.byref(n)))
    return out[: n.value].tolist()


def prune_queries(x: np.ndarray, n: int) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros((n, x.shape[1]))
    _check(lib().oracle_prune_queries(_p(x, f64p), x.shape[0], x.shape[1], n, _p(out, f64p)))
    return out


def rmsnorm(x: np.ndarray, gain: np.ndarray) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    g = np.ascontiguousarray(gain, dtype=np.float64).reshape(-1)
    y = np.zeros_like(x)
    _check(lib().oracle_rmsnorm_forward(_p(x, f64p), x.shape[0], x.shape[1], _p(g, f64p),
                                        _p(y, f64p), None))
    return y


def rope(x: np.ndarray, pos: Sequence[int], theta: float = 10000.0, inverse=False) -> np.ndarray:
    x = np.ascontiguousarray(x, dtype=np.float64)
    p = np.ascontiguousarray(pos, dtype=np.int32)
    y = np.zeros_like(x)
    lib().oracle_rope_apply.argtypes = [f64p, C.c_int, C.c_int, i32p, C.c_double, C.c_int, f64p]
    _check(lib().oracle_rope_apply(_p(x, f64p), x.shape[0], x.shape[1], _p(p, i32p), theta,
                                   int(inverse), _p(y, f64p)))
    return y


def dense_attention(q, k, v, mask, dtype=np.float64) -> np.ndarray:
    q, k, v, mask = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v, mask))
    out = np.zeros((q.shape[0], v.shape[1]), dtype=dtype)
    fn = lib().oracle_dense_masked_attention_f64 if dtype == np.float64 else \
        lib().oracle_dense_masked_attention_f32
    t = f64p if dtype == np.float64 else f32p
    _check(fn(_p(q, t), _p(k, t), _p(v, t), _p(mask, t), q.shape[0], k.shape[0], q.shape[1],
              v.shape[1], _p(out, t)))
    return out


def blockwise_attention(q, k, v, mask, block=16, dtype=np.float64):
    q, k, v, mask = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v, mask))
    out = np.zeros((q.shape[0], v.shape[1]), dtype=dtype)
    sk, tot = C.c_int64(0), C.c_int64(0)
    fn = lib().oracle_blockwise_masked_attention_f64 if dtype == np.float64 else \
        lib().oracle_blockwise_masked_attention_f32
    t = f64p if dtype == np.float64 else f32p
    _check(fn(_p(q, t), _p(k, t), _p(v, t), _p(mask, t), q.shape[0], k.shape[0], q.shape[1],
              v.shape[1], block, _p(out, t), C.byref(sk), C.byref(tot)))
    return out, sk.value, tot.value


def swishglu(x, w_gate, w_up, w_down) -> np.ndarray:
    x, wg, wu, wd = (np.ascontiguousarray(a, dtype=np.float64) for a in (x, w_gate, w_up, w_down))
    out = np.zeros((x.shape[0], wd.shape[1]))
    _check(lib().oracle_swishglu(_p(x, f64p), x.shape[0], x.shape[1], wg.shape[1], _p(wg, f64p),
                                 _p(wu, f64p), _p(wd, f64p), _p(out, f64p)))
    return out


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


def moe_route(x, router, bias, k: int):
    """route_topk, DeepSeek style: (sel [rows, k], w [rows, k], margin [rows])."""
    x, router = _f64(x), _f64(router)
    E = router.shape[1]
    b = _f64(np.zeros(E) if bias is None else bias).reshape(-1)
    sel = np.zeros((x.shape[0], k), np.int32)
    w = np.zeros((x.shape[0], k))
    mg = np.zeros(x.shape[0])
    _check(lib().oracle_moe_route(_p(x, f64p), x.shape[0], x.shape[1], E, k, _p(router, f64p),
                                  _p(b, f64p), _p(sel, i32p), _p(w, f64p), _p(mg, f64p)))
    return sel, w, mg


def moe_ffn(x, router, bias, k: int, w_gate, w_up, w_down, shared: int = 0, forced=None):
    """moe_forward. w_gate/w_up [E+shared, d, m], w_down [E+shared, m, d],
    shared expert last. Returns (out [rows, d], sel [rows, k], w [rows, k])."""
    x, router = _f64(x), _f64(router)
    E = router.shape[1]
    wg, wu, wd = _f64(w_gate), _f64(w_up), _f64(w_down)
    b = _f64(np.zeros(E) if bias is None else bias).reshape(-1)
    rows, d = x.shape
    m = wg.shape[2]
    out = np.zeros((rows, d))
    sel = np.zeros((rows, k), np.int32)
    w = np.zeros((rows, k))
    fp = None
    if forced is not None:
        forced = np.ascontiguousarray(forced, dtype=np.int32)
        fp = _p(forced, i32p)
    _check(lib().oracle_moe_ffn(_p(x, f64p), rows, d, m, E, k, shared, _p(router, f64p), _p(b, f64p),
                                _p(wg, f64p), _p(wu, f64p), _p(wd, f64p), fp, _p(out, f64p),
                                _p(sel, i32p), _p(w, f64p)))
    return out, sel, w


def moe_update_bias(load, bias, gamma: float = 1e-3) -> np.ndarray:
    """update_balance, DeepSeek style: returns the new bias vector."""
    ld = np.ascontiguousarray(load, dtype=np.int64)
    b = _f64(bias).copy()
    _check(lib().oracle_moe_update_bias(_p(ld, i64p), len(ld), gamma, _p(b, f64p)))
    return b


# ------------------------------------------------------------------ model
class _SampleHold:
    """Keeps the numpy buffers alive while an OrSample points into them."""

    def __init__(self, batch: Dict[str, np.ndarray], b: int):
        self.arrs = {
            "hist_item": np.ascontiguousarray(batch["hist_item"][b], dtype=np.int32),
            "hist_action": np.ascontiguousarray(batch["hist_action"][b], dtype=np.int32),
            "hist_scene": np.ascontiguousarray(batch["hist_scene"][b], dtype=np.int32),
            "hist_ts": np.ascontiguousarray(batch["hist_ts"][b], dtype=np.int64),
            "profile": np.ascontiguousarray(batch["profile"][b], dtype=np.int32),
            "cand_item": np.ascontiguousarray(batch["cand_item"][b], dtype=np.int32),
        }
        a = self.arrs
        self.s = OrSample(int(batch["req_ts"][b]), len(a["hist_item"]), _p(a["hist_item"], i32p),
                          _p(a["hist_action"], i32p), _p(a["hist_scene"], i32p),
                          _p(a["hist_ts"], i64p), len(a["profile"]), _p(a["profile"], i32p),
                          len(a["cand_item"]), _p(a["cand_item"], i32p))


def or_cfg(cfg) -> OrModelCfg:
    """SortConfig -> the C struct both liboracle.so and oracle/_ref/libref.so take."""
    c = OrModelCfg()
    c.model_dim, c.item_dim, c.action_dim = cfg.model_dim, cfg.item_dim, cfg.action_dim
    c.scene_dim, c.time_dim, c.profile_dim = cfg.scene_dim, cfg.time_dim, cfg.profile_dim
    c.n_items, c.n_actions, c.n_scenes = cfg.n_items, cfg.n_actions, cfg.n_scenes
    c.n_time_buckets, c.n_profile_fields = cfg.n_time_buckets, len(cfg.profile_vocab)
    for i, v in enumerate(cfg.profile_vocab):
        c.profile_vocab[i] = v
    c.special_tokens = int(cfg.special_tokens)
    c.layers, c.heads, c.ffn_dim = cfg.layers, cfg.heads, cfg.ffn_dim
    c.qknorm, c.gate, c.rope_theta = int(cfg.qknorm), int(cfg.gate), cfg.rope_theta
    c.local_window, c.full_suffix = cfg.local_window, cfg.full_suffix
    for i, k in enumerate(cfg.keep_schedule()):
        c.keep[i] = k
    c.keep_specials, c.head_hidden = int(cfg.keep_specials), cfg.head_hidden
    c.moe_experts = getattr(cfg, "moe_experts", 0)
    c.moe_topk = getattr(cfg, "moe_topk", 1)
    c.moe_shared = getattr(cfg, "moe_shared", 0)
    c.moe_ffn_dim = getattr(cfg, "moe_ffn_dim", 0)
    return c


class OracleModel:
    def __init__(self, cfg, params: Dict[str, np.ndarray]):
        c = or_cfg(cfg)
        self.cfg = cfg
        h = C.c_void_p()
        _check(lib().oracle_model_create(C.byref(c), C.byref(h)))
        self.h = h
        for name, a in params.items():
            a64 = np.ascontiguousarray(a, dtype=np.float64)
            _check(lib().oracle_model_set_param(self.h, name.encode(), _p(a64, f64p),
                                                a64.shape[0], a64.shape[1]))

    def set_item_trainable(self, trainable: bool = True) -> None:
        _check(lib().oracle_model_set_item_trainable(self.h, int(trainable)))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.oracle_model_destroy(self.h)
            self.h = None

    def tokenize(self, batch, b: int = 0):
        hold = _SampleHold(batch, b)
        cfg = self.cfg
        L = (3 if cfg.special_tokens else 0) + hold.s.n_hist + hold.s.n_prof + hold.s.n_cand
        tokens = np.zeros((L, cfg.model_dim))
        pos, roles, cidx = (np.zeros(L, np.int32) for _ in range(3))
        ht = np.zeros(max(hold.s.n_hist, 1), np.int32)
        n = C.c_int(0)
        _check(lib().oracle_tokenize(self.h, C.byref(hold.s), _p(tokens, f64p), _p(pos, i32p),
                                     _p(roles, i32p), _p(cidx, i32p), _p(ht, i32p), C.byref(n)))
        return {"tokens": tokens, "position_ids": pos, "roles": roles, "candidate_index": cidx,
                "hist_time": ht[: hold.s.n_hist]}

    def forward(self, batch, b: int = 0):
        hold = _SampleHold(batch, b)
        n = hold.s.n_cand
        probs, logits = np.zeros((n, 3)), np.zeros((n, 3))
        _check(lib().oracle_model_forward(self.h, C.byref(hold.s), _p(probs, f64p),
                                          _p(logits, f64p)))
        return probs, logits

    def tokenize_clicks(self, batch, b: int = 0):
        """tokenize_click_sequence (tokenizer.cpp:240-284) of sequence b's hist_* clicks."""
        hold = _SampleHold(batch, b)
        n = hold.s.n_hist
        tokens = np.zeros((1 + n, self.cfg.model_dim))
        ht = np.zeros(n, np.int32)
        _check(lib().oracle_tokenize_clicks(self.h, C.byref(hold.s), _p(tokens, f64p), _p(ht, i32p)))
        return tokens, ht

    def pretrain_forward(self, batch, b: int = 0):
        """pretrain_forward: (lse [n], target logit [n], h [1 + n, item_dim])."""
        hold = _SampleHold(batch, b)
        n = hold.s.n_hist
        lse, tgt = np.zeros(n), np.zeros(n)
        hp = np.zeros((1 + n, self.cfg.item_dim))
        _check(lib().oracle_pretrain_forward(self.h, C.byref(hold.s), _p(lse, f64p), _p(tgt, f64p),
                                             _p(hp, f64p)))
        return lse, tgt, hp

    def pretrain_backward(self, batch, b: int, scale: float, names):
        """fp64 pre-training backward of sequence b: gradients of scale * sum_t CE_t for the
        requested names (None if off the path) and sum_t CE_t."""
        hold = _SampleHold(batch, b)
        ce = C.c_double(0.0)
        g = C.c_void_p()
        lib().oracle_pretrain_backward.argtypes = [C.c_void_p, C.c_void_p, C.c_double, C.POINTER(C.c_double),
                                                   C.POINTER(C.c_void_p)]
        _check(lib().oracle_pretrain_backward(self.h, C.byref(hold.s), scale, C.byref(ce), C.byref(g)))
        return self._grads(g, names), ce.value

    def forward_moe(self, batch, b: int = 0, forced=None):
        """Forward with MoE routing control: forced = list (per layer) of [l_q, k] expert ids or
        None. Returns (probs, logits, sel per layer, margin per layer)."""
        hold = _SampleHold(batch, b)
        n = hold.s.n_cand
        lq = self.layer_meta(batch, b)["l_q"]
        k = self.cfg.moe_topk
        tot = int(sum(lq))
        probs, logits = np.zeros((n, 3)), np.zeros((n, 3))
        sel = np.zeros(tot * k, np.int32)
        mg = np.zeros(tot)
        fp = None
        if forced is not None:
            fa = np.ascontiguousarray(np.concatenate([np.asarray(f, np.int32).reshape(-1) for f in forced]))
            assert fa.size == tot * k
            fp = _p(fa, i32p)
        _check(lib().oracle_model_forward_moe(self.h, C.byref(hold.s), fp, _p(probs, f64p),
                                              _p(logits, f64p), _p(sel, i32p), _p(mg, f64p)))
        sels, mgs, o = [], [], 0
        for q in lq:
            sels.append(sel[o * k:(o + q) * k].reshape(q, k))
            mgs.append(mg[o:o + q])
            o += q
        return probs, logits, sels, mgs

    def forward_batch(self, batch, threads: int = 1, limit: Optional[int] = None) -> np.ndarray:
        B = batch["req_ts"].shape[0] if limit is None else limit
        holds = [_SampleHold(batch, b) for b in range(B)]
        arr = (OrSample * B)(*[h.s for h in holds])
        total = sum(h.s.n_cand for h in holds)
        probs = np.zeros((total, 3))
        _check(lib().oracle_model_forward_batch(self.h, arr, B, threads, _p(probs, f64p)))
        return probs

    def layer_meta(self, batch, b: int = 0):
        hold = _SampleHold(batch, b)
        nl = self.cfg.layers
        lq = np.zeros(nl, np.int32)
        vis = np.zeros(nl, np.int64)
        L = (3 if self.cfg.special_tokens else 0) + hold.s.n_hist + hold.s.n_prof + hold.s.n_cand
        qr = np.zeros(L * nl, np.int32)
        tot = C.c_int(0)
        _check(lib().oracle_model_layer_meta(self.h, C.byref(hold.s), _p(lq, i32p), _p(vis, i64p),
                                             _p(qr, i32p), C.byref(tot)))
        rows, off = [], 0
        for l in range(nl):
            rows.append(qr[off: off + lq[l]].tolist())
            off += lq[l]
        return {"l_q": lq.tolist(), "visible": vis.tolist(), "query_rows": rows}

    def attention(self, layer: int, xn: np.ndarray, query_rows, visible: np.ndarray, pos):
        xn = np.ascontiguousarray(xn, dtype=np.float64)
        qr = np.ascontiguousarray(query_rows, dtype=np.int32)
        vis = np.ascontiguousarray(visible, dtype=np.uint8)
        p = np.ascontiguousarray(pos, dtype=np.int32)
        out = np.zeros((len(qr), self.cfg.model_dim))
        _check(lib().oracle_attention_forward(self.h, layer, _p(xn, f64p), xn.shape[0],
                                              _p(qr, i32p), len(qr), _p(vis, u8p), _p(p, i32p),
                                              _p(out, f64p)))
        return out

    def _grads(self, g, names):
        out = {}
        try:
            for name in names:
                r, c = C.c_int32(0), C.c_int32(0)
                _check(lib().oracle_grads_get(g, name.encode(), None, C.byref(r), C.byref(c)))
                a = np.zeros((max(r.value, 1), max(c.value, 1)))
                if r.value:
                    _check(lib().oracle_grads_get(g, name.encode(), _p(a, f64p), None, None))
                    out[name] = a
                else:
                    out[name] = None
        finally:
            lib().oracle_grads_destroy(g)
        return out

    def attention_backward(self, layer, xn, query_rows, visible, pos, dout, names):
        """(dxn, {name: grad}) of the restated AttentionLayer::backward for layer alone."""
        xn = np.ascontiguousarray(xn, dtype=np.float64)
        dout = np.ascontiguousarray(dout, dtype=np.float64)
        qr = np.ascontiguousarray(query_rows, dtype=np.int32)
        vis = np.ascontiguousarray(visible, dtype=np.uint8)
        p = np.ascontiguousarray(pos, dtype=np.int32)
        dxn = np.zeros_like(xn)
        g = C.c_void_p()
        _check(lib().oracle_attention_backward(self.h, layer, _p(xn, f64p), xn.shape[0], _p(qr, i32p), len(qr),
                                               _p(vis, u8p), _p(p, i32p), _p(dout, f64p), _p(dxn, f64p),
                                               C.byref(g)))
        return dxn, self._grads(g, names)

    def tokenizer_backward(self, batch, b: int, dtokens, names):
        hold = _SampleHold(batch, b)
        dt = np.ascontiguousarray(dtokens, dtype=np.float64)
        g = C.c_void_p()
        _check(lib().oracle_tokenizer_backward(self.h, C.byref(hold.s), _p(dt, f64p), C.byref(g)))
        return self._grads(g, names)

    def backward(self, batch, b: int, dlogits: np.ndarray, names):
        """fp64 backward of forward(batch, b) given dL/dlogits [n_cand, 3]: returns
        ({name: gradient} for the requested parameter names, dtokens [L, d])."""
        hold = _SampleHold(batch, b)
        cfg = self.cfg
        L = (3 if cfg.special_tokens else 0) + hold.s.n_hist + hold.s.n_prof + hold.s.n_cand
        dz = np.ascontiguousarray(dlogits, dtype=np.float64)
        dtok = np.zeros((L, cfg.model_dim))
        g = C.c_void_p()
        _check(lib().oracle_model_backward(self.h, C.byref(hold.s), _p(dz, f64p), _p(dtok, f64p),
                                           C.byref(g)))
        out = {}
        try:
            for name in names:
                r, c = C.c_int32(0), C.c_int32(0)
                _check(lib().oracle_grads_get(g, name.encode(), None, C.byref(r), C.byref(c)))
                a = np.zeros((max(r.value, 1), max(c.value, 1)))
                if r.value:
                    _check(lib().oracle_grads_get(g, name.encode(), _p(a, f64p), None, None))
                    out[name] = a
                else:
                    out[name] = None
        finally:
            lib().oracle_grads_destroy(g)
        return out, dtok


# ------------------------------------------------------------------ training references (numpy)
def bce_loss(logits: np.ndarray, labels: np.ndarray, weights=(1.0, 0.5, 0.5), eps: float = 1e-7):
    """total_loss: sum_obj w_obj * mean BCE over candidates, eps-clamped logs;
    returns (loss, dL/dlogits)."""
    z = np.asarray(logits, np.float64).reshape(-1, 3)
    y = np.asarray(labels, np.float64).reshape(-1, 3)
    w = np.asarray(weights, np.float64)
    p = 1.0 / (1.0 + np.exp(-z))
    pc = np.clip(p, eps, 1 - eps)
    n = z.shape[0]
    loss = float((w * -(y * np.log(pc) + (1 - y) * np.log(1 - pc))).sum() / n)
    return loss, (w * (p - y) / n).reshape(np.shape(logits))


def adamw(p, g, m, v, t, lr, b1=0.9, b2=0.99, eps=1e-8, wd=0.01):
    """adamw_step: bias-corrected moments, decoupled weight decay. Returns
    (p', m', v')."""
    m = b1 * m + (1 - b1) * g
    v = b2 * v + (1 - b2) * g * g
    mh, vh = m / (1 - b1 ** t), v / (1 - b2 ** t)
    return p - lr * wd * p - lr * mh / (np.sqrt(vh) + eps), m, v
