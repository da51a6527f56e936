# SPDX-License-Identifier: Apache-2.0
"""TEST INFRASTRUCTURE ONLY -- ctypes binding of oracle/_ref/libref.so, the REFERENCE's own
mask.cpp / tokenizer.cpp / attention.cpp compiled unmodified against an Eigen-subset shim
(oracle/Makefile, oracle/ref_harness.cpp). tests/ use it to pin the fp64 restatement
(liboracle.so) and the CUDA path to the reference's code; nothing in the product loads it.

`available()` is False when the library was not built (it is built from /root/reference,
which exists in the development container only; the built .so travels to the GPU box)."""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional, Sequence

import numpy as np

from oracle import OrModelCfg, OrSample, _SampleHold, f32p, f64p, i32p, i64p, u8p  # noqa: F401

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "_ref", "libref.so")
_lib = None


class RefError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"[status {status}] {msg}")
        self.status = status


def available() -> bool:
    return os.path.exists(LIB_PATH)


def lib():
    global _lib
    if _lib is None:
        L = C.CDLL(LIB_PATH)
        L.ref_last_error.restype = C.c_char_p
        L.ref_time_bucket.argtypes = [C.c_int64, C.c_int]
        L.ref_build_mask.argtypes = [C.c_int, C.c_int, C.c_int, C.c_int, i32p, i32p, i32p, u8p, i64p]
        L.ref_geometric_schedule.argtypes = [C.c_int, C.c_int, C.c_int, i32p]
        L.ref_full_schedule.argtypes = [C.c_int, C.c_int, i32p]
        L.ref_retained_rows.argtypes = [i32p, C.c_int, C.c_int, C.c_int, i32p, i32p]
        L.ref_prune_queries.argtypes = [f64p, C.c_int, C.c_int, C.c_int, f64p]
        L.ref_rmsnorm_forward.argtypes = [f64p, C.c_int, C.c_int, f64p, f64p, f64p]
        L.ref_rmsnorm_backward.argtypes = [f64p, f64p, C.c_int, C.c_int, f64p, f64p, f64p]
        L.ref_rope_apply.argtypes = [f64p, C.c_int, C.c_int, i32p, C.c_double, C.c_int, f64p]
        for suf, t in (("f64", f64p), ("f32", f32p)):
            getattr(L, f"ref_dense_attention_{suf}").argtypes = [t, t, t, t, C.c_int, C.c_int, C.c_int, C.c_int, t]
            getattr(L, f"ref_blockwise_attention_{suf}").argtypes = [t, t, t, t, C.c_int, C.c_int, C.c_int,
                                                                     C.c_int, C.c_int, t, i64p, i64p]
        L.ref_model_create.argtypes = [C.POINTER(OrModelCfg), C.POINTER(C.c_void_p)]
        L.ref_model_destroy.argtypes = [C.c_void_p]
        L.ref_model_set_param.argtypes = [C.c_void_p, C.c_char_p, f64p, C.c_int, C.c_int]
        L.ref_set_frozen.argtypes = [C.c_void_p, C.c_char_p, C.c_int]
        L.ref_tokenize.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, i32p, i32p, i32p, i32p, i32p]
        L.ref_tokenize_clicks.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, i32p]
        L.ref_tokenizer_backward.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, C.POINTER(C.c_void_p)]
        L.ref_attention_forward.argtypes = [C.c_void_p, C.c_int, f64p, C.c_int, i32p, C.c_int, u8p, i32p, f64p]
        L.ref_attention_backward.argtypes = [C.c_void_p, C.c_int, f64p, C.c_int, i32p, C.c_int, u8p, i32p,
                                             f64p, f64p, C.POINTER(C.c_void_p)]
        L.ref_grads_get.argtypes = [C.c_void_p, C.c_char_p, f64p, i32p, i32p]
        L.ref_grads_destroy.argtypes = [C.c_void_p]
        L.ref_model_forward.argtypes = [C.c_void_p, C.POINTER(OrSample), f64p, f64p]
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status != 0:
        raise RefError(status, lib().ref_last_error().decode())


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def _f64(a):
    return np.ascontiguousarray(a, dtype=np.float64)


# ------------------------------------------------------------------ free functions
def time_bucket(delta: int, n_buckets: int) -> int:
    return lib().ref_time_bucket(int(delta), int(n_buckets))


def build_mask(l_q, roles, pos, local_window, full_suffix, query_rows=None):
    """(visible [l_q, l_kv] uint8, mask_visible_count) from rankformer::build_mask."""
    roles = np.ascontiguousarray(roles, dtype=np.int32)
    pos = np.ascontiguousarray(pos, dtype=np.int32)
    out = np.zeros((l_q, len(roles)), np.uint8)
    cnt = C.c_int64(0)
    qr = None if query_rows is None else np.ascontiguousarray(query_rows, dtype=np.int32)
    _check(lib().ref_build_mask(l_q, len(roles), local_window, full_suffix, _p(roles, i32p), _p(pos, i32p),
                                None if qr is None else _p(qr, i32p), _p(out, u8p), C.byref(cnt)))
    return out, cnt.value


def geometric_schedule(prefix_len, depth, target):
    out = np.zeros(max(depth, 1), np.int32)
    _check(lib().ref_geometric_schedule(prefix_len, depth, target, _p(out, i32p)))
    return out.tolist()


def full_schedule(prefix_len, depth):
    out = np.zeros(max(depth, 1), np.int32)
    _check(lib().ref_full_schedule(prefix_len, depth, _p(out, i32p)))
    return out.tolist()


def retained_rows(roles, keep, keep_specials):
    roles = np.ascontiguousarray(roles, dtype=np.int32)
    out = np.zeros(len(roles), np.int32)
    n = C.c_int(0)
    _check(lib().ref_retained_rows(_p(roles, i32p), len(roles), keep, int(keep_specials), _p(out, i32p),
                                   C.byref(n)))
    return out[: n.value].tolist()


def prune_queries(x, n):
    x = _f64(x)
    out = np.zeros((n, x.shape[1]))
    _check(lib().ref_prune_queries(_p(x, f64p), x.shape[0], x.shape[1], n, _p(out, f64p)))
    return out


def rmsnorm(x, gain):
    x, g = _f64(x), _f64(gain).reshape(-1)
    y, inv = np.zeros_like(x), np.zeros(x.shape[0])
    _check(lib().ref_rmsnorm_forward(_p(x, f64p), x.shape[0], x.shape[1], _p(g, f64p), _p(y, f64p), _p(inv, f64p)))
    return y, inv


def rmsnorm_backward(dy, x, gain):
    """(dx, dgain) of rmsnorm_backward (norm.hpp:32-45)."""
    dy, x, g = _f64(dy), _f64(x), _f64(gain).reshape(-1)
    dg, dx = np.zeros(x.shape[1]), np.zeros_like(x)
    _check(lib().ref_rmsnorm_backward(_p(dy, f64p), _p(x, f64p), x.shape[0], x.shape[1], _p(g, f64p),
                                      _p(dg, f64p), _p(dx, f64p)))
    return dx, dg


def rope(x, pos, theta=10000.0, inverse=False):
    x = _f64(x)
    p = np.ascontiguousarray(pos, dtype=np.int32)
    y = np.zeros_like(x)
    _check(lib().ref_rope_apply(_p(x, f64p), x.shape[0], x.shape[1], _p(p, i32p), theta, int(inverse), _p(y, f64p)))
    return y


def dense_attention(q, k, v, mask, dtype=np.float64):
    q, k, v, mask = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v, mask))
    out = np.zeros((q.shape[0], v.shape[1]), dtype=dtype)
    suf, t = ("f64", f64p) if dtype == np.float64 else ("f32", f32p)
    _check(getattr(lib(), f"ref_dense_attention_{suf}")(_p(q, t), _p(k, t), _p(v, t), _p(mask, t), q.shape[0],
                                                        k.shape[0], q.shape[1], v.shape[1], _p(out, t)))
    return out


def blockwise_attention(q, k, v, mask, block=16, dtype=np.float64):
    q, k, v, mask = (np.ascontiguousarray(a, dtype=dtype) for a in (q, k, v, mask))
    out = np.zeros((q.shape[0], v.shape[1]), dtype=dtype)
    sk, tot = C.c_int64(0), C.c_int64(0)
    suf, t = ("f64", f64p) if dtype == np.float64 else ("f32", f32p)
    _check(getattr(lib(), f"ref_blockwise_attention_{suf}")(_p(q, t), _p(k, t), _p(v, t), _p(mask, t), q.shape[0],
                                                            k.shape[0], q.shape[1], v.shape[1], block, _p(out, t),
                                                            C.byref(sk), C.byref(tot)))
    return out, sk.value, tot.value


# ------------------------------------------------------------------ model objects
def _grads(g, names):
    out = {}
    try:
        for name in names:
            r, c = C.c_int32(0), C.c_int32(0)
            _check(lib().ref_grads_get(g, name.encode(), None, C.byref(r), C.byref(c)))
            a = np.zeros((r.value, c.value))
            _check(lib().ref_grads_get(g, name.encode(), _p(a, f64p), None, None))
            out[name] = a
    finally:
        lib().ref_grads_destroy(g)
    return out


class RefModel:
    """The reference's Tokenizer + AttentionLayer objects (one per layer) loaded with the same
    named parameters as the oracle / the GPU handle; forward() composes them with the
    spec-only block / FFN / head (oracle/ref_harness.cpp)."""

    def __init__(self, cfg, params: Dict[str, np.ndarray]):
        import oracle as O
        oc = O.or_cfg(cfg)
        self.cfg = cfg
        h = C.c_void_p()
        _check(lib().ref_model_create(C.byref(oc), C.byref(h)))
        self.h = h
        for name, a in params.items():
            a64 = _f64(a)
            _check(lib().ref_model_set_param(self.h, name.encode(), _p(a64, f64p), a64.shape[0], a64.shape[1]))

    def __del__(self):
        if getattr(self, "h", None) and _lib is not None:
            _lib.ref_model_destroy(self.h)
            self.h = None

    def set_frozen(self, name: str, frozen: bool = True):
        _check(lib().ref_set_frozen(self.h, name.encode(), int(frozen)))

    def tokenize(self, batch, b: int = 0):
        hold = _SampleHold(batch, b)
        cfg = self.cfg
        L = (3 if cfg.special_tokens else 0) + hold.s.n_hist + hold.s.n_prof + hold.s.n_cand
        tokens = np.zeros((L, cfg.model_dim))
        pos, roles, cidx = (np.zeros(L, np.int32) for _ in range(3))
        ht = np.zeros(max(hold.s.n_hist, 1), np.int32)
        n = C.c_int(0)
        _check(lib().ref_tokenize(self.h, C.byref(hold.s), _p(tokens, f64p), _p(pos, i32p), _p(roles, i32p),
                                  _p(cidx, i32p), _p(ht, i32p), C.byref(n)))
        return {"tokens": tokens, "position_ids": pos, "roles": roles, "candidate_index": cidx,
                "hist_time": ht[: hold.s.n_hist]}

    def tokenize_clicks(self, batch, b: int = 0):
        hold = _SampleHold(batch, b)
        n = hold.s.n_hist
        tokens = np.zeros((1 + n, self.cfg.model_dim))
        ht = np.zeros(max(n, 1), np.int32)
        _check(lib().ref_tokenize_clicks(self.h, C.byref(hold.s), _p(tokens, f64p), _p(ht, i32p)))
        return tokens, ht[:n]

    def tokenizer_backward(self, batch, b: int, dtokens, names):
        hold = _SampleHold(batch, b)
        dt = _f64(dtokens)
        g = C.c_void_p()
        _check(lib().ref_tokenizer_backward(self.h, C.byref(hold.s), _p(dt, f64p), C.byref(g)))
        return _grads(g, names)

    def forward(self, batch, b: int = 0):
        hold = _SampleHold(batch, b)
        n = hold.s.n_cand
        probs, logits = np.zeros((n, 3)), np.zeros((n, 3))
        _check(lib().ref_model_forward(self.h, C.byref(hold.s), _p(probs, f64p), _p(logits, f64p)))
        return probs, logits

    def attention(self, layer, xn, query_rows, visible, pos):
        xn = _f64(xn)
        qr = np.ascontiguousarray(query_rows, dtype=np.int32)
        vis = np.ascontiguousarray(visible, dtype=np.uint8)
        p = np.ascontiguousarray(pos, dtype=np.int32)
        out = np.zeros((len(qr), self.cfg.model_dim))
        _check(lib().ref_attention_forward(self.h, layer, _p(xn, f64p), xn.shape[0], _p(qr, i32p), len(qr),
                                           _p(vis, u8p), _p(p, i32p), _p(out, f64p)))
        return out

    def attention_backward(self, layer, xn, query_rows, visible, pos, dout, names):
        """(dxn, {name: grad}) of AttentionLayer::backward (attention.cpp:134-202)."""
        xn, dout = _f64(xn), _f64(dout)
        qr = np.ascontiguousarray(query_rows, dtype=np.int32)
        vis = np.ascontiguousarray(visible, dtype=np.uint8)
        p = np.ascontiguousarray(pos, dtype=np.int32)
        dxn = np.zeros_like(xn)
        g = C.c_void_p()
        _check(lib().ref_attention_backward(self.h, layer, _p(xn, f64p), xn.shape[0], _p(qr, i32p), len(qr),
                                            _p(vis, u8p), _p(p, i32p), _p(dout, f64p), _p(dxn, f64p), C.byref(g)))
        return dxn, _grads(g, names)
