# SPDX-License-Identifier: Apache-2.0
"""ctypes binding of libsort_b200.so (include/sort_b200.h).

Mirrors the reference's operator API for the hot path with the same names and
error behaviour: config/input problems raise :class:`ConfigError` (status 1,
rankformer::ConfigError), runtime failures raise :class:`RuntimeFailure`
(status 2). There is no CPU fallback: if the library is missing or no sm_100
GPU is present, construction fails loudly.
"""
from __future__ import annotations

import ctypes as C
import os
from typing import Dict, Optional

import numpy as np

from .config import ConfigError, RuntimeFailure, SortConfig

_PKG = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_PKG, "libsort_b200.so")

i32p = C.POINTER(C.c_int32)
i64p = C.POINTER(C.c_int64)
f32p = C.POINTER(C.c_float)


class CSortConfig(C.Structure):
    _fields_ = [
        ("model_dim", C.c_int32), ("heads", C.c_int32), ("layers", C.c_int32),
        ("ffn_dim", C.c_int32), ("head_hidden", C.c_int32),
        ("item_dim", C.c_int32), ("action_dim", C.c_int32), ("scene_dim", C.c_int32),
        ("time_dim", C.c_int32), ("profile_dim", C.c_int32),
        ("n_items", C.c_int32), ("n_actions", C.c_int32), ("n_scenes", C.c_int32),
        ("n_time_buckets", C.c_int32), ("n_profile_fields", C.c_int32),
        ("profile_vocab", C.c_int32 * 16),
        ("special_tokens", C.c_int32), ("qknorm", C.c_int32), ("gate", C.c_int32),
        ("rope_theta", C.c_double), ("local_window", C.c_int32), ("full_suffix", C.c_int32),
        ("keep", C.c_int32 * 64), ("keep_specials", C.c_int32),
        ("max_batch", C.c_int32), ("n_hist", C.c_int32), ("n_cand", C.c_int32),
        ("moe_experts", C.c_int32), ("moe_topk", C.c_int32), ("moe_shared", C.c_int32),
        ("moe_ffn_dim", C.c_int32), ("pretrain", C.c_int32),
    ]


class CSortBatch(C.Structure):
    _fields_ = [
        ("batch", C.c_int32), ("hist_item", C.c_void_p), ("hist_action", C.c_void_p),
        ("hist_scene", C.c_void_p), ("hist_ts", C.c_void_p), ("req_ts", C.c_void_p),
        ("profile", C.c_void_p), ("cand_item", C.c_void_p),
    ]


EXPORTS = [
    "sort_last_error", "sort_version", "sort_create", "sort_destroy", "sort_set_stream",
    "sort_load_param", "sort_finalize_params", "sort_forward", "sort_sync", "sort_forward_logits",
    "sort_tokenize", "sort_layer_plan", "sort_attention_forward", "sort_block_attention",
    "sort_time_bucket", "sort_geometric_schedule", "sort_retained_rows", "sort_mask_intervals",
    "sort_kernel_count", "sort_enable_stage_timing", "sort_stage_times", "sort_set_option",
    "sort_train_step", "sort_grad_info", "sort_grads_copy", "sort_dtokens",
    "sort_set_item_table", "sort_gather_rows", "sort_train_step_bce", "sort_adamw_step",
    "sort_get_param", "sort_dataset_open", "sort_dataset_close", "sort_dataset_size",
    "sort_dataset_batch", "sort_moe_routing", "sort_moe_load", "sort_moe_update_bias",
    "sort_moe_forward", "sort_pretrain_forward", "sort_forward_async",
    "sort_nccl_unique_id", "sort_exchange_create_nccl", "sort_exchange_create_host",
    "sort_exchange_destroy", "sort_exchange_lookup", "sort_exchange_allreduce_f32", "sort_op_gemm",
    "sort_op_rmsnorm", "sort_op_rmsnorm_backward", "sort_op_rope", "sort_op_attention_layer",
    "sort_get_grad", "sort_set_frozen", "sort_transfer_item_table", "sort_pretrain_train_step",
]

_lib = None

# host-transport callbacks of the exchange (sort_alltoallv_fn / sort_allreduce_fn)
ALLTOALLV_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.POINTER(C.c_int64), C.c_void_p,
                           C.POINTER(C.c_int64), C.c_int)
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.POINTER(C.c_float), C.c_int64)


def lib():
    """Load the CUDA library (raises if it was not built -- no fallback)."""
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            raise RuntimeFailure(f"{LIB_PATH} not built; run __graft_entry__.build()")
        L = C.CDLL(LIB_PATH)
        L.sort_last_error.restype = C.c_char_p
        L.sort_create.argtypes = [C.POINTER(CSortConfig), C.c_int, C.POINTER(C.c_void_p)]
        L.sort_destroy.argtypes = [C.c_void_p]
        L.sort_set_stream.argtypes = [C.c_void_p, C.c_void_p]
        L.sort_load_param.argtypes = [C.c_void_p, C.c_char_p, f32p, C.c_int64, C.c_int64]
        L.sort_finalize_params.argtypes = [C.c_void_p]
        L.sort_forward.argtypes = [C.c_void_p, C.POINTER(CSortBatch), C.c_int, C.c_void_p, C.c_int]
        L.sort_sync.argtypes = [C.c_void_p]
        L.sort_forward_logits.argtypes = [C.c_void_p, C.POINTER(CSortBatch), f32p, f32p]
        L.sort_tokenize.argtypes = [C.c_void_p, C.POINTER(CSortBatch), f32p, i32p, i32p, i32p, i32p]
        L.sort_layer_plan.argtypes = [C.c_void_p, C.c_int, i32p, i32p, i32p, i32p, i32p, i32p, i64p,
                                      i64p, i64p]
        L.sort_attention_forward.argtypes = [C.c_void_p, C.c_int, C.c_int32, f32p, f32p]
        L.sort_block_attention.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, f32p, f32p,
                                           f32p, i32p, i32p, i32p, f32p, i64p, i64p]
        L.sort_time_bucket.argtypes = [C.c_int64, C.c_int32]
        L.sort_geometric_schedule.argtypes = [C.c_int32, C.c_int32, C.c_int32, i32p]
        L.sort_retained_rows.argtypes = [i32p, C.c_int32, C.c_int32, C.c_int32, i32p, i32p]
        L.sort_mask_intervals.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, i32p, i32p,
                                          i32p, i32p, i32p, i32p]
        L.sort_kernel_count.argtypes = [C.c_void_p, i32p]
        L.sort_enable_stage_timing.argtypes = [C.c_void_p, C.c_int]
        L.sort_set_option.argtypes = [C.c_void_p, C.c_char_p, C.c_int32]
        L.sort_train_step.argtypes = [C.c_void_p, C.c_void_p, f32p, f32p]
        L.sort_grad_info.argtypes = [C.c_void_p, C.c_char_p, i64p, i64p, i64p, i64p]
        L.sort_grads_copy.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_int]
        L.sort_dtokens.argtypes = [C.c_void_p, C.c_int32, f32p]
        L.sort_set_item_table.argtypes = [C.c_void_p, C.c_void_p, C.c_int64]
        L.sort_train_step_bce.argtypes = [C.c_void_p, C.c_void_p, f32p, f32p, f32p]
        L.sort_adamw_step.argtypes = [C.c_void_p, C.c_float, C.c_float, C.c_float, C.c_float, C.c_float]
        L.sort_get_param.argtypes = [C.c_void_p, C.c_char_p, f32p]
        L.sort_get_grad.argtypes = [C.c_void_p, C.c_char_p, f32p]
        L.sort_pretrain_train_step.argtypes = [C.c_void_p, C.c_void_p, f32p]
        L.sort_set_frozen.argtypes = [C.c_void_p, C.c_char_p, C.c_int32]
        L.sort_transfer_item_table.argtypes = [C.c_void_p, C.c_void_p, C.c_int32]
        L.sort_moe_routing.argtypes = [C.c_void_p, C.c_int, C.c_int32, i32p, i32p, f32p]
        L.sort_moe_load.argtypes = [C.c_void_p, C.c_int, i64p]
        L.sort_moe_update_bias.argtypes = [C.c_void_p, C.c_double]
        L.sort_moe_forward.argtypes = [C.c_void_p, C.c_int, f32p, C.c_int, f32p]
        L.sort_forward_async.argtypes = [C.c_void_p, C.c_void_p, C.c_void_p]
        L.sort_pretrain_forward.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_void_p, C.c_int]
        L.sort_dataset_open.argtypes = [C.c_char_p, C.POINTER(C.c_void_p)]
        L.sort_dataset_close.argtypes = [C.c_void_p]
        L.sort_dataset_size.argtypes = [C.c_void_p]
        L.sort_dataset_size.restype = C.c_int64
        L.sort_dataset_batch.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_int32, C.c_int32, C.c_int32,
                                         C.POINTER(CSortBatch), f32p, i64p]
        L.sort_gather_rows.argtypes = [C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                       C.c_void_p, C.c_void_p]
        L.sort_stage_times.argtypes = [C.c_void_p, f32p, C.c_int32, i32p, C.c_char_p, C.c_int32]
        L.sort_nccl_unique_id.argtypes = [C.c_void_p]
        L.sort_exchange_create_nccl.argtypes = [C.c_void_p, C.c_int, C.c_int, C.c_int, C.POINTER(C.c_void_p)]
        L.sort_exchange_create_host.argtypes = [ALLTOALLV_FN, ALLREDUCE_FN, C.c_void_p, C.c_int, C.c_int, C.c_int,
                                                C.POINTER(C.c_void_p)]
        L.sort_exchange_destroy.argtypes = [C.c_void_p]
        L.sort_exchange_lookup.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_int32, C.c_void_p, C.c_int64,
                                           C.c_void_p, C.c_void_p]
        L.sort_exchange_allreduce_f32.argtypes = [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p]
        L.sort_op_gemm.argtypes = [C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, C.c_int32, f32p, f32p, f32p]
        L.sort_op_rmsnorm.argtypes = [C.c_int32, C.c_int32, f32p, f32p, f32p, f32p]
        L.sort_op_rmsnorm_backward.argtypes = [C.c_int32, C.c_int32, f32p, f32p, f32p, f32p, f32p, f32p]
        L.sort_op_rope.argtypes = [C.c_int32, C.c_int32, f32p, i32p, C.c_double, C.c_int32, f32p]
        L.sort_op_attention_layer.argtypes = [C.c_int32, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_int32,
                                              C.c_int32, f32p, i32p, i32p, i32p, i32p, i32p,
                                              C.POINTER(f32p), f32p, f32p, f32p, C.POINTER(f32p)]
        _lib = L
    return _lib


def _check(status: int) -> None:
    if status == 0:
        return
    msg = lib().sort_last_error().decode()
    if status == 1:
        raise ConfigError(msg)
    raise RuntimeFailure(msg)


def _p(a: np.ndarray, t):
    return a.ctypes.data_as(t)


def to_c_config(cfg: SortConfig, max_batch: Optional[int] = None) -> CSortConfig:
    cfg.validate()
    c = CSortConfig()
    c.model_dim, c.heads, c.layers, c.ffn_dim = cfg.model_dim, cfg.heads, cfg.layers, cfg.ffn_dim
    c.head_hidden = cfg.head_hidden
    c.item_dim, c.action_dim, c.scene_dim = cfg.item_dim, cfg.action_dim, cfg.scene_dim
    c.time_dim, c.profile_dim = cfg.time_dim, cfg.profile_dim
    c.n_items, c.n_actions, c.n_scenes = cfg.n_items, cfg.n_actions, cfg.n_scenes
    c.n_time_buckets, c.n_profile_fields = cfg.n_time_buckets, cfg.n_prof
    for i, v in enumerate(cfg.profile_vocab):
        c.profile_vocab[i] = v
    c.special_tokens, c.qknorm, c.gate = int(cfg.special_tokens), int(cfg.qknorm), int(cfg.gate)
    c.rope_theta = cfg.rope_theta
    c.local_window, c.full_suffix = cfg.local_window, cfg.full_suffix
    for i, k in enumerate(cfg.keep_schedule()):
        c.keep[i] = k
    c.keep_specials = int(cfg.keep_specials)
    c.max_batch = max_batch or cfg.batch
    c.n_hist, c.n_cand = cfg.n_hist, cfg.n_cand
    c.moe_experts, c.moe_topk = cfg.moe_experts, cfg.moe_topk
    c.moe_shared, c.moe_ffn_dim = cfg.moe_shared, cfg.moe_ffn_dim
    c.pretrain = int(cfg.pretrain)
    return c


# ----------------------------------------------------------------- host planner (no GPU)
def time_bucket(delta: int, n_buckets: int = 32) -> int:
    return lib().sort_time_bucket(int(delta), int(n_buckets))


def geometric_schedule(prefix_len: int, depth: int, target: int):
    out = np.zeros(max(depth, 1), np.int32)
    _check(lib().sort_geometric_schedule(prefix_len, depth, target, _p(out, i32p)))
    return out.tolist()


def retained_rows(roles, keep: int, keep_specials: bool):
    r = np.ascontiguousarray(roles, np.int32)
    out = np.zeros(len(r), np.int32)
    n = C.c_int32(0)
    _check(lib().sort_retained_rows(_p(r, i32p), len(r), keep, int(keep_specials), _p(out, i32p),
                                    C.byref(n)))
    return out[: n.value].tolist()


def mask_intervals(roles, pos, query_rows, window: int, full_suffix: int):
    r = np.ascontiguousarray(roles, np.int32)
    p = np.ascontiguousarray(pos, np.int32)
    q = np.ascontiguousarray(query_rows, np.int32)
    lo, hi, se = (np.zeros(len(q), np.int32) for _ in range(3))
    _check(lib().sort_mask_intervals(len(q), len(r), window, full_suffix, _p(r, i32p), _p(p, i32p),
                                     _p(q, i32p), _p(lo, i32p), _p(hi, i32p), _p(se, i32p)))
    return lo, hi, se


def block_attention(q: np.ndarray, k: np.ndarray, v: np.ndarray, lo, hi, self_idx):
    """blockwise_masked_attention on the GPU kernel: q [nh, lq, dk], k/v [nh, lkv, dk]."""
    q, k, v = (np.ascontiguousarray(a, np.float32) for a in (q, k, v))
    nh, lq, dk = q.shape
    lkv = k.shape[1]
    lo, hi, se = (np.ascontiguousarray(a, np.int32) for a in (lo, hi, self_idx))
    out = np.zeros((nh, lq, dk), np.float32)
    sk, tot = C.c_int64(0), C.c_int64(0)
    _check(lib().sort_block_attention(nh, lq, lkv, dk, _p(q, f32p), _p(k, f32p), _p(v, f32p),
                                      _p(lo, i32p), _p(hi, i32p), _p(se, i32p), _p(out, f32p),
                                      C.byref(sk), C.byref(tot)))
    return out, sk.value, tot.value


# ----------------------------------------------------------------- model handle
class _BatchHold:
    KEYS = ("hist_item", "hist_action", "hist_scene", "hist_ts", "req_ts", "profile", "cand_item")
    DT = {"hist_ts": np.int64, "req_ts": np.int64}

    def __init__(self, batch: Dict[str, np.ndarray]):
        self.arrs = {k: np.ascontiguousarray(batch[k], dtype=self.DT.get(k, np.int32)) for k in self.KEYS}
        a = self.arrs
        self.c = CSortBatch(int(a["req_ts"].shape[0]), *[a[k].ctypes.data for k in self.KEYS])


class _DevBatch:
    """SortBatch of device pointers (torch CUDA tensors) for the device-resident path."""

    def __init__(self, tensors):
        self.t = tensors
        self.c = CSortBatch(int(tensors["req_ts"].shape[0]),
                            *[tensors[k].data_ptr() for k in _BatchHold.KEYS])


class SortModel:
    """One handle per GPU: the batched SORT forward behind the C ABI."""

    def __init__(self, cfg: SortConfig, params: Dict[str, np.ndarray], device: int = 0,
                 max_batch: Optional[int] = None):
        self.cfg = cfg
        self.max_batch = max_batch or cfg.batch
        h = C.c_void_p()
        _check(lib().sort_create(C.byref(to_c_config(cfg, self.max_batch)), device, C.byref(h)))
        self.h = h
        for name, a in params.items():
            a32 = np.ascontiguousarray(a, np.float32)
            if a32.ndim != 2:
                raise ConfigError(f"parameter {name} must be 2-D")
            _check(lib().sort_load_param(self.h, name.encode(), _p(a32, f32p), a32.shape[0],
                                         a32.shape[1]))
        _check(lib().sort_finalize_params(self.h))
        # experiments only: SORT_OPTIONS="graphs=0" sets library options (A/B runs)
        for kv in filter(None, os.environ.get("SORT_OPTIONS", "").split(",")):
            k, v = kv.split("=")
            self.set_option(k.strip(), int(v))

    def close(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.sort_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def set_stream(self, stream_ptr: int):
        _check(lib().sort_set_stream(self.h, C.c_void_p(stream_ptr)))

    # -- forward (model_forward) ---------------------------------
    def forward(self, batch: Dict[str, np.ndarray]) -> np.ndarray:
        hold = _BatchHold(batch)
        B = hold.c.batch
        out = np.zeros((B, self.cfg.n_cand, 3), np.float32)
        _check(lib().sort_forward(self.h, C.byref(hold.c), 0, out.ctypes.data, 0))
        return out

    def forward_logits(self, batch: Dict[str, np.ndarray]):
        hold = _BatchHold(batch)
        B = hold.c.batch
        probs = np.zeros((B, self.cfg.n_cand, 3), np.float32)
        logits = np.zeros((B, self.cfg.n_cand, 3), np.float32)
        _check(lib().sort_forward_logits(self.h, C.byref(hold.c), _p(probs, f32p), _p(logits, f32p)))
        return probs, logits

    def forward_device(self, dev_batch: "_DevBatch", scores_ptr: int):
        """Device-resident inputs and outputs: enqueue only (no host sync)."""
        _check(lib().sort_forward(self.h, C.byref(dev_batch.c), 1, C.c_void_p(scores_ptr), 1))

    def sync(self):
        _check(lib().sort_sync(self.h))

    # -- row-sharded item table --------------------------------------------------
    def set_item_table(self, ptr: int, n_rows: int):
        """Batch-local item rows (device bf16 [n_rows, item_dim]) for the next calls; ptr=0
        restores the handle's own table."""
        _check(lib().sort_set_item_table(self.h, C.c_void_p(ptr) if ptr else None, int(n_rows)))

    # -- pre-training -----------------------------------------
    def pretrain_forward(self, batch: Dict[str, np.ndarray]):
        """(lse [B, n], target_logit [B, n]) of the tied next-item head; CE = lse - target."""
        hold = _BatchHold(batch)
        B, n = hold.c.batch, self.cfg.n_hist
        lse = np.zeros((B, n), np.float32)
        tgt = np.zeros((B, n), np.float32)
        _check(lib().sort_pretrain_forward(self.h, C.byref(hold.c), 0, lse.ctypes.data, tgt.ctypes.data, 0))
        return lse, tgt

    def pretrain_forward_device(self, dev_batch: "_DevBatch", lse_ptr: int, tgt_ptr: int):
        """Device-resident inputs and outputs: enqueue only (no host sync)."""
        _check(lib().sort_pretrain_forward(self.h, C.byref(dev_batch.c), 1, C.c_void_p(lse_ptr),
                                           C.c_void_p(tgt_ptr), 1))

    # -- MoE FFN ----------------------------------------------
    def moe_routing(self, layer: int, rows: int | None = None):
        """(sel [rows, k] int32, weights [rows, k]) of `layer` in the last forward. `rows` is
        checked against the routed row count (ConfigError if the buffers would be too small);
        None sizes the buffers from the library's own count."""
        k = self.cfg.moe_topk
        n = C.c_int32(0)
        _check(lib().sort_moe_routing(self.h, layer, 0, C.byref(n), None, None))
        rows = n.value if rows is None else rows
        sel = np.zeros((rows, k), np.int32)
        w = np.zeros((rows, k), np.float32)
        _check(lib().sort_moe_routing(self.h, layer, rows, None, _p(sel, i32p), _p(w, f32p)))
        return sel[:n.value], w[:n.value]

    def moe_load(self, layer: int) -> np.ndarray:
        out = np.zeros(self.cfg.moe_experts, np.int64)
        _check(lib().sort_moe_load(self.h, layer, _p(out, i64p)))
        return out

    def moe_update_bias(self, gamma: float = 1e-3) -> None:
        _check(lib().sort_moe_update_bias(self.h, float(gamma)))

    def moe_forward(self, layer: int, x: np.ndarray) -> np.ndarray:
        """out = x + MoE(RMSNorm(x; ffn_norm)) through the device path (bf16 residual)."""
        x = np.ascontiguousarray(x, dtype=np.float32)
        out = np.zeros_like(x)
        _check(lib().sort_moe_forward(self.h, layer, _p(x, f32p), x.shape[0], _p(out, f32p)))
        return out

    # -- training (sort_train_step) --------------------------------------------
    def train_step(self, batch: Dict[str, np.ndarray], dlogits: np.ndarray) -> np.ndarray:
        """Forward + backward given dL/dlogits [B, n_cand, 3]; returns the step's logits.
        Gradients stay on the device (grad(), grads_flat())."""
        hold = _BatchHold(batch)
        B = hold.c.batch
        dz = np.ascontiguousarray(dlogits, np.float32).reshape(B, self.cfg.n_cand, 3)
        logits = np.zeros((B, self.cfg.n_cand, 3), np.float32)
        _check(lib().sort_train_step(self.h, C.byref(hold.c), _p(dz, f32p), _p(logits, f32p)))
        return logits

    def train_step_bce(self, batch: Dict[str, np.ndarray], labels: np.ndarray,
                       obj_weights=(1.0, 0.5, 0.5)) -> float:
        """Forward + ranking loss (weighted mean BCE of click / cart /
        purchase, labels [B, n_cand, 3]) + backward, all on the device; returns the loss."""
        hold = _BatchHold(batch)
        lab = np.ascontiguousarray(labels, np.float32)
        w = np.ascontiguousarray(obj_weights, np.float32)
        loss = C.c_float(0.0)
        _check(lib().sort_train_step_bce(self.h, C.byref(hold.c), _p(lab, f32p), _p(w, f32p),
                                         C.byref(loss)))
        return float(loss.value)

    def pretrain_train_step(self, batch: Dict[str, np.ndarray]) -> float:
        """Pre-training step: mean next-item CE over the predicted positions,
        gradients of every parameter (item table included unless frozen) on the device."""
        hold = _BatchHold(batch)
        loss = np.zeros(1, np.float32)
        _check(lib().sort_pretrain_train_step(self.h, C.byref(hold.c), _p(loss, f32p)))
        return float(loss[0])

    def adamw_step(self, lr: float, beta1: float = 0.9, beta2: float = 0.99, eps: float = 1e-8,
                   weight_decay: float = 0.01):
        """adamw_step (paper defaults beta = (0.9, 0.99), wd = 0.01) on the fp32
        masters, then the bf16 inference weights are rebuilt on the device."""
        _check(lib().sort_adamw_step(self.h, lr, beta1, beta2, eps, weight_decay))

    def _shape(self, name: str):
        if name == "tok.item_table":
            return self.cfg.n_items, self.cfg.item_dim
        return self.grad_layout(name)[1:3]

    def get_param(self, name: str) -> np.ndarray:
        out = np.zeros(self._shape(name), np.float32)
        _check(lib().sort_get_param(self.h, name.encode(), _p(out, f32p)))
        return out

    def get_grad(self, name: str) -> np.ndarray:
        """Gradient of `name` from the last training step (tok.item_table when not frozen)."""
        out = np.zeros(self._shape(name), np.float32)
        _check(lib().sort_get_grad(self.h, name.encode(), _p(out, f32p)))
        return out

    def set_frozen(self, name: str, frozen: bool = True) -> None:
        """Parameter::frozen (params.hpp:15-25): no gradient, no optimizer update."""
        _check(lib().sort_set_frozen(self.h, name.encode(), int(frozen)))

    def transfer_item_table(self, source: "SortModel", freeze: bool = True) -> None:
        """transfer_item_table(source -> self, freeze) (tokenizer.cpp:376-383)."""
        _check(lib().sort_transfer_item_table(source.h, self.h, int(freeze)))

    def grad_layout(self, name: Optional[str] = None):
        off, r, c, tot = (C.c_int64(0) for _ in range(4))
        _check(lib().sort_grad_info(self.h, name.encode() if name else None, C.byref(off), C.byref(r),
                                    C.byref(c), C.byref(tot)))
        return off.value, r.value, c.value, tot.value

    def grads_flat(self) -> np.ndarray:
        n = self.grad_layout()[3]
        out = np.zeros(n, np.float32)
        _check(lib().sort_grads_copy(self.h, C.c_void_p(out.ctypes.data), 0, 0))
        return out

    def grads_to_device(self, ptr: int, on_device: bool = True, to_handle: bool = False):
        """Copy the flat gradient buffer to (or, to_handle=True, from) caller memory, e.g. a
        torch tensor that torch.distributed all-reduces across data-parallel ranks."""
        _check(lib().sort_grads_copy(self.h, C.c_void_p(ptr), int(on_device), int(to_handle)))

    def grad(self, name: str) -> np.ndarray:
        off, r, c, _ = self.grad_layout(name)
        return self.grads_flat()[off: off + r * c].reshape(r, c)

    def dtokens(self, batch_size: int) -> np.ndarray:
        out = np.zeros((batch_size, self.cfg.seq_len, self.cfg.model_dim), np.float32)
        _check(lib().sort_dtokens(self.h, batch_size, _p(out, f32p)))
        return out

    # -- parity ops ------------------------------------------------------------
    def tokenize(self, batch: Dict[str, np.ndarray]):
        hold = _BatchHold(batch)
        B, L = hold.c.batch, self.cfg.seq_len
        tokens = np.zeros((B, L, self.cfg.model_dim), np.float32)
        ht = np.zeros((B, max(self.cfg.n_hist, 1)), np.int32)
        pos, roles, cidx = (np.zeros(L, np.int32) for _ in range(3))
        _check(lib().sort_tokenize(self.h, C.byref(hold.c), _p(tokens, f32p), _p(ht, i32p),
                                   _p(pos, i32p), _p(roles, i32p), _p(cidx, i32p)))
        return {"tokens": tokens, "hist_time": ht[:, : self.cfg.n_hist], "position_ids": pos,
                "roles": roles, "candidate_index": cidx}

    def layer_plan(self, layer: int):
        L = self.cfg.seq_len
        lq, lkv = C.c_int32(0), C.c_int32(0)
        qr, lo, hi, se = (np.zeros(L, np.int32) for _ in range(4))
        vis, ti, tt = C.c_int64(0), C.c_int64(0), C.c_int64(0)
        _check(lib().sort_layer_plan(self.h, layer, C.byref(lq), C.byref(lkv), _p(qr, i32p),
                                     _p(lo, i32p), _p(hi, i32p), _p(se, i32p), C.byref(vis),
                                     C.byref(ti), C.byref(tt)))
        n = lq.value
        return {"l_q": n, "l_kv": lkv.value, "query_rows": qr[:n], "lo": lo[:n], "hi": hi[:n],
                "self": se[:n], "visible": vis.value, "tiles_issued": ti.value,
                "tiles_total": tt.value}

    def attention_forward(self, layer: int, x: np.ndarray) -> np.ndarray:
        x = np.ascontiguousarray(x, np.float32)
        B = x.shape[0]
        plan = self.layer_plan(layer)
        out = np.zeros((B, plan["l_q"], self.cfg.model_dim), np.float32)
        _check(lib().sort_attention_forward(self.h, layer, B, _p(x, f32p), _p(out, f32p)))
        return out

    # -- instrumentation -------------------------------------------------------
    def kernel_count(self) -> int:
        n = C.c_int32(0)
        _check(lib().sort_kernel_count(self.h, C.byref(n)))
        return n.value

    def set_option(self, name: str, value: int):
        """Kernel-selection knob (sort_set_option), e.g. ("fused_tail", 0) for the unfused
        Wo / FFN GEMM chain."""
        _check(lib().sort_set_option(self.h, name.encode(), int(value)))

    def enable_stage_timing(self, on: bool = True):
        _check(lib().sort_enable_stage_timing(self.h, int(on)))

    def stage_times(self):
        ms = np.zeros(256, np.float32)
        n = C.c_int32(0)
        names = C.create_string_buffer(8192)
        _check(lib().sort_stage_times(self.h, _p(ms, f32p), 256, C.byref(n), names, 8192))
        keys = names.value.decode().split(";") if n.value else []
        return dict(zip(keys, ms[: n.value].tolist()))


def op_gemm(A: np.ndarray, B: np.ndarray, trans_a: bool = False, trans_b: bool = False, tf32: bool = False) -> np.ndarray:
    """C = op(A) op(B) on the library's GEMM engines (sort_op_gemm): bf16 (tcgen05 streaming
    GEMM) or fp32 at TF32 precision; A [M, K] (or [K, M] when trans_a), B [K, N] (or [N, K])."""
    A = np.ascontiguousarray(A, np.float32)
    B = np.ascontiguousarray(B, np.float32)
    M, K = (A.shape[1], A.shape[0]) if trans_a else A.shape
    N = B.shape[0] if trans_b else B.shape[1]
    C_ = np.zeros((M, N), np.float32)
    _check(lib().sort_op_gemm(M, N, K, int(trans_a), int(trans_b), int(tf32), _p(A, f32p), _p(B, f32p), _p(C_, f32p)))
    return C_


def gather_rows(table_ptr: int, n_rows: int, row_bytes: int, ids_ptr: int, n: int, out_ptr: int,
                stream_ptr: int = 0) -> None:
    """out[i] = table[ids[i]] on the device (the owner-local step of a sharded lookup)."""
    _check(lib().sort_gather_rows(C.c_void_p(table_ptr), int(n_rows), int(row_bytes),
                                  C.c_void_p(ids_ptr), int(n), C.c_void_p(out_ptr),
                                  C.c_void_p(stream_ptr) if stream_ptr else None))


class Exchange:
    """One rank's end of the library's cross-rank exchange (csrc/exchange.cuh): the
    row-sharded item lookup and the data-parallel gradient sum, run by the C++ host.

    Exchange.nccl(rank, world, device): NCCL communicator (the 128-byte unique id is made on
    rank 0 and broadcast over the torch.distributed group). Exchange.host(rank, world,
    device): payloads staged through host memory and moved by torch.distributed collectives
    of the current (e.g. gloo) group -- several ranks may share one GPU (tests)."""

    def __init__(self, handle, keep=()):
        self.h = handle
        self._keep = keep  # the ctypes callbacks must outlive the handle

    @classmethod
    def nccl(cls, rank: int, world: int, device: int = 0, group=None):
        uid = (C.c_uint8 * 128)()
        if rank == 0:
            _check(lib().sort_nccl_unique_id(uid))
        if world > 1:
            import torch.distributed as dist
            obj = [bytes(uid)]
            dist.broadcast_object_list(obj, src=0, group=group)
            C.memmove(uid, obj[0], 128)
        h = C.c_void_p()
        _check(lib().sort_exchange_create_nccl(uid, rank, world, device, C.byref(h)))
        return cls(h)

    @classmethod
    def host(cls, rank: int, world: int, device: int = 0, group=None):
        fa, fr = host_transport(group)
        h = C.c_void_p()
        _check(lib().sort_exchange_create_host(fa, fr, None, rank, world, device, C.byref(h)))
        return cls(h, (fa, fr))

    def close(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.sort_exchange_destroy(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def lookup(self, shard_ptr: int, rows_per_rank: int, row_bytes: int, ids_ptr: int, n: int, out_ptr: int,
               stream_ptr: int = 0):
        """out[i] = table[ids[i]] for global ids against the row-sharded table (collective)."""
        _check(lib().sort_exchange_lookup(self.h, C.c_void_p(shard_ptr), int(rows_per_rank), int(row_bytes),
                                          C.c_void_p(ids_ptr), int(n), C.c_void_p(out_ptr),
                                          C.c_void_p(stream_ptr) if stream_ptr else None))

    def allreduce(self, buf_ptr: int, n: int, stream_ptr: int = 0):
        _check(lib().sort_exchange_allreduce_f32(self.h, C.c_void_p(buf_ptr), int(n),
                                                 C.c_void_p(stream_ptr) if stream_ptr else None))


def host_transport(group=None):
    """The (alltoallv, allreduce) host callbacks over torch.distributed CPU collectives."""
    import torch
    import torch.distributed as dist

    def a2a(ctx, send, send_bytes, recv, recv_bytes, world):
        try:
            sb = [int(send_bytes[i]) for i in range(world)]
            rb = [int(recv_bytes[i]) for i in range(world)]
            src = (torch.frombuffer((C.c_uint8 * sum(sb)).from_address(send), dtype=torch.uint8)
                   if sum(sb) else torch.empty(0, dtype=torch.uint8))
            out = torch.empty(sum(rb), dtype=torch.uint8)
            dist.all_to_all_single(out, src.clone(), rb, sb, group=group)
            if sum(rb):
                C.memmove(recv, out.data_ptr(), sum(rb))
            return 0
        except Exception:  # noqa: BLE001 -- reported to the library as a failed callback
            return 1

    def red(ctx, buf, n):
        try:
            if int(n) == 0:
                return 0
            t = torch.frombuffer((C.c_float * int(n)).from_address(C.addressof(buf.contents)), dtype=torch.float32)
            tmp = t.clone()
            dist.all_reduce(tmp, group=group)
            t.copy_(tmp)
            return 0
        except Exception:  # noqa: BLE001
            return 1

    return ALLTOALLV_FN(a2a), ALLREDUCE_FN(red)


class Dataset:
    """The reference's JSONL dataset (schema "rankformer.dataset" v1, read_dataset,
    dataset_io.cpp:58-162) parsed by the library's host reader into pinned SoA batches."""

    def __init__(self, path: str):
        h = C.c_void_p()
        _check(lib().sort_dataset_open(path.encode(), C.byref(h)))
        self.h = h

    def __len__(self) -> int:
        return int(lib().sort_dataset_size(self.h))

    def close(self):
        if getattr(self, "h", None) is not None and _lib is not None:
            _lib.sort_dataset_close(self.h)
            self.h = None

    def __del__(self):
        self.close()

    def batch(self, first: int, count: int, cfg: SortConfig):
        """(SortBatch over the dataset's pinned arrays, labels [count, n_cand, 3], request ids,
        numpy views of the arrays). The arrays stay valid until the next batch() call."""
        cb = CSortBatch()
        labels = np.zeros((count, cfg.n_cand, 3), np.float32)
        ids = np.zeros(count, np.int64)
        P = len(cfg.profile_vocab)
        _check(lib().sort_dataset_batch(self.h, first, count, cfg.n_hist, cfg.n_cand, P, C.byref(cb),
                                        _p(labels, f32p), _p(ids, i64p)))

        def view(ptr, shape, dt):
            n = int(np.prod(shape))
            ct = C.c_int64 if dt == np.int64 else C.c_int32
            return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(ct)), shape=(n,)).reshape(shape).view(dt)

        arrs = {"hist_item": view(cb.hist_item, (count, cfg.n_hist), np.int32),
                "hist_action": view(cb.hist_action, (count, cfg.n_hist), np.int32),
                "hist_scene": view(cb.hist_scene, (count, cfg.n_hist), np.int32),
                "hist_ts": view(cb.hist_ts, (count, cfg.n_hist), np.int64),
                "req_ts": view(cb.req_ts, (count,), np.int64),
                "profile": view(cb.profile, (count, P), np.int32),
                "cand_item": view(cb.cand_item, (count, cfg.n_cand), np.int32)}
        return cb, labels, ids, arrs


def write_dataset(path: str, batch: Dict[str, np.ndarray], labels: Optional[np.ndarray] = None,
                  request_ids=None) -> None:
    """write_dataset (dataset_io.cpp:14-56) for a SoA batch: header line + one JSON record per
    request (history events [item, action, ts, scene], candidates [item, click, cart,
    purchase, side])."""
    import json
    B = int(batch["req_ts"].shape[0])
    with open(path, "w") as f:
        f.write(json.dumps({"schema": "rankformer.dataset", "version": 1, "records": B}) + "\n")
        for b in range(B):
            hist = [[int(batch["hist_item"][b, i]), int(batch["hist_action"][b, i]), int(batch["hist_ts"][b, i]),
                     int(batch["hist_scene"][b, i])] for i in range(batch["hist_item"].shape[1])]
            cands = []
            for j in range(batch["cand_item"].shape[1]):
                lab = [0, 0, 0] if labels is None else [int(x) for x in labels[b, j]]
                cands.append([int(batch["cand_item"][b, j]), lab[0], lab[1], lab[2], []])
            rec = {"request_id": int(request_ids[b]) if request_ids is not None else b,
                   "ts": int(batch["req_ts"][b]), "profile": [int(x) for x in batch["profile"][b]],
                   "history": hist, "candidates": cands}
            f.write(json.dumps(rec) + "\n")
