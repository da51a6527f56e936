# SPDX-License-Identifier: Apache-2.0
"""Request sharding across the GPUs of one node.

SORT requests are independent (one request-centric sample = one shared history with its
candidates), so data parallelism needs no collective in the forward pass: each rank scores
a contiguous shard of the requests with its own replica of the weights. The only
cross-rank traffic is host-side bookkeeping -- gathering scores to rank 0 when a caller
wants the whole batch, and the max-over-ranks step time a benchmark reports. Every kernel
is row-independent (no split-K, fixed reduction orders), so a request's scores are
bit-identical at 1, 2, 4 or 8 GPUs (tests/test_gpu_parity.py::test_batch_position_independence).
"""
from __future__ import annotations

from typing import Dict, List, Tuple

import numpy as np


def shard_range(total: int, world: int, rank: int) -> Tuple[int, int]:
    """Contiguous [begin, end) of `total` requests for `rank` (sizes differ by at most one)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError("bad world/rank")
    base, extra = divmod(total, world)
    begin = rank * base + min(rank, extra)
    return begin, begin + base + (1 if rank < extra else 0)


def shard_batch(batch: Dict[str, np.ndarray], world: int, rank: int) -> Dict[str, np.ndarray]:
    total = int(batch["req_ts"].shape[0])
    b, e = shard_range(total, world, rank)
    return {k: np.ascontiguousarray(v[b:e]) for k, v in batch.items()}


def gather_scores(local: np.ndarray, world: int, rank: int, group=None) -> np.ndarray:
    """Concatenate per-rank score shards [b_r, N, 3] on every rank, in rank order."""
    if world == 1:
        return local
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(local))
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([t.shape[0]], dtype=torch.int64), group=group)
    mx = int(max(s.item() for s in sizes))
    pad = torch.zeros((mx,) + tuple(t.shape[1:]), dtype=t.dtype)
    pad[: t.shape[0]] = t
    parts = [torch.zeros_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return np.concatenate([p[: int(s.item())].numpy() for p, s in zip(parts, sizes)], axis=0)


def max_over_ranks(values: List[float], world: int, device=None, group=None) -> List[float]:
    """Element-wise max of per-rank timings (the multi-GPU step time is the slowest rank)."""
    if world == 1:
        return list(values)
    import torch
    import torch.distributed as dist
    t = torch.tensor(values, dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t.cpu().tolist()


def allreduce_grads(flat, world: int, group=None):
    """Data-parallel training (BASELINE configs[2]): sum the flat fp32 gradient buffer of
    every rank's request shard (sort_grads_copy layout) in place. `flat` is a torch tensor
    (CUDA under NCCL, CPU under gloo). The per-request gradients of the reference's
    GradBuffer are additive (params.hpp:42-70), so the sum over shards equals the gradient
    of the whole batch."""
    if world == 1:
        return flat
    import torch.distributed as dist
    dist.all_reduce(flat, op=dist.ReduceOp.SUM, group=group)
    return flat


class ShardedItemTable:
    """Row-sharded item embedding table ("embedding-heavy": a
    100M-row table split over the GPUs of one node). Rank r owns global rows
    [r * rows_per_rank, (r + 1) * rows_per_rank) in `shard` (a torch tensor [rows, dim] on
    this rank's device). lookup() serves one batch through the library's C++ exchange
    (runtime.Exchange -> sort_exchange_lookup, csrc/exchange.cuh): ids grouped by owner on
    the device, ids to the owners and rows back by two all-to-all exchanges (NCCL, or the
    host transport), the owner gather and the batch-order scatter as CUDA kernels. It
    returns the batch-local table (row i = item row of the batch's i-th id, history ids first,
    then candidate ids) and the batch with ids replaced by those positions, ready for
    SortModel.set_item_table() (the reference reads item_table_.value.row(id) from its own
    table, tokenizer.cpp:95-127)."""

    def __init__(self, shard, rows_per_rank: int, rank: int, world: int, exchange, stream_ptr: int = 0):
        self.shard, self.R, self.rank, self.world = shard, rows_per_rank, rank, world
        self.x, self.stream_ptr = exchange, stream_ptr
        self._iota = {}

    def lookup(self, batch: Dict):
        import torch
        hist, cand = batch["hist_item"], batch["cand_item"]
        ids = torch.cat([hist.reshape(-1), cand.reshape(-1)]).to(torch.int32).contiguous()
        n, dim = ids.numel(), self.shard.shape[1]
        rows = torch.empty((n, dim), dtype=self.shard.dtype, device=ids.device)
        self.x.lookup(self.shard.data_ptr(), self.R, dim * self.shard.element_size(), ids.data_ptr(), n,
                      rows.data_ptr(), self.stream_ptr)
        key = (tuple(hist.shape), tuple(cand.shape), ids.device)
        if key not in self._iota:
            nh = hist.numel()
            pos = torch.arange(n, dtype=torch.int32, device=ids.device)
            self._iota[key] = (pos[:nh].reshape(hist.shape).contiguous(), pos[nh:].reshape(cand.shape).contiguous())
        out = dict(batch)
        out["hist_item"], out["cand_item"] = self._iota[key]
        return rows, out
