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
    this rank's device). lookup() serves one batch:

      1. dedupe the batch's item ids (history + candidates)          torch.unique
      2. exchange per-owner counts, then the ids                      all_to_all (NCCL)
      3. each owner gathers its rows                                  sort_gather_rows
      4. rows travel back in the requester's unique-id order          all_to_all (NCCL)

    and returns the batch-local table plus the batch with ids remapped into it, ready for
    SortModel.set_item_table(). `gather(shard, local_ids) -> rows` defaults to the CUDA
    kernel; the CPU gloo tests pass torch.index_select to exercise the exchange logic."""

    def __init__(self, shard, rows_per_rank: int, rank: int, world: int, group=None, gather=None,
                 stream_ptr: int = 0):
        self.shard, self.R, self.rank, self.world, self.group = shard, rows_per_rank, rank, world, group
        self.stream_ptr = stream_ptr
        self.gather = gather or self._cuda_gather

    def _cuda_gather(self, shard, local_ids):
        import torch
        from . import runtime as R
        out = torch.empty((local_ids.numel(), shard.shape[1]), dtype=shard.dtype, device=shard.device)
        R.gather_rows(shard.data_ptr(), shard.shape[0], shard.shape[1] * shard.element_size(),
                      local_ids.data_ptr(), local_ids.numel(), out.data_ptr(), self.stream_ptr)
        return out

    def _a2a(self, out, inp, out_splits, in_splits):
        import torch.distributed as dist
        dist.all_to_all_single(out, inp, out_splits, in_splits, group=self.group)

    def lookup(self, batch: Dict):
        """batch: dict of torch tensors with "hist_item" [B, H] and "cand_item" [B, N] on this
        rank's device. Returns (table [n_unique, dim], batch with remapped int32 item ids)."""
        import torch
        hist, cand = batch["hist_item"], batch["cand_item"]
        ids = torch.cat([hist.reshape(-1), cand.reshape(-1)]).to(torch.int64)
        uniq, inv = torch.unique(ids, sorted=True, return_inverse=True)
        # range check BEFORE any collective, agreed over the ranks: a rank that raised alone
        # would leave its peers blocked inside the all-to-all (reference: check_id,
        # tokenizer.cpp:14-19 -> ConfigError)
        bad = torch.zeros(1, dtype=torch.int32, device=ids.device)
        if uniq.numel():
            bad[0] = ((uniq[0] < 0) | (uniq[-1] >= self.world * self.R)).to(torch.int32)
        if self.world > 1:
            import torch.distributed as dist
            dist.all_reduce(bad, op=dist.ReduceOp.MAX, group=self.group)
        if int(bad.item()):
            from .config import ConfigError
            raise ConfigError(f"tokenizer: item id outside vocabulary of size {self.world * self.R} "
                              f"(sharded table, detected on at least one rank)")
        owner = torch.div(uniq, self.R, rounding_mode="floor")
        if self.world == 1:
            rows = self.gather(self.shard, uniq)
        else:
            send = torch.bincount(owner, minlength=self.world)
            recv = torch.empty_like(send)
            self._a2a(recv, send, [1] * self.world, [1] * self.world)
            send_l, recv_l = send.tolist(), recv.tolist()
            req = torch.empty(sum(recv_l), dtype=torch.int64, device=ids.device)
            self._a2a(req, uniq, recv_l, send_l)
            local = self.gather(self.shard, req - self.rank * self.R)
            dim = self.shard.shape[1]
            rows = torch.empty((uniq.numel(), dim), dtype=self.shard.dtype, device=ids.device)
            self._a2a(rows.view(-1), local.reshape(-1), [n * dim for n in send_l], [n * dim for n in recv_l])
        out = dict(batch)
        nh = hist.numel()
        out["hist_item"] = inv[:nh].reshape(hist.shape).to(torch.int32).contiguous()
        out["cand_item"] = inv[nh:].reshape(cand.shape).to(torch.int32).contiguous()
        return rows, out
