# SPDX-License-Identifier: Apache-2.0
"""N>1 host path on CPU: 2-rank gloo process group exercising request sharding, the scores
gather and the max-over-ranks timing reduction that bench.py uses under torchrun. The
per-rank "scores" come from the CPU oracle so the test also checks that sharded scoring
reproduces the unsharded result exactly (requests are independent)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

from paper_2603_03988_b200 import sharding as S


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_shard_range_partitions_exactly():
    for total in (0, 1, 5, 16, 256, 257):
        for world in (1, 2, 3, 4, 8):
            seen = []
            for r in range(world):
                b, e = S.shard_range(total, world, r)
                seen.extend(range(b, e))
                assert e - b in (total // world, total // world + 1)
            assert seen == list(range(total))


def _worker(rank, world, port, out_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle")]
    import torch.distributed as dist
    import oracle as O
    from paper_2603_03988_b200 import synth
    from paper_2603_03988_b200.config import tiny_config
    from paper_2603_03988_b200 import sharding as S2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = tiny_config()
    P = synth.make_params(cfg, seed=3)
    batch = synth.make_batch(cfg, 5, seed=9)
    local = S2.shard_batch(batch, world, rank)
    om = O.OracleModel(cfg, P)
    scores = np.stack([om.forward(local, i)[0] for i in range(local["req_ts"].shape[0])]) \
        if local["req_ts"].shape[0] else np.zeros((0, cfg.n_cand, 3))
    full = S2.gather_scores(scores.astype(np.float32), world, rank)
    t = S2.max_over_ranks([float(rank + 1), 10.0 - rank], world)
    if rank == 0:
        ref = np.stack([om.forward(batch, i)[0] for i in range(5)]).astype(np.float32)
        out_q.put((bool(np.array_equal(full, ref)), t))
    dist.destroy_process_group()


def test_two_rank_gloo_sharded_scoring_and_max_time():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok, t = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
    assert t == [2.0, 10.0]


def _grad_worker(rank, world, port, out_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here), os.path.join(os.path.dirname(here), "oracle")]
    import torch
    import torch.distributed as dist
    import oracle as O
    from paper_2603_03988_b200 import synth
    from paper_2603_03988_b200.config import tiny_config
    from paper_2603_03988_b200 import sharding as S2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    cfg = tiny_config(n_hist=40, n_cand=5, keep=[46, 20], local_window=8, full_suffix=6)
    P = synth.make_params(cfg, seed=3)
    names = sorted(n for n in P if not n.startswith("tok."))
    batch = synth.make_batch(cfg, 3, seed=9)
    dz = np.random.default_rng(2).normal(size=(3, cfg.n_cand, 3))
    om = O.OracleModel(cfg, P)

    def flat_grads(b, idx):
        tot = np.zeros(sum(P[n].size for n in names))
        for j, i in enumerate(idx):
            g, _ = om.backward(b, j, dz[i], names)
            tot += np.concatenate([g[n].ravel() for n in names])
        return tot

    lo, hi = S2.shard_range(3, world, rank)
    local = flat_grads(S2.shard_batch(batch, world, rank), range(lo, hi))
    t = torch.from_numpy(local)
    S2.allreduce_grads(t, world)
    if rank == 0:
        ref = flat_grads(batch, range(3))
        out_q.put(float(np.max(np.abs(t.numpy() - ref)) / np.max(np.abs(ref))))
    dist.destroy_process_group()


def test_two_rank_gloo_gradient_allreduce_equals_full_batch():
    """Data-parallel training step (configs[2]): per-shard gradients (the oracle backward
    stands in for each rank's sort_train_step) summed by allreduce_grads equal the gradient of
    the whole batch."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_grad_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    err = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert err < 1e-12


def _table_worker(rank, world, port, out_q):
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here)]
    import torch
    import torch.distributed as dist
    from paper_2603_03988_b200 import sharding as S2
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    n_items, dim = 1000, 32
    full = torch.from_numpy(np.random.default_rng(0).normal(size=(n_items, dim)).astype(np.float32))
    R = n_items // world
    shard = full[rank * R:(rank + 1) * R].clone()
    rng = np.random.default_rng(10 + rank)  # each rank serves a different batch
    batch = {"hist_item": torch.from_numpy(rng.integers(0, n_items, (3, 50)).astype(np.int32)),
             "cand_item": torch.from_numpy(rng.integers(0, n_items, (3, 7)).astype(np.int32))}
    tab = S2.ShardedItemTable(shard, R, rank, world, gather=lambda t, i: torch.index_select(t, 0, i))
    rows, mapped = tab.lookup(batch)
    ok = all(torch.equal(rows[mapped[k].long()], full[batch[k].long()]) for k in ("hist_item", "cand_item"))
    uniq = int(torch.unique(torch.cat([batch["hist_item"].reshape(-1), batch["cand_item"].reshape(-1)])).numel())
    ok = ok and rows.shape[0] == uniq
    # an out-of-vocabulary id on ONE rank must raise on EVERY rank before any all-to-all
    # (otherwise the clean rank would block in the collective)
    bad = dict(batch)
    if rank == 1:
        bad["cand_item"] = batch["cand_item"].clone()
        bad["cand_item"][0, 0] = n_items + 5
    from paper_2603_03988_b200.config import ConfigError
    try:
        tab.lookup(bad)
        ok = False
    except ConfigError:
        pass
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    if rank == 0:
        out_q.put(all(oks))
    dist.destroy_process_group()


def test_two_rank_gloo_row_sharded_item_table_lookup():
    """Embedding-heavy path (configs[4]): a row-sharded item table served by dedupe +
    all-to-all of ids + owner gather + all-to-all of rows reproduces the full-table lookup
    bit-exactly on every rank, with one row per unique id."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_table_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
