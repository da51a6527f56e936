# SPDX-License-Identifier: Apache-2.0
"""The library's row-sharded item lookup (csrc/exchange.cuh, sort_exchange_lookup) on the GPU:

* 2 ranks sharing GPU 0 over the host transport (gloo moves the staged payloads): every
  rank's lookup against the row-sharded table equals the full-table rows bit for bit, and
  SORT-base scores through sort_set_item_table equal the full-table forward bit for bit;
  an out-of-vocabulary id on one rank is a ConfigError on BOTH ranks (no hang);
* 1 rank over NCCL (the production transport; N > 1 needs N GPUs): identical to the full
  table; the gradient all-reduce is the identity at world 1.
Reference: item_table_.value.row(id) in history_concat_row / candidate_concat_row
(tokenizer.cpp:95-127)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, q):
    import sys
    sys.path[:0] = [ROOT]
    import torch
    import torch.distributed as dist
    from paper_2603_03988_b200 import runtime as R, synth
    from paper_2603_03988_b200.config import ConfigError, tiny_config
    from paper_2603_03988_b200.sharding import ShardedItemTable
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    dev = torch.device("cuda", 0)
    cfg = tiny_config(n_items=4000)
    P = synth.make_params(cfg, seed=3)
    full = torch.from_numpy(synth.bf16_round(P["tok.item_table"])).to(torch.bfloat16).to(dev)
    Rr = cfg.n_items // world
    shard = full[rank * Rr:(rank + 1) * Rr].contiguous()
    x = R.Exchange.host(rank, world, 0)
    tab = ShardedItemTable(shard, Rr, rank, world, x)
    b = synth.make_batch(cfg, 3, seed=20 + rank)  # each rank serves different requests
    tb = {k: torch.from_numpy(v).to(dev) for k, v in b.items()}
    rows, mapped = tab.lookup(tb)
    torch.cuda.synchronize()
    ok = torch.equal(rows[mapped["hist_item"].long()], full[tb["hist_item"].long()])
    ok = ok and torch.equal(rows[mapped["cand_item"].long()], full[tb["cand_item"].long()])
    gm = R.SortModel(cfg, P, device=0, max_batch=3)
    p_full = gm.forward(b)
    gm.set_item_table(rows.data_ptr(), rows.shape[0])
    p_sh = gm.forward({k: v.cpu().numpy() for k, v in mapped.items()})
    gm.set_item_table(0, 0)
    ok = ok and np.array_equal(p_full, p_sh)
    bad = {k: v.clone() for k, v in tb.items()}
    if rank == 1:
        bad["cand_item"][0, 0] = cfg.n_items + 7
    try:
        tab.lookup(bad)
        ok = False
    except ConfigError:
        pass
    # the gradient sum over the host transport
    g = torch.full((1000,), float(rank + 1), device=dev)
    x.allreduce(g.data_ptr(), g.numel())
    ok = ok and bool(torch.all(g == 3.0))
    oks = [None] * world
    dist.all_gather_object(oks, bool(ok))
    if rank == 0:
        q.put(all(oks))
    dist.destroy_process_group()


def test_two_ranks_one_gpu_host_transport():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok


def test_nccl_world_one_lookup_and_allreduce():
    import torch
    from paper_2603_03988_b200 import runtime as R
    from paper_2603_03988_b200.sharding import ShardedItemTable
    dev = torch.device("cuda", 0)
    table = (torch.randn((5000, 32), device=dev) * 0.1).to(torch.bfloat16)
    x = R.Exchange.nccl(0, 1, 0)
    tab = ShardedItemTable(table, 5000, 0, 1, x)
    ids = {"hist_item": torch.randint(0, 5000, (4, 100), device=dev, dtype=torch.int32),
           "cand_item": torch.randint(0, 5000, (4, 9), device=dev, dtype=torch.int32)}
    rows, mapped = tab.lookup(ids)
    torch.cuda.synchronize()
    assert torch.equal(rows[mapped["hist_item"].long()], table[ids["hist_item"].long()])
    assert torch.equal(rows[mapped["cand_item"].long()], table[ids["cand_item"].long()])
    g = torch.arange(100, dtype=torch.float32, device=dev)
    x.allreduce(g.data_ptr(), 100)
    assert torch.equal(g, torch.arange(100, dtype=torch.float32, device=dev))
    x.close()
