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


def _transport_worker(rank, world, port, out_q):
    import ctypes as C
    import sys
    here = os.path.dirname(os.path.abspath(__file__))
    sys.path[:0] = [os.path.dirname(here)]
    import torch.distributed as dist
    from paper_2603_03988_b200 import runtime as R
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    a2a, red = R.host_transport()
    # rank r sends (r + 1) * (p + 1) bytes of value 10 r + p to rank p
    send_b = (C.c_int64 * world)(*[(rank + 1) * (p + 1) for p in range(world)])
    recv_b = (C.c_int64 * world)(*[(p + 1) * (rank + 1) for p in range(world)])
    payload = bytes(b for p in range(world) for b in [10 * rank + p] * ((rank + 1) * (p + 1)))
    send = (C.c_uint8 * len(payload)).from_buffer_copy(payload)
    recv = (C.c_uint8 * sum(recv_b))()
    ok = a2a(None, C.addressof(send), send_b, C.addressof(recv), recv_b, world) == 0
    want = bytes(b for p in range(world) for b in [10 * p + rank] * ((p + 1) * (rank + 1)))
    ok = ok and bytes(recv) == want
    buf = (C.c_float * 5)(*[float(rank + i) for i in range(5)])
    ok = ok and red(None, buf, 5) == 0
    ok = ok and list(buf) == [float(sum(r + i for r in range(world))) for i in range(5)]
    oks = [None] * world
    dist.all_gather_object(oks, ok)
    if rank == 0:
        out_q.put(all(oks))
    dist.destroy_process_group()


def test_two_rank_gloo_exchange_host_transport():
    """Embedding-heavy path (configs[4]) / data-parallel gradient sum: the host transport the
    library's C++ exchange (csrc/exchange.cuh) calls back into -- all-to-all-v of byte blocks
    and the in-place float sum -- moves exactly the right bytes between 2 gloo ranks. (The
    device side of the exchange runs in tests/test_gpu_exchange.py.)"""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_transport_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    ok = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert ok
