# SPDX-License-Identifier: Apache-2.0
"""SORT-base forward throughput on B200 (BASELINE.json metric: candidates scored/sec and
tensor-pipe MFU, SORT forward at 1/2/4/8 B200).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

One step = one SORT-base forward (tokenizer -> 4 blocks with pruning after layer 2 ->
fp32 head) over 256 synthetic requests x (1024 history + 64 targets) per GPU. Multi-GPU
runs are launched with torchrun, one process per GPU; requests shard across ranks with no
data-path collective (weak scaling, 256 requests per GPU); a barrier + synchronize bracket
the timed region and the reported time is the max over ranks.

value   : device-resident throughput (inputs already in HBM), CUDA events on the library's
          stream, L2 flushed (256 MB write) before every timed step, summed over K steps.
e2e     : the same forward through the C ABI with pinned HOST inputs and a host score
          buffer (H2D of the batch + D2H of the scores inside the timed region).
--impl reference: the reference algorithm's CPU implementation (the fp64 oracle restating
          rankformer::, since the reference itself does not build here -- DESIGN.md) on all
          host cores, bounded samples of the same workload.
"""
from __future__ import annotations

import argparse
import json
import os
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

from paper_2603_03988_b200 import synth  # noqa: E402
from paper_2603_03988_b200.config import base_config  # noqa: E402
from paper_2603_03988_b200.flops import forward_flops  # noqa: E402

METRIC = "candidates scored/sec (SORT-base forward)"
UNIT = "candidates/s"
REQ_PER_GPU = 256


def workload_desc(cfg):
    return (f"SORT-base: {cfg.layers} layers, d={cfg.model_dim}, {cfg.heads} heads, m={cfg.ffn_dim}, "
            f"{REQ_PER_GPU} requests/GPU x ({cfg.n_hist} history + {cfg.n_cand} targets), "
            f"L={cfg.seq_len}, W={cfg.local_window}, F={cfg.full_suffix}, keep={cfg.keep_schedule()}")


def bench_config(cfg, world, B):
    """The `config` object of BOTH arms (ours and --impl reference): it names the workload
    only, so the driver can compare the two lines key for key."""
    return {"workload": workload_desc(cfg), "global_batch": world * B, "requests_per_gpu": B,
            "seq_len": cfg.seq_len, "parallelism": f"dp{world} (request-sharded replicas, no forward collective)",
            "l2": "flushed (256 MB write) before every timed step",
            "weights": "random init (synth.make_params, fan-in), bf16-rounded"}


def cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    import platform
    return platform.processor() or "unknown"


def measured_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            p = json.load(f)
        return p, "measured"
    except Exception:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, "fallback"


class ClockSampler:
    """nvidia-smi style clock / throttle sampling during the timed region (NVML)."""

    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap",
               0x8: "hw_slowdown", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
               0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        self.stop = threading.Event()
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception:
            self.max_mhz = None

    def _run(self):
        while not self.stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.02)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self.stop.set()
            self.t.join()

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": sorted(self.reasons),
                    "samples": 0}
        return {"sm_mhz": float(np.median(self.samples)), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


class CpuReference:
    """The CPU reference algorithm (fp64 oracle port of rankformer::, dense masked attention as
    attention.cpp:118-121), one request per host thread.

    A sample is time-bounded: chunks of `threads` requests are scored until at least
    `min_requests` requests and `target_s` seconds of work are done."""

    def __init__(self, cfg, params, threads):
        sys.path.insert(0, os.path.join(ROOT, "oracle"))
        import oracle as O
        self.cfg, self.threads = cfg, threads
        self.om = O.OracleModel(cfg, params)
        self.batch = synth.make_batch(cfg, threads, seed=1000)

    def sample(self, target_s, min_requests):
        n, t0 = 0, time.perf_counter()
        while True:
            self.om.forward_batch(self.batch, threads=self.threads)
            n += self.threads
            dt = time.perf_counter() - t0
            if dt >= target_s and n >= min_requests:
                return n * self.cfg.n_cand / dt, dt, n


def run_reference(args, cfg, rank, world):
    if rank != 0:
        return
    threads = os.cpu_count() or 1
    params = synth.make_params(cfg, seed=5)
    ref = CpuReference(cfg, params, threads)
    # each step is a bounded sample so that --steps K --warmup W ends within ~3 minutes
    per_step = min(20.0, max(1.0, 150.0 / max(1, args.steps + min(args.warmup, 1))))
    if args.warmup:
        ref.sample(0.0, threads)  # one untimed warm-up chunk (page-in, allocator)
    total_c, total_t, total_r = 0.0, 0.0, 0
    for _ in range(args.steps):
        rate, dt, n = ref.sample(per_step, 1)
        total_c += n * cfg.n_cand
        total_t += dt
        total_r += n
    value = total_c / total_t
    sample = (f"{total_r} SORT-base requests over {args.steps} steps ({int(total_c)} candidates, "
              f"{total_t:.1f} s), fp64 oracle port, one request per thread, {threads} threads on "
              f"{cpu_model()}")
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": total_t / args.steps * 1e3,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic", "config": bench_config(cfg, world, args.requests),
        "execution": f"CPU: {threads} host threads ({cpu_model()}), one request per thread",
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "cpu_model": cpu_model(), "sample": sample},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


def run_train(args, cfg, rank, world, local, dist):
    """BASELINE configs[2]: SORT-base training step (forward + backward of the scoring path,
    sort_train_step) with the global batch sharded over the ranks and the flat fp32 gradient
    all-reduced over NCCL (torch.distributed) every step. Loss: mean BCE of the three heads
    against synthetic labels;
    ranking loss and dL/dlogits computed on the device, AdamW step on the
    fp32 masters and the bf16 inference weights rebuilt on the device every step."""
    import torch
    from paper_2603_03988_b200 import runtime as R
    from paper_2603_03988_b200.sharding import shard_range
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    b0, b1 = shard_range(args.requests, world, rank)
    B = b1 - b0
    params = synth.make_params(cfg, seed=5)
    model = R.SortModel(cfg, params, device=local, max_batch=B)
    full = synth.make_batch(cfg, args.requests, seed=100)
    batch = {k: np.ascontiguousarray(v[b0:b1]) for k, v in full.items()}
    labels = (np.random.default_rng(7).random((args.requests, cfg.n_cand, 3)) < 0.2).astype(np.float32)[b0:b1]
    gbuf = torch.zeros(model.grad_layout()[3], dtype=torch.float32, device=dev)
    exchange = R.Exchange.nccl(rank, world, local) if dist else None  # gradient sum in the C++ host (NCCL)
    # per-rank mean BCE scaled by 1/world: the all-reduced sum is the global-batch mean
    w_obj = np.array([1.0, 0.5, 0.5], np.float32) / world
    losses = []

    def step():
        losses.append(model.train_step_bce(batch, labels, w_obj))  # fwd + loss + bwd on device
        if dist:
            model.grads_to_device(gbuf.data_ptr())
            exchange.allreduce(gbuf.data_ptr(), gbuf.numel())
            model.grads_to_device(gbuf.data_ptr(), to_handle=True)
        model.adamw_step(lr=2e-4)  # PAPER.md:4.1.3 base lr, beta (0.9, 0.99), wd 0.01
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    if rank == 0:
        print(json.dumps({
            "metric": "requests trained/sec (SORT-base forward+backward+AdamW, data parallel)",
            "value": args.requests / (ms / 1e3), "unit": "requests/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
            "higher_is_better": True, "scaling": "strong", "vs_baseline": None, "dtype": "bf16/fp32",
            "data": "synthetic",
            "loss_first_last": [losses[0], losses[-1]],
            "config": {"workload": workload_desc(cfg) + " -- training step, weighted BCE on 3 heads, AdamW",
                       "global_batch": args.requests, "requests_per_gpu": B,
                       "parallelism": f"dp{world} (request shards, NCCL all-reduce of "
                                      f"{model.grad_layout()[3]} fp32 gradients per step)"},
            "timing": "wall clock per synchronized step (host-driven: the step returns logits "
                      "and gradients), max over ranks",
        }))
    if dist:
        dist.destroy_process_group()


def run_pretrain_train(args, rank, world, local, dist):
    """SURVEY 8(f) "next 4" training: pre-training step (sort_pretrain_train_step: forward of 64
    click sequences x 1024 clicks, mean full-softmax next-item CE over a 65,536-item vocabulary,
    backward of every parameter incl. the tied item table) + AdamW, per rank; gradients summed
    over the ranks by the C++ exchange (NCCL) when N > 1."""
    import torch
    from paper_2603_03988_b200 import runtime as R
    from paper_2603_03988_b200.config import pretrain_config
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = pretrain_config()
    B = cfg.batch
    model = R.SortModel(cfg, synth.make_params(cfg, seed=5), device=local, max_batch=B)
    batch = synth.make_batch(cfg, B, seed=100 + rank)
    gbuf = torch.zeros(model.grad_layout()[3], dtype=torch.float32, device=dev)
    exchange = R.Exchange.nccl(rank, world, local) if dist else None
    losses = []

    def step():
        losses.append(model.pretrain_train_step(batch))
        if dist:  # dense gradients (the item-table gradient stays per rank in this build)
            model.grads_to_device(gbuf.data_ptr())
            exchange.allreduce(gbuf.data_ptr(), gbuf.numel())
            model.grads_to_device(gbuf.data_ptr(), to_handle=True)
        model.adamw_step(lr=2e-4)
        torch.cuda.synchronize(dev)

    for _ in range(args.warmup):
        step()
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    if rank == 0:
        print(json.dumps({
            "metric": "next-item positions trained/sec (pre-training forward+backward+AdamW)",
            "value": world * B * cfg.n_hist / (ms / 1e3), "unit": "positions/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16/fp32 (bf16 dL/dlogits)", "data": "synthetic",
            "loss_first_last": [losses[0], losses[-1]],
            "config": {"workload": f"pre-training step: {cfg.layers} layers, d={cfg.model_dim}, {cfg.heads} heads, "
                                   f"m={cfg.ffn_dim}, {B} sequences/GPU x {cfg.n_hist} clicks, vocab {cfg.n_items}, "
                                   "tied full-softmax CE, item table trained",
                       "requests_per_gpu": B, "parallelism": f"dp{world}"},
            "timing": "wall clock per synchronized step (host-driven), max over ranks",
        }))
    if dist:
        dist.destroy_process_group()


def run_embed(args, cfg, rank, world, local, dist):
    """BASELINE configs[4]: SORT-base scoring whose item table (--table-rows x item_dim bf16,
    6.4 GB at 100M rows) is row-sharded over the ranks. Per step and rank, inside the C++
    library (sort_exchange_lookup over NCCL): group the shard's 256 requests' item ids by
    owner, all-to-all ids to their owners, owner-side CUDA gather, all-to-all rows back,
    batch-order scatter -> batch-local table -> sort_set_item_table -> SORT-base forward."""
    import torch
    from paper_2603_03988_b200 import runtime as R
    from paper_2603_03988_b200.sharding import ShardedItemTable
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    rows_per_rank = (args.table_rows + world - 1) // world
    g = torch.Generator(device=dev)
    g.manual_seed(1000 + rank)
    shard = (torch.randn((rows_per_rank, cfg.item_dim), generator=g, device=dev) * 0.1).to(torch.bfloat16)
    small = base_config(batch=args.requests, n_items=1024)  # the handle's own table is unused
    model = R.SortModel(small, synth.make_params(small, seed=5), device=local, max_batch=args.requests)
    stream = torch.cuda.Stream(device=dev)
    model.set_stream(stream.cuda_stream)
    rng = np.random.default_rng(100 + rank)
    B = args.requests
    batch = synth.make_batch(small, B, seed=100 + rank)
    batch["hist_item"] = rng.integers(0, args.table_rows, size=batch["hist_item"].shape, dtype=np.int64).astype(np.int32)
    batch["cand_item"] = np.stack([rng.choice(args.table_rows, size=cfg.n_cand, replace=False)
                                   for _ in range(B)]).astype(np.int32)
    tb = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    exchange = R.Exchange.nccl(rank, world, local)
    table = ShardedItemTable(shard, rows_per_rank, rank, world, exchange, stream_ptr=stream.cuda_stream)
    scores = torch.empty((B, max(cfg.n_cand, 1), 3), dtype=torch.float32, device=dev)

    def step():
        with torch.cuda.stream(stream):
            rows, mapped = table.lookup(tb)
            model.set_item_table(rows.data_ptr(), rows.shape[0])
            model.forward_device(R._DevBatch(mapped), scores.data_ptr())
            model.sync()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize(dev)
    if dist:
        dist.barrier()
    t0 = time.perf_counter()
    for _ in range(args.steps):
        step()
    ms = (time.perf_counter() - t0) * 1e3 / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    if rank == 0:
        print(json.dumps({
            "metric": "candidates scored/sec (SORT-base forward, row-sharded 100M-row item table)",
            "value": world * B * cfg.n_cand / (ms / 1e3), "unit": "candidates/s", "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
            "config": {"workload": workload_desc(cfg) + f" -- item table {args.table_rows} x "
                                                        f"{cfg.item_dim} bf16 row-sharded over {world} rank(s)",
                       "requests_per_gpu": B, "ids_per_step": int(B * (cfg.n_hist + cfg.n_cand)),
                       "parallelism": f"dp{world} + row-sharded table, C++ exchange (NCCL all-to-all of ids/rows)"},
            "timing": "wall clock per synchronized step (the exchange needs host-visible counts), max over ranks",
        }))
    exchange.close()
    if dist:
        dist.destroy_process_group()


def run_large(args, rank, world, local, dist, moe=False, pretrain=False):
    """BASELINE configs[3]: SORT-large (12 layers, d=1024, 16 heads, 4096 history, W=256,
    128 targets, geometric pruning) forward, 8 requests per GPU, requests sharded over the
    ranks (weak scaling). Generic path: bf16 library GEMMs + the tcgen05 attention core.
    moe=True: SURVEY.md 8(f) "next 1", SORT-base with the DeepSeek-style MoE FFN (8 routed
    experts, top-1, 1 shared, expert width 320), 256 requests per GPU."""
    import torch
    from paper_2603_03988_b200 import runtime as R
    from paper_2603_03988_b200.config import base_moe_config, large_config, pretrain_config
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    B = args.requests if moe else (64 if pretrain else 8)
    cfg = base_moe_config(batch=B) if moe else (pretrain_config(batch=B) if pretrain else large_config(batch=B))
    model = R.SortModel(cfg, synth.make_params(cfg, seed=5), device=local, max_batch=B)
    stream = torch.cuda.Stream(device=dev)
    model.set_stream(stream.cuda_stream)
    batch = synth.make_batch(cfg, B, seed=200 + rank)
    dbatch = R._DevBatch({k: torch.from_numpy(v).to(dev) for k, v in batch.items()})
    scores = torch.empty((B, max(cfg.n_cand, 1), 3), dtype=torch.float32, device=dev)
    lse_t = torch.empty((B, cfg.n_hist), dtype=torch.float32, device=dev)
    tgt_t = torch.empty((B, cfg.n_hist), dtype=torch.float32, device=dev)

    def step():
        if pretrain:
            model.pretrain_forward_device(dbatch, lse_t.data_ptr(), tgt_t.data_ptr())
        else:
            model.forward_device(dbatch, scores.data_ptr())
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            step()
        model.sync()
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
        if dist:
            dist.barrier()
        for i in range(args.steps):
            flush.fill_(float(i))
            ev[i][0].record(stream)
            step()
            ev[i][1].record(stream)
        model.sync()
    ms = sum(a.elapsed_time(b) for a, b in ev) / args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t[0])
    fl = forward_flops(cfg)
    peaks, _ = measured_peaks()
    units = B * cfg.n_cand
    if pretrain:
        wl = (f"pre-training (causal next-item, tied full-softmax head): {cfg.layers} layers, d={cfg.model_dim}, "
              f"{cfg.heads} heads, m={cfg.ffn_dim}, {B} sequences/GPU x {cfg.n_hist} clicks, "
              f"vocab {cfg.n_items}")
        metric = "next-item positions scored/sec (pre-training forward + full-softmax CE)"
        dtype = "bf16 (fp32 accumulation, fp32 log-sum-exp)"
        units = B * cfg.n_hist
        ce_flop = 2.0 * B * cfg.seq_len * cfg.n_items * cfg.item_dim
    elif moe:
        wl = (f"SORT-base + MoE FFN: {cfg.layers} layers, d={cfg.model_dim}, {cfg.heads} heads, "
              f"{cfg.moe_experts} routed experts top-{cfg.moe_topk} + {cfg.moe_shared} shared, expert "
              f"m={cfg.moe_ffn_dim}, {B} requests/GPU x ({cfg.n_hist} history + {cfg.n_cand} targets), "
              f"keep={cfg.keep_schedule()}")
        metric = "candidates scored/sec (SORT-base MoE forward)"
        dtype = "bf16 (fp32 accumulation, fp32 router)"
    else:
        wl = (f"SORT-large: {cfg.layers} layers, d={cfg.model_dim}, {cfg.heads} heads, "
              f"m={cfg.ffn_dim}, {B} requests/GPU x ({cfg.n_hist} history + {cfg.n_cand} "
              f"targets), L={cfg.seq_len}, W={cfg.local_window}, keep={cfg.keep_schedule()}")
        metric = "candidates scored/sec (SORT-large forward)"
        dtype = "bf16 (fp32 accumulation and residual stream)"
    if rank == 0:
        print(json.dumps({
            "metric": metric, "value": world * units / (ms / 1e3),
            "unit": "positions/s" if pretrain else "candidates/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup,
            "ms_per_step": ms, "higher_is_better": True, "scaling": "weak", "vs_baseline": None,
            "dtype": dtype, "data": "synthetic",
            "mfu_vs_bf16_peak": (fl["block"] * B + (ce_flop if pretrain else fl["total"] * B - fl["block"] * B))
            / (ms / 1e3) / (peaks["bf16_tflops"] * 1e12),
            "algorithmic_tflop_per_step": (fl["block"] * B + (ce_flop if pretrain else fl["total"] * B - fl["block"] * B)) / 1e12,
            "config": {"workload": wl, "requests_per_gpu": B,
                       "l2": "flushed (256 MB write) before every timed step"},
        }))
    if dist:
        dist.destroy_process_group()


def launch_ranks(n):
    """Re-run this command under torch.distributed.run with n ranks on 127.0.0.1 (the
    driver's own multi-GPU form); rank 0 prints the JSON line."""
    import socket
    import subprocess
    with socket.socket() as sk:
        sk.bind(("127.0.0.1", 0))
        port = sk.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), os.path.abspath(__file__), *sys.argv[1:]]
    sys.exit(subprocess.call(cmd))


def run_dry(args, cfg, rank, world, dist):
    """--dry-run: the launcher, barrier and max-over-ranks plumbing of the real run on gloo
    (CPU), with a trivial host step. Used by tests/test_bench_launch.py."""
    t0 = time.perf_counter()
    acc = 0.0
    for i in range(args.warmup + args.steps):
        acc += float(np.sum(np.arange(1000 * (rank + 1), dtype=np.float64)))
    ms = (time.perf_counter() - t0) * 1e3 / max(1, args.steps)
    t = [ms]
    if dist:
        import torch
        tt = torch.tensor(t, dtype=torch.float64)
        dist.all_reduce(tt, op=dist.ReduceOp.MAX)
        t = tt.tolist()
        ranks = torch.tensor([1.0])
        dist.all_reduce(ranks)
        n_ranks = int(ranks.item())
    else:
        n_ranks = 1
    if rank == 0:
        print(json.dumps({"metric": METRIC, "value": None, "unit": UNIT, "n_gpus": world, "steps": args.steps,
                          "warmup": args.warmup, "ms_per_step": t[0], "dry_run": True, "ranks_seen": n_ranks,
                          "config": bench_config(cfg, world, args.requests)}), flush=True)
    if dist:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--requests", type=int, default=REQ_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--cpu-seconds", type=float, default=12.0,
                    help="minimum length of the CPU-baseline sample (>= 32 requests)")
    ap.add_argument("--mode", default="forward", choices=["forward", "train", "embed", "large", "moe", "pretrain", "pretrain_train"],
                    help="train: SORT-base training step (BASELINE configs[2]), global batch "
                         "--requests sharded over the ranks, gradient all-reduce over NCCL; "
                         "embed: BASELINE configs[4], 100M-row item table row-sharded over the "
                         "ranks, all-to-all tokenization feeding SORT-base")
    ap.add_argument("--table-rows", type=int, default=100_000_000)
    ap.add_argument("--profile-launches", action="store_true",
                    help="short run for ncu launch lists (no CPU leg, no e2e)")
    ap.add_argument("--dry-run", action="store_true",
                    help="launcher check without a GPU: N gloo ranks, barrier + max-over-ranks "
                         "timing of a trivial host step, one JSON line from rank 0")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if not args.profile_launches else args.warmup

    if "WORLD_SIZE" not in os.environ and args.gpus > 1 and args.impl == "ours":
        # `python bench.py --gpus N` launches its own N ranks (one process per GPU) exactly as
        # the driver's torchrun form does; this process only waits for them
        launch_ranks(args.gpus)
        return

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if "WORLD_SIZE" not in os.environ and args.impl == "reference":
        world = args.gpus  # CPU arm: rank 0's work only, reported for the N-GPU run it sits beside
    elif world != args.gpus:
        print(f"bench.py: WORLD_SIZE={world} overrides --gpus {args.gpus}", file=sys.stderr)
    cfg = base_config(batch=args.requests)

    import torch
    dist = None
    if "WORLD_SIZE" in os.environ and world > 1:
        import torch.distributed as dist
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        use_nccl = args.impl == "ours" and not args.dry_run
        torch.cuda.set_device(local) if use_nccl else None
        dist.init_process_group("nccl" if use_nccl else "gloo")

    if args.dry_run:
        run_dry(args, cfg, rank, world, dist)
        return

    if args.impl == "reference":
        run_reference(args, cfg, rank, world)
        if dist:
            dist.barrier()
            dist.destroy_process_group()
        return

    if args.mode == "train":
        run_train(args, cfg, rank, world, local, dist)
        return
    if args.mode == "pretrain_train":
        return run_pretrain_train(args, rank, world, local, dist)
    if args.mode == "embed":
        run_embed(args, cfg, rank, world, local, dist)
        return
    if args.mode in ("large", "moe", "pretrain"):
        run_large(args, rank, world, local, dist, moe=args.mode == "moe", pretrain=args.mode == "pretrain")
        return

    from paper_2603_03988_b200 import runtime as R
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    params = synth.make_params(cfg, seed=5)  # replicated weights (same seed on every rank)
    model = R.SortModel(cfg, params, device=local, max_batch=args.requests)
    stream = torch.cuda.Stream(device=dev)
    model.set_stream(stream.cuda_stream)
    B = args.requests
    batch = synth.make_batch(cfg, B, seed=100 + rank)  # this rank's shard of requests
    dev_batch = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    dbatch = R._DevBatch(dev_batch)
    scores = torch.empty((B, max(cfg.n_cand, 1), 3), dtype=torch.float32, device=dev)
    flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)  # 256 MB > 126 MB L2

    def barrier():
        torch.cuda.synchronize(dev)
        if dist:
            dist.barrier()
        torch.cuda.synchronize(dev)

    # ---------------------------------------------------------------- device-resident timing
    with torch.cuda.stream(stream):
        for _ in range(args.warmup):
            model.forward_device(dbatch, scores.data_ptr())
        model.sync()
        if args.profile_launches:
            for _ in range(args.steps):
                model.forward_device(dbatch, scores.data_ptr())
            model.sync()
            return
        starts = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        ends = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps)]
        launches_per_step = 0
        barrier()
        with ClockSampler(local) as clk:
            for i in range(args.steps):
                flush.fill_(float(i))  # evict L2 between timed steps (untimed)
                starts[i].record(stream)
                model.forward_device(dbatch, scores.data_ptr())
                ends[i].record(stream)
                launches_per_step = model.kernel_count()
            model.sync()
            barrier()
        dev_ms = sum(s.elapsed_time(e) for s, e in zip(starts, ends))

    # ---------------------------------------------------------------- e2e through the C ABI
    pinned = {k: torch.from_numpy(v).pin_memory() for k, v in batch.items()}
    host_scores = torch.empty((B, cfg.n_cand, 3), dtype=torch.float32).pin_memory()

    class _PinnedBatch(R._BatchHold):
        def __init__(self, t):
            self.t = t
            self.c = R.CSortBatch(B, *[t[k].data_ptr() for k in R._BatchHold.KEYS])

    pb = _PinnedBatch(pinned)
    import ctypes
    h2d = sum(int(v.nbytes) for v in batch.values())
    d2h = int(host_scores.numel() * 4)
    for _ in range(2):
        R._check(R.lib().sort_forward(model.h, ctypes.byref(pb.c), 0,
                                      ctypes.c_void_p(host_scores.data_ptr()), 0))
    barrier()
    # (a) one synchronous call per step (copy in, forward, copy out, sync), L2 flushed
    #     outside the timed region
    e2e_sync_ms = 0.0
    for i in range(args.steps):
        flush.fill_(float(i))
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        R._check(R.lib().sort_forward(model.h, ctypes.byref(pb.c), 0,
                                      ctypes.c_void_p(host_scores.data_ptr()), 0))
        e2e_sync_ms += (time.perf_counter() - t0) * 1e3
    barrier()
    # (b) the serving loop: sort_forward_async per step (each step's host->device copy rides
    #     the copy stream and overlaps the previous step's kernels; scores copied back every
    #     step), the L2 flush enqueued before every step INSIDE the timed region, one sync at
    #     the end. This is the e2e value.
    with torch.cuda.stream(stream):
        for _ in range(2):
            R._check(R.lib().sort_forward_async(model.h, ctypes.byref(pb.c), host_scores.data_ptr()))
        model.sync()
        barrier()
        torch.cuda.synchronize(dev)
        t0 = time.perf_counter()
        for i in range(args.steps):
            flush.fill_(float(i))
            R._check(R.lib().sort_forward_async(model.h, ctypes.byref(pb.c), host_scores.data_ptr()))
        model.sync()
        e2e_ms = (time.perf_counter() - t0) * 1e3
    barrier()

    # ---------------------------------------------------------------- per-stage breakdown
    model.enable_stage_timing(True)
    with torch.cuda.stream(stream):
        stage_acc = {}
        for i in range(3):
            flush.fill_(float(i))
            model.forward_device(dbatch, scores.data_ptr())
            model.sync()
            for k, v in model.stage_times().items():
                stage_acc[k] = stage_acc.get(k, 0.0) + v / 3
    model.enable_stage_timing(False)

    t = torch.tensor([dev_ms, e2e_ms, e2e_sync_ms], dtype=torch.float64, device=dev)
    if dist:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    dev_ms, e2e_ms, e2e_sync_ms = float(t[0]), float(t[1]), float(t[2])
    if rank != 0:
        dist.destroy_process_group() if dist else None
        return

    cand_per_step = world * B * cfg.n_cand
    value = cand_per_step * args.steps / (dev_ms / 1e3)
    e2e_value = cand_per_step * args.steps / (e2e_ms / 1e3)
    fl = forward_flops(cfg)
    peaks, peak_kind = measured_peaks()
    step_flops = fl["total"] * B
    mfu = step_flops / (dev_ms / args.steps / 1e3) / (peaks["bf16_tflops"] * 1e12)

    # dominant kernel (largest stage group) -> roofline entry
    groups = {}
    for k, v in stage_acc.items():
        g = k.split(".")[-1]
        groups[g] = groups.get(g, 0.0) + v
    per_group_flops = {
        "attention": fl["attn"] * B, "qkvg": sum(2 * 2 * (L["l_q"] + L["l_kv"]) * cfg.model_dim ** 2
                                                  for L in fl["layers"]) * B,
        "wo": sum(2 * L["l_q"] * cfg.model_dim ** 2 for L in fl["layers"]) * B,
        "ffn_up": sum(2 * 2 * L["l_q"] * cfg.model_dim * cfg.ffn_dim for L in fl["layers"]) * B,
        "ffn_down": sum(2 * L["l_q"] * cfg.model_dim * cfg.ffn_dim for L in fl["layers"]) * B,
        "head": fl["head"] * B, "tokenizer": fl["tokenizer"] * B,
    }
    dom = max(groups, key=groups.get) if groups else "attention"
    n_launch = 4 if dom in ("attention", "qkvg", "wo", "ffn_up", "ffn_down") else 1
    dom_ms = groups.get(dom, 0.0)
    achieved = per_group_flops.get(dom, 0.0) / (dom_ms / 1e3) / 1e12 if dom_ms else None
    traffic = None
    prof = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(prof):
        try:
            traffic = json.load(open(prof)).get(dom)
        except Exception:
            traffic = None
    roofline = {
        "kernel": dom, "bound": "tensor", "achieved": achieved, "peak": peaks["bf16_tflops"],
        "unit": "TFLOP/s", "frac": (achieved / peaks["bf16_tflops"]) if achieved else None,
        "traffic": traffic, "peak_kind": f"{peak_kind} (MEASURED_PEAKS.json bf16_tflops)",
        "launches_per_step": n_launch, "ms_per_step": dom_ms,
        "algorithmic_flops_per_step": per_group_flops.get(dom),
        "stage_ms": {k: round(v, 4) for k, v in groups.items()},
    }
    if dom == "attention" and dom_ms:
        # the attention core's binding unit is the exp (MUFU), one per visible logit: report
        # that roofline next to the tensor one (peak: tools/micro/mufu_peak.cu on a B200)
        mufu = os.path.join(ROOT, "profiles", "mufu_peak.json")
        mufu_peak = 4.61e12
        if os.path.exists(mufu):
            try:
                mufu_peak = json.loads(open(mufu).readline())["ex2_per_s"]
            except Exception:
                pass
        exps = sum(L["visible_per_head"] for L in fl["layers"]) * cfg.heads * B
        roofline["exp_roofline"] = {
            "bound": "mufu", "achieved": exps / (dom_ms / 1e3) / 1e12, "peak": mufu_peak / 1e12,
            "unit": "Texp/s", "frac": exps / (dom_ms / 1e3) / mufu_peak,
            "algorithmic_exps_per_step": exps,
            "peak_kind": "measured (profiles/mufu_peak.json: ex2.approx throughput, 16/clk/SM)"}

    cpu = None
    if world == 1 and not args.no_cpu_baseline:
        threads = os.cpu_count() or 1
        ref = CpuReference(cfg, params, threads)
        rate, dt, n_req = ref.sample(args.cpu_seconds, 32)
        cpu = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port", "cpu_model": cpu_model(),
               "sample": f"{n_req} SORT-base requests ({n_req * cfg.n_cand} candidates) in "
                         f"{dt:.1f} s, fp64 oracle port of the reference, one request per thread, "
                         f"{threads} threads on {cpu_model()}"}

    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": dev_ms / args.steps, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "bf16", "data": "synthetic",
        "config": bench_config(cfg, world, B),
        "mfu": mfu, "mfu_peak": f"{peaks['bf16_tflops']} TFLOP/s bf16 ({peak_kind})",
        "algorithmic_tflop_per_step": step_flops * world / 1e12,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": h2d,
                "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms / args.steps,
                "form": "pipelined sort_forward_async loop, L2 flush inside the timed region",
                "sync_call_ms_per_step": e2e_sync_ms / args.steps},
        "gpu_launches": launches_per_step * args.steps,
        "roofline": roofline, "cpu_baseline": cpu, "clocks": clk.summary(),
    }
    print(json.dumps(line), flush=True)
    if dist:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
