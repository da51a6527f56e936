"""Where the e2e time goes beyond the device-resident forward: the same async serving loop
with and without the in-loop L2 flush, and the flush alone (CUDA events)."""
import ctypes
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch

from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config

cfg = base_config()
B = 256
dev = torch.device("cuda", 0)
model = R.SortModel(cfg, synth.make_params(cfg, seed=5), device=0, max_batch=B)
stream = torch.cuda.Stream(device=dev)
model.set_stream(stream.cuda_stream)
batch = synth.make_batch(cfg, B, seed=100)
pinned = {k: torch.from_numpy(v).pin_memory() for k, v in batch.items()}
host_scores = torch.empty((B, cfg.n_cand, 3), dtype=torch.float32).pin_memory()
c = R.CSortBatch(B, *[pinned[k].data_ptr() for k in R._BatchHold.KEYS])
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
steps = 40
with torch.cuda.stream(stream):
    for _ in range(3):
        R._check(R.lib().sort_forward_async(model.h, ctypes.byref(c), host_scores.data_ptr()))
    model.sync()
    for use_flush in (True, False, True, False):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(steps):
            if use_flush:
                flush.fill_(float(i))
            R._check(R.lib().sort_forward_async(model.h, ctypes.byref(c), host_scores.data_ptr()))
        model.sync()
        print(f"async loop, flush={use_flush}: {(time.perf_counter() - t0) * 1e3 / steps:.4f} ms/step", flush=True)
    dev_batch = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
    db = R._DevBatch(dev_batch)
    scores = torch.empty((B, cfg.n_cand, 3), dtype=torch.float32, device=dev)
    for use_flush in (True, False):
        ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(steps)]
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i in range(steps):
            if use_flush:
                flush.fill_(float(i))
            ev[i][0].record(stream)
            model.forward_device(db, scores.data_ptr())
            ev[i][1].record(stream)
        model.sync()
        wall = (time.perf_counter() - t0) * 1e3 / steps
        devt = sum(a.elapsed_time(b) for a, b in ev) / steps
        print(f"device-resident loop, flush={use_flush}: events {devt:.4f} ms/step, wall {wall:.4f} ms/step", flush=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream)
    for i in range(steps):
        flush.fill_(float(i))
    e1.record(stream)
    torch.cuda.synchronize()
    print(f"flush alone: {e0.elapsed_time(e1) / steps:.4f} ms", flush=True)
