import ctypes, os, sys, time
ROOT = "/root/repo"; sys.path.insert(0, ROOT)
import torch
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config
cfg = base_config(); B = 256; dev = torch.device("cuda", 0)
model = R.SortModel(cfg, synth.make_params(cfg, seed=5), device=0, max_batch=B)
stream = torch.cuda.Stream(device=dev); model.set_stream(stream.cuda_stream)
batch = synth.make_batch(cfg, B, seed=100)
pinned = {k: torch.from_numpy(v).pin_memory() for k, v in batch.items()}
hs = torch.empty((B, cfg.n_cand, 3), dtype=torch.float32).pin_memory()
c = R.CSortBatch(B, *[pinned[k].data_ptr() for k in R._BatchHold.KEYS])
flush = torch.empty(64 * 1024 * 1024, dtype=torch.float32, device=dev)
dev_batch = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
db = R._DevBatch(dev_batch); scores = torch.empty((B, cfg.n_cand, 3), dtype=torch.float32, device=dev)
steps = 30
with torch.cuda.stream(stream):
    for _ in range(4):
        R._check(R.lib().sort_forward_async(model.h, ctypes.byref(c), hs.data_ptr()))
        model.forward_device(db, scores.data_ptr())
    model.sync()
    for rep in range(3):
        for mode in ("async", "device"):
            ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
            fe = [torch.cuda.Event(enable_timing=True) for _ in range(steps)]
            torch.cuda.synchronize(); t0 = time.perf_counter()
            ev[0].record(stream)
            for i in range(steps):
                flush.fill_(float(i)); fe[i].record(stream)
                if mode == "async":
                    R._check(R.lib().sort_forward_async(model.h, ctypes.byref(c), hs.data_ptr()))
                else:
                    model.forward_device(db, scores.data_ptr())
                ev[i + 1].record(stream)
            model.sync(); wall = (time.perf_counter() - t0) * 1e3 / steps
            per = sum(ev[i].elapsed_time(ev[i + 1]) for i in range(steps)) / steps
            fw = sum(fe[i].elapsed_time(ev[i + 1]) for i in range(steps)) / steps
            print(f"{mode}: wall {wall:.4f}  stream/step {per:.4f}  after-flush/step {fw:.4f} ms", flush=True)
