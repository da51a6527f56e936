# Wall-clock split of one SORT-base training step (host-driven calls), for profiling only.
import sys, time
sys.path.insert(0, '.')
import numpy as np
import torch
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config
cfg = base_config()
B = 256
model = R.SortModel(cfg, synth.make_params(cfg, seed=5), max_batch=B)
batch = synth.make_batch(cfg, B, seed=100)
labels = (np.random.default_rng(7).random((B, cfg.n_cand, 3)) < 0.2).astype(np.float32)
for _ in range(3):
    model.train_step_bce(batch, labels); model.adamw_step(2e-4)
torch.cuda.synchronize()
t = {"fwd+bwd": 0.0, "adamw": 0.0, "forward only": 0.0}
for _ in range(5):
    t0 = time.perf_counter(); model.train_step_bce(batch, labels); torch.cuda.synchronize(); t1 = time.perf_counter()
    model.adamw_step(2e-4); torch.cuda.synchronize(); t2 = time.perf_counter()
    model.forward(batch); torch.cuda.synchronize(); t3 = time.perf_counter()
    t["fwd+bwd"] += (t1 - t0) / 5 * 1e3; t["adamw"] += (t2 - t1) / 5 * 1e3; t["forward only"] += (t3 - t2) / 5 * 1e3
print({k: round(v, 2) for k, v in t.items()})
