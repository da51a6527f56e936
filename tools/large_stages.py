# Stage split of one SORT-large forward (generic path), CUDA events on the library stream.
import sys
sys.path.insert(0, '.')
import numpy as np
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import large_config
cfg = large_config(batch=8)
m = R.SortModel(cfg, synth.make_params(cfg, seed=5), max_batch=8)
b = synth.make_batch(cfg, 8, seed=1)
for _ in range(3): m.forward(b)
m.enable_stage_timing(True)
acc = {}
for _ in range(3):
    m.forward(b)
    for k, v in m.stage_times().items():
        g = k.split(".")[-1]
        acc[g] = acc.get(g, 0.0) + v / 3
print({k: round(v, 3) for k, v in acc.items()}, "total", round(sum(acc.values()), 3))
