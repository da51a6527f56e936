import sys; sys.path.insert(0, '.')
import numpy as np
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_moe_config
cfg = base_moe_config(batch=2)
P = synth.make_params(cfg, seed=51)
gm = R.SortModel(cfg, P, max_batch=2)
x = np.random.default_rng(0).normal(size=(2000, 256)).astype(np.float32)
y1 = gm.moe_forward(1, x)
gm.set_option("moe_fused", 0)
y0 = gm.moe_forward(1, x)
d = np.abs(y1 - y0)
rows = np.where(d.max(1) > 0)[0]
print("rows differing", len(rows), "of", len(x), "max", d.max())
if len(rows):
    print("first rows", rows[:20])
    r = rows[0]; c = np.where(d[r] > 0)[0]; print("cols", c[:20], len(c))
    print(y1[r, c[:5]], y0[r, c[:5]])
sel, w = gm.moe_routing(1, 2000)
print("sel of differing rows", sel[rows[:10], 0] if len(rows) else None)
