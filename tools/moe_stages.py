# Stage split of one SORT-base + MoE forward (256 requests), CUDA events on the library stream.
import sys
sys.path.insert(0, '.')
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_moe_config, base_config
which = sys.argv[1] if len(sys.argv) > 1 else "moe"
cfg = base_moe_config(batch=256) if which == "moe" else base_config(batch=256)
m = R.SortModel(cfg, synth.make_params(cfg, seed=5), max_batch=256)
if which == "dense_split":
    m.set_option("fused_tail", 0)
b = synth.make_batch(cfg, 256, seed=1)
for _ in range(3): m.forward(b)
m.enable_stage_timing(True)
acc = {}
for _ in range(3):
    m.forward(b)
    for k, v in m.stage_times().items():
        g = k.split(".")[-1]
        acc[g] = acc.get(g, 0.0) + v / 3
print(which, {k: round(v, 3) for k, v in acc.items()}, "total", round(sum(acc.values()), 3))
if which == "moe":
    print("loads", [m.moe_load(l).tolist() for l in range(cfg.layers)])
