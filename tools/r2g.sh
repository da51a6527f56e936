set -x
timeout 300 python - <<'PY' 2>&1 | tail -40
import time, numpy as np, torch
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config
cfg = base_config(batch=256); P = synth.make_params(cfg, seed=5)
gm = R.SortModel(cfg, P, max_batch=256); b = synth.make_batch(cfg, 256, seed=1)
for g in (0, 1):
    gm.set_option("graphs", g)
    for i in range(4):
        t = time.time(); p = gm.forward(b); print("graphs", g, "forward", i, round(time.time() - t, 4), float(p.mean()), flush=True)
dev = torch.device("cuda", 0)
st = torch.cuda.Stream(device=dev); gm.set_stream(st.cuda_stream)
db = R._DevBatch({k: torch.from_numpy(v).to(dev) for k, v in b.items()})
sc = torch.empty((256, 64, 3), device=dev)
for i in range(6):
    t = time.time(); gm.forward_device(db, sc.data_ptr()); gm.sync(); print("device", i, round(time.time() - t, 4), flush=True)
gm.enable_stage_timing(True)
gm.forward_device(db, sc.data_ptr()); gm.sync(); print(gm.stage_times())
PY
