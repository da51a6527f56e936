import time, sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
import bench
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config
from paper_2603_03988_b200.sharding import ShardedItemTable
cfg = base_config(batch=256)
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
rows_per_rank = 100_000_000
g = torch.Generator(device=dev); g.manual_seed(1000)
shard = (torch.randn((rows_per_rank, cfg.item_dim), generator=g, device=dev) * 0.1).to(torch.bfloat16)
small = base_config(batch=256, n_items=1024)
model = R.SortModel(small, synth.make_params(small, seed=5), device=0, max_batch=256)
stream = torch.cuda.Stream(device=dev); model.set_stream(stream.cuda_stream)
rng = np.random.default_rng(100)
batch = synth.make_batch(small, 256, seed=100)
batch["hist_item"] = rng.integers(0, rows_per_rank, size=batch["hist_item"].shape, dtype=np.int64).astype(np.int32)
batch["cand_item"] = np.stack([rng.choice(rows_per_rank, size=cfg.n_cand, replace=False) for _ in range(256)]).astype(np.int32)
tb = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
ex = R.Exchange.nccl(0, 1, 0)
table = ShardedItemTable(shard, rows_per_rank, 0, 1, ex, stream_ptr=stream.cuda_stream)
scores = torch.empty((256, 64, 3), dtype=torch.float32, device=dev)
T = {"lookup": 0.0, "set": 0.0, "devbatch": 0.0, "fwd": 0.0, "sync": 0.0}
def step(tm):
    with torch.cuda.stream(stream):
        t0 = time.perf_counter(); rows, mapped = table.lookup(tb); t1 = time.perf_counter()
        model.set_item_table(rows.data_ptr(), rows.shape[0]); t2 = time.perf_counter()
        db = R._DevBatch(mapped); t3 = time.perf_counter()
        model.forward_device(db, scores.data_ptr()); t4 = time.perf_counter()
        model.sync(); t5 = time.perf_counter()
    if tm:
        for k, a, b in (("lookup", t0, t1), ("set", t1, t2), ("devbatch", t2, t3), ("fwd", t3, t4), ("sync", t4, t5)):
            T[k] += (b - a) * 1e3
for _ in range(5): step(False)
n = 20
t0 = time.perf_counter()
for _ in range(n): step(True)
print("total ms/step", (time.perf_counter() - t0) * 1e3 / n, {k: round(v / n, 3) for k, v in T.items()})
