import time, sys, os, numpy as np, torch
sys.path.insert(0, os.getcwd())
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config
from paper_2603_03988_b200.sharding import ShardedItemTable
dev = torch.device("cuda", 0); torch.cuda.set_device(0)
rows_per_rank = 100_000_000
shard = (torch.randn((rows_per_rank, 32), device=dev) * 0.1).to(torch.bfloat16)
small = base_config(batch=256, n_items=1024)
model = R.SortModel(small, synth.make_params(small, seed=5), device=0, max_batch=256)
stream = torch.cuda.Stream(device=dev); model.set_stream(stream.cuda_stream)
rng = np.random.default_rng(100)
batch = synth.make_batch(small, 256, seed=100)
batch["hist_item"] = rng.integers(0, rows_per_rank, size=batch["hist_item"].shape).astype(np.int32)
batch["cand_item"] = rng.integers(0, rows_per_rank, size=batch["cand_item"].shape).astype(np.int32)
tb = {k: torch.from_numpy(v).to(dev) for k, v in batch.items()}
ex = R.Exchange.nccl(0, 1, 0)
table = ShardedItemTable(shard, rows_per_rank, 0, 1, ex, stream_ptr=stream.cuda_stream)
scores = torch.empty((256, 64, 3), dtype=torch.float32, device=dev)
def run(name, fwd, endsync):
    T = [0.0, 0.0]
    def step(tm):
        with torch.cuda.stream(stream):
            t0 = time.perf_counter(); rows, mapped = table.lookup(tb); t1 = time.perf_counter()
            if fwd:
                model.set_item_table(rows.data_ptr(), rows.shape[0])
                model.forward_device(R._DevBatch(mapped), scores.data_ptr())
            if endsync == "model": model.sync()
            elif endsync == "torch": torch.cuda.synchronize()
            elif endsync == "stream": stream.synchronize()
            t2 = time.perf_counter()
        if tm: T[0] += t1 - t0; T[1] += t2 - t1
    for _ in range(4): step(False)
    for _ in range(10): step(True)
    print(name, "lookup ms", round(T[0] * 100, 3), "rest ms", round(T[1] * 100, 3), flush=True)
run("fwd+model.sync", True, "model")
run("fwd+torch.sync", True, "torch")
run("fwd+stream.sync", True, "stream")
run("nofwd+model.sync", False, "model")
