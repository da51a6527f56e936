#!/usr/bin/env bash
set -u
O=gpurun_out/r02j
mkdir -p $O
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/embed_launches.csv python bench.py --mode embed --steps 2 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 300 python - > $O/embed_timing.txt 2>&1 <<'PY'
import time, numpy as np, torch, sys
sys.argv=['bench.py']
from paper_2603_03988_b200 import runtime as R, synth
from paper_2603_03988_b200.config import base_config
from paper_2603_03988_b200.sharding import ShardedItemTable
dev=torch.device('cuda',0)
rows=100_000_000
shard=(torch.randn((rows,32),device=dev)*0.1).to(torch.bfloat16)
small=base_config(batch=256,n_items=1024)
m=R.SortModel(small, synth.make_params(small, seed=5), device=0, max_batch=256)
st=torch.cuda.Stream(device=dev); m.set_stream(st.cuda_stream)
b=synth.make_batch(small,256,seed=1); rng=np.random.default_rng(1)
b['hist_item']=rng.integers(0,rows,size=b['hist_item'].shape).astype(np.int32)
b['cand_item']=rng.integers(0,rows,size=b['cand_item'].shape).astype(np.int32)
tb={k:torch.from_numpy(v).to(dev) for k,v in b.items()}
x=R.Exchange.nccl(0,1,0)
t=ShardedItemTable(shard,rows,0,1,x,stream_ptr=st.cuda_stream)
sc=torch.empty((256,64,3),device=dev)
def lk():
    with torch.cuda.stream(st):
        r,mp=t.lookup(tb); torch.cuda.synchronize()
        return r,mp
for _ in range(3): r,mp=lk()
t0=time.perf_counter()
for _ in range(10): r,mp=lk()
print('lookup ms', (time.perf_counter()-t0)*100)
db=R._DevBatch(mp)
def fw():
    with torch.cuda.stream(st):
        m.set_item_table(r.data_ptr(), r.shape[0]); m.forward_device(db, sc.data_ptr()); m.sync()
for _ in range(3): fw()
t0=time.perf_counter()
for _ in range(10): fw()
print('forward (eager, ext table) ms', (time.perf_counter()-t0)*100)
t0=time.perf_counter()
for _ in range(10): R._DevBatch(mp)
print('DevBatch ms', (time.perf_counter()-t0)*100)
PY
cat $O/embed_timing.txt
