#!/usr/bin/env bash
# Re-entry state check (fresh container): GPU tests, smoke, every bench mode, the reference arm.
set -u
O=gpurun_out/r02z
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_forward.json 2>$O/bench_forward.err
for m in train embed large moe pretrain pretrain_train; do
  timeout 600 python bench.py --mode $m --no-cpu-baseline > $O/bench_$m.json 2>$O/bench_$m.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1
tail -3 $O/gpu_tests.txt; tail -2 $O/smoke.txt
for f in $O/bench_*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d.get('impl','ours'), d['metric'][:40], d.get('value'), d.get('ms_per_step'), d.get('mfu'), d.get('roofline',{}).get('frac'), d.get('clocks',{}).get('sm_mhz'))" 2>&1; done
