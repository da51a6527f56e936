#!/usr/bin/env bash
# Round-2 final check after the training-backward write elisions: every GPU test, smoke,
# forward + training bench, training-step launch list.
set -u
O=gpurun_out/r02u
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 600 python bench.py > $O/bench_forward.json 2>$O/bench_forward.err
timeout 600 python bench.py --mode train --no-cpu-baseline > $O/bench_train.json 2>$O/bench_train.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/train_launches.csv python bench.py --mode train --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -2 $O/gpu_tests.txt; tail -1 $O/smoke.txt
for f in $O/bench_*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['metric'][:40], d.get('value'), d.get('ms_per_step'), d.get('mfu'), d.get('clocks',{}).get('sm_mhz'))"; done
