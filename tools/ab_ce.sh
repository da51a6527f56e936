#!/usr/bin/env bash
set -u
O=gpurun_out/r02z
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pretrain.py -q -p no:cacheprovider > $O/tests.txt 2>&1
tail -3 $O/tests.txt
for rep in 1 2 3; do
  for v in 0 1; do
    SORT_OPTIONS=ce_tc=$v timeout 300 python bench.py --mode pretrain --no-cpu-baseline --steps 30 > $O/pt_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/pt_${v}_$rep.json').read().strip().splitlines()[-1]); print('ce_tc=$v', round(d['ms_per_step'],4))"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 100 --csv --log-file $O/pt_launches.csv python bench.py --mode pretrain --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
