#!/usr/bin/env bash
set -u
O=gpurun_out/r02v
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_moe.py -q -p no:cacheprovider > $O/tests.txt 2>&1
tail -3 $O/tests.txt
for rep in 1 2 3; do
  for v in 0 1; do
    SORT_OPTIONS=moe_route_lane=$v timeout 300 python bench.py --mode moe --no-cpu-baseline --steps 30 > $O/moe_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/moe_${v}_$rep.json').read().strip().splitlines()[-1]); print('lane=$v', round(d['ms_per_step'],4))"
  done
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 200 --csv --log-file $O/moe_launches.csv python bench.py --mode moe --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
