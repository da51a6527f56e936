#!/usr/bin/env bash
set -u
O=gpurun_out/r02ac
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pretrain.py -q -p no:cacheprovider > $O/tests.txt 2>&1
tail -3 $O/tests.txt
for rep in 1 2 3; do
  for v in 0 1; do
    SORT_OPTIONS=pre_proj_tc=$v timeout 300 python bench.py --mode pretrain --no-cpu-baseline --steps 30 > $O/pt_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/pt_${v}_$rep.json').read().strip().splitlines()[-1]); print('pre_proj_tc=$v', round(d['ms_per_step'],4))"
  done
done
