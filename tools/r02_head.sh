#!/usr/bin/env bash
# tensor-core head: GPU tests, then A/B of head_tc on the SORT-base forward (head stage printed)
set -u
O=gpurun_out/r02h
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
for rep in 1 2; do
  for v in 0 1; do
    SORT_OPTIONS=head_tc=$v timeout 300 python bench.py --no-cpu-baseline --steps 40 > $O/fwd_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/fwd_${v}_$rep.json').read().strip().splitlines()[-1]); s=d['roofline']['stage_ms']; print('head_tc=$v', round(d['ms_per_step'],4), d['e2e']['ms_per_step'], s.get('head'), d.get('mfu'))"
  done
done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:'k_gather_cand|k_gemm_stream|k_head' -c 12 --csv --log-file $O/head_launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1
grep -c gpu__time $O/head_launches.csv
