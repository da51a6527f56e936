#!/usr/bin/env bash
# exp2 polynomial offload ratio with the pre-scaled attention: prebuilt variants swapped in
set -u
O=gpurun_out/r02h
mkdir -p $O
L=paper_2603_03988_b200/libsort_b200.so
cp $L /tmp/orig.so
for rep in 1 2; do
  for pe in 2 3 4; do
    cp tools/ablib/lib_pe$pe.so $L; touch $L
    timeout 300 python bench.py --no-cpu-baseline --steps 30 > $O/fwd_pe${pe}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/fwd_pe${pe}_$rep.json').read().strip().splitlines()[-1]); print('pe=$pe', round(d['ms_per_step'],4), d['roofline']['stage_ms'].get('attention'))"
  done
done
cp /tmp/orig.so $L
