#!/usr/bin/env bash
# alternate prebuilt library variants (tools/ablib/lib_<name>.so) on the SORT-base forward
set -u
O=gpurun_out/${ABOUT:-r02i}
mkdir -p $O
L=paper_2603_03988_b200/libsort_b200.so
cp $L /tmp/orig.so
for rep in 1 2 3; do
  for v in "$@"; do
    cp tools/ablib/lib_$v.so $L; touch $L
    timeout 300 python bench.py --no-cpu-baseline --steps 30 > $O/fwd_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/fwd_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],4), d['roofline']['stage_ms'])"
  done
done
cp /tmp/orig.so $L
