#!/usr/bin/env bash
# alternate prebuilt library variants (tools/ablib/lib_<name>.so) on the SORT-base training step
set -u
O=gpurun_out/${ABOUT:-r02tr}
mkdir -p $O
L=paper_2603_03988_b200/libsort_b200.so
cp $L /tmp/orig.so
for rep in 1 2 3; do
  for v in "$@"; do
    cp tools/ablib/lib_$v.so $L; touch $L
    timeout 600 python bench.py --mode train --no-cpu-baseline --steps 10 > $O/train_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/train_${v}_$rep.json').read().strip().splitlines()[-1]); print('$v', round(d['ms_per_step'],3))"
  done
done
cp /tmp/orig.so $L
