#!/usr/bin/env bash
# A/B of one library option on the SORT-base forward (same box, alternating): ab_opt.sh NAME OUT
set -u
N=$1; O=gpurun_out/$2
mkdir -p $O
for rep in 1 2 3; do
  for v in ${VALS:-0 1}; do
    SORT_OPTIONS=$N=$v timeout 300 python bench.py --no-cpu-baseline --steps 40 > $O/fwd_${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/fwd_${v}_$rep.json').read().strip().splitlines()[-1]); print('$N=$v', round(d['ms_per_step'],4), d['e2e']['ms_per_step'], d['roofline']['stage_ms'].get('tokenizer'))"
  done
done
