#!/usr/bin/env bash
# A/B of the pre-scaled-Q attention (attn_prescale) on the SORT-base forward, same box,
# alternating runs; parity suite first.
set -u
O=gpurun_out/r02g
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider -x > $O/parity.txt 2>&1
tail -2 $O/parity.txt
for rep in 1 2 3; do
  for v in 0 1; do
    SORT_OPTIONS=attn_prescale=$v timeout 300 python bench.py --no-cpu-baseline --steps 30 > $O/fwd_p${v}_$rep.json 2>/dev/null
    python -c "import json; d=json.loads(open('$O/fwd_p${v}_$rep.json').read().strip().splitlines()[-1]); print('prescale=$v', round(d['ms_per_step'],4), d['roofline']['stage_ms'].get('attention'), d['e2e']['ms_per_step'])"
  done
done
