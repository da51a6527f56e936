#!/usr/bin/env bash
# Attention exp2 offload sweep (run on the GPU box): rebuild with each ratio, bench once.
for k in 4 3 2; do
  SORT_NVCC_EXTRA="-DSORT_ATTN_POLY_EVERY=$k" python -c "from paper_2603_03988_b200 import build as B; B.build(force=True)" > /dev/null 2>&1
  python bench.py --no-cpu-baseline --steps 20 > gpurun_out/poly_$k.log 2>&1
  tail -1 gpurun_out/poly_$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('every', $k, round(d['ms_per_step'],4), d['roofline']['stage_ms']['attention'])"
done
