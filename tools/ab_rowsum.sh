#!/usr/bin/env bash
# Same-box A/B of tensor-core row sums in the attention softmax (ab_r1: -DSORT_ATTN_MMA_ROWSUM=1).
cp ab_r1.so paper_2603_03988_b200/libsort_b200.so
python -m pytest tests -m gpu -x -q 2>&1 | tail -3 | sed "s/^/rowsum parity: /"
for rep in 1 2 3; do for k in 0 1; do
  cp ab_r$k.so paper_2603_03988_b200/libsort_b200.so
  python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_r$k.log 2>&1
  tail -1 gpurun_out/ab_r$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('rowsum', $k, round(d['ms_per_step'],4), d['roofline']['stage_ms']['attention'])"
done; done
