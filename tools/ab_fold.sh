#!/usr/bin/env bash
# Same-box A/B of the attention fold position (ab_f{0,1,2}.so built with -DSORT_ATTN_FOLD_AT=k).
for k in 0 2; do
  cp ab_f$k.so paper_2603_03988_b200/libsort_b200.so
  python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 | sed "s/^/fold $k parity: /"
done
for rep in 1 2; do for k in 0 1 2; do
  cp ab_f$k.so paper_2603_03988_b200/libsort_b200.so
  python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_f$k.log 2>&1
  tail -1 gpurun_out/ab_f$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('fold', $k, round(d['ms_per_step'],4), d['roofline']['stage_ms']['attention'])"
done; done
