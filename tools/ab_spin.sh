#!/usr/bin/env bash
# Same-box A/B: softmax-warp mbarrier waits with the suspend hint (ab_w0) vs plain spin (ab_w1).
cp ab_w1.so paper_2603_03988_b200/libsort_b200.so
python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1 | sed "s/^/spin parity: /"
for rep in 1 2 3; do for k in 0 1; do
  cp ab_w$k.so paper_2603_03988_b200/libsort_b200.so
  python bench.py --no-cpu-baseline --steps 30 > gpurun_out/ab_w$k.log 2>&1
  tail -1 gpurun_out/ab_w$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('spin', $k, round(d['ms_per_step'],4), d['roofline']['stage_ms']['attention'])"
done; done
