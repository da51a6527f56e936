#!/usr/bin/env bash
# Same-box A/B of k_moe_route_scatter8 variants (ab_m0 = committed, ab_m1 = candidate).
cp ab_m1.so paper_2603_03988_b200/libsort_b200.so
python -m pytest tests/test_gpu_moe.py -x -q 2>&1 | tail -1 | sed "s/^/m1 moe tests: /"
for rep in 1 2; do for k in 0 1; do
  cp ab_m$k.so paper_2603_03988_b200/libsort_b200.so
  python bench.py --mode moe --no-cpu-baseline --steps 30 > gpurun_out/ab_m$k.log 2>&1
  tail -1 gpurun_out/ab_m$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('moe', $k, round(d['ms_per_step'],4))"
done; done
for k in 0 1; do
  cp ab_m$k.so paper_2603_03988_b200/libsort_b200.so
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:route_scatter -c 4 --csv python bench.py --mode moe --no-cpu-baseline --steps 1 --warmup 1 2>/dev/null | grep '"k_moe\|route_scatter' | awk -F'","' -v k=$k '{print "m" k " route ns:", $NF}' | head -4
done
