#!/usr/bin/env bash
# Same-box A/B: MoE route+scatter re-reading rows from global (ab_s0) vs staged in shared memory (ab_s1).
cp ab_s1.so paper_2603_03988_b200/libsort_b200.so
python -m pytest tests/test_gpu_moe.py -x -q 2>&1 | tail -1 | sed "s/^/s1 moe tests: /"
for rep in 1 2 3; do for k in 0 1; do
  cp ab_s$k.so paper_2603_03988_b200/libsort_b200.so
  python bench.py --mode moe --no-cpu-baseline --steps 30 > gpurun_out/ab_s$k.log 2>&1
  tail -1 gpurun_out/ab_s$k.log | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('stage', $k, round(d['ms_per_step'],4))"
done; done
for k in 0 1; do
  cp ab_s$k.so paper_2603_03988_b200/libsort_b200.so
  ncu --metrics gpu__time_duration.sum --clock-control none -k regex:route_scatter -c 2 --csv python bench.py --mode moe --no-cpu-baseline --steps 1 --warmup 1 2>/dev/null | grep route_scatter | awk -F'","' -v k=$k '{print "s" k " route ns:", $NF}'
done
