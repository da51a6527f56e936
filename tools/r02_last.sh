#!/usr/bin/env bash
# last state check: GPU tests, smoke, forward bench x2 (default flags), tokenizer ncu launch times
set -u
O=gpurun_out/r02last
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -2 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -1 $O/smoke.txt
for rep in 1 2; do
  timeout 600 python bench.py > $O/bench_forward_$rep.json 2>$O/bench_forward_$rep.err
  tail -1 $O/bench_forward_$rep.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(round(d['ms_per_step'],4), round(d['mfu'],4), round(d['e2e']['ms_per_step'],4), d['clocks'])"
done
