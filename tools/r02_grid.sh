#!/usr/bin/env bash
# coprime persistent grids: GPU tests, forward x3, train x1, attention launch times per layer
set -u
O=gpurun_out/${TAG:-r02grid}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -2 $O/gpu_tests.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --steps 40 > $O/fwd_$rep.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/fwd_$rep.json').read().strip().splitlines()[-1]); s=d['roofline']['stage_ms']; print(round(d['ms_per_step'],4), d['e2e']['ms_per_step'], s, round(d.get('mfu'),4))"
done
timeout 600 python bench.py --mode train --no-cpu-baseline --steps 10 > $O/train.json 2>/dev/null
python -c "import json; d=json.loads(open('$O/train.json').read().strip().splitlines()[-1]); print('train', round(d['ms_per_step'],3))"
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_attention -c 8 --csv --log-file $O/attn_launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1
grep gpu__time $O/attn_launches.csv | awk -F'","' '{print $NF}' | tr '\n' ' '; echo
