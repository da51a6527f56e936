#!/usr/bin/env bash
set -u
O=gpurun_out/r02c
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_cpp_reference_api.py -m gpu -q -p no:cacheprovider > $O/tests.txt 2>&1
timeout 600 python bench.py --mode train --no-cpu-baseline > $O/bench_train.json 2>$O/bench_train.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/train_launches.csv python bench.py --mode train --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attn_bwd_tc -s 4 -c 2 -f -o $O/attn_bwd python bench.py --mode train --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu_bwd.log 2>&1
ncu -i $O/attn_bwd.ncu-rep --page raw --csv > $O/attn_bwd_raw.csv 2>/dev/null
ncu -i $O/attn_bwd.ncu-rep --page source --csv --print-source sass > $O/attn_bwd_source.csv 2>/dev/null
rm -f $O/attn_bwd.ncu-rep
tail -3 $O/tests.txt
tail -1 $O/bench_train.json | head -c 400
