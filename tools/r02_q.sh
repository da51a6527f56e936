#!/usr/bin/env bash
set -u
O=gpurun_out/r02q
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_frozen.py tests/test_gpu_pretrain.py tests/test_cpp_reference_api.py -q -p no:cacheprovider > $O/tests.txt 2>&1
tail -3 $O/tests.txt
timeout 600 python bench.py --mode train --no-cpu-baseline > $O/bench_train.json 2>$O/bench_train.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/train_launches.csv python bench.py --mode train --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -1 $O/bench_train.json | head -c 300; echo
