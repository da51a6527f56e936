#!/usr/bin/env bash
set -u
O=gpurun_out/r02d
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/tests.txt 2>&1
timeout 600 python bench.py --mode train --no-cpu-baseline > $O/bench_train.json 2>$O/bench_train.err
tail -15 $O/tests.txt
tail -1 $O/bench_train.json | head -c 300
