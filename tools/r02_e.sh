#!/usr/bin/env bash
set -u
O=gpurun_out/r02e
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_pretrain.py tests/test_gpu_frozen.py tests/test_gpu_train.py -q -p no:cacheprovider > $O/tests.txt 2>&1
tail -30 $O/tests.txt
