#!/usr/bin/env bash
set -u
O=gpurun_out/r02y
mkdir -p $O
SORT_OPTIONS=attn_s16=1 timeout 900 python -m pytest tests/test_gpu_parity.py -q -p no:cacheprovider > $O/parity_s16.txt 2>&1
tail -3 $O/parity_s16.txt
VALS="0 1" bash tools/ab_opt.sh attn_s16 r02y
