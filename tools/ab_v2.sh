#!/usr/bin/env bash
set -u
O=gpurun_out/r02aa
mkdir -p $O
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -p no:cacheprovider > $O/parity.txt 2>&1
tail -3 $O/parity.txt
VALS="0 1" timeout 900 bash tools/ab_opt.sh attn_v2 r02aa
