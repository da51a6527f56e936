#!/usr/bin/env bash
set -u
O=gpurun_out/r02w
mkdir -p $O


timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gemm_bf16 -s 16 -c 1 -f -o $O/qkvg python bench.py --profile-launches --steps 1 --warmup 3 > $O/ncu.log 2>&1
ncu -i $O/qkvg.ncu-rep --page source --csv --print-source sass > $O/qkvg_source.csv 2>/dev/null
python tools/ncu_summary.py $O/qkvg.ncu-rep > $O/qkvg_summary.txt 2>&1
rm -f $O/qkvg.ncu-rep
head -20 $O/qkvg_summary.txt
