#!/usr/bin/env bash
set -u
O=gpurun_out/r02ab
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_attention2 -s 13 -c 1 -f -o $O/a2 python bench.py --profile-launches --steps 1 --warmup 3 > $O/ncu.log 2>&1
ncu -i $O/a2.ncu-rep --page source --csv --print-source sass > $O/a2_source.csv 2>/dev/null
python tools/ncu_summary.py $O/a2.ncu-rep > $O/a2_summary.txt 2>&1
rm -f $O/a2.ncu-rep
head -20 $O/a2_summary.txt
