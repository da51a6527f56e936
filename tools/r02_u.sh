#!/usr/bin/env bash
set -u
O=gpurun_out/r02u
mkdir -p $O
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_tokenize -s 3 -c 1 -f -o $O/tok python bench.py --profile-launches --steps 1 --warmup 3 > $O/ncu.log 2>&1
ncu -i $O/tok.ncu-rep --page raw --csv > $O/tok_raw.csv 2>/dev/null
ncu -i $O/tok.ncu-rep --page source --csv --print-source sass > $O/tok_source.csv 2>/dev/null
python tools/ncu_summary.py $O/tok.ncu-rep > $O/tok_summary.txt 2>&1
rm -f $O/tok.ncu-rep
head -30 $O/tok_summary.txt
