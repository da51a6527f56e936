#!/usr/bin/env bash
set -u
O=gpurun_out/r02r
mkdir -p $O
timeout 900 ncu --set full --clock-control none -k regex:k_gemm_stream -s 40 -c 5 -f -o $O/large_gemm python bench.py --mode large --steps 1 --warmup 3 --no-cpu-baseline > $O/ncu.log 2>&1
ncu -i $O/large_gemm.ncu-rep --page raw --csv > $O/large_gemm_raw.csv 2>/dev/null
rm -f $O/large_gemm.ncu-rep
tail -2 $O/ncu.log
