#!/usr/bin/env bash
# tokenizer rework: GPU tests, forward bench x3 (tokenizer stage printed), ncu launch times + one
# --set full capture of k_tokenize with source counters
set -u
O=gpurun_out/${TAG:-r02tok}
mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -3 $O/gpu_tests.txt
for rep in 1 2 3; do
  timeout 300 python bench.py --no-cpu-baseline --steps 40 > $O/fwd_$rep.json 2>/dev/null
  python -c "import json; d=json.loads(open('$O/fwd_$rep.json').read().strip().splitlines()[-1]); s=d['roofline']['stage_ms']; print(round(d['ms_per_step'],4), d['e2e']['ms_per_step'], s, round(d.get('mfu'),4))"
done
timeout 300 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_tokenize -c 4 --csv --log-file $O/tok_launches.csv python bench.py --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1
grep k_tokenize $O/tok_launches.csv | head -12
timeout 300 ncu --set full --import-source on --clock-control none -k regex:k_tokenize -s 2 -c 1 -f -o $O/tok python bench.py --profile-launches --steps 1 --warmup 2 > $O/tok_ncu.log 2>&1
ncu -i $O/tok.ncu-rep --page source --csv --print-source sass > $O/tok_source.csv 2>/dev/null
ncu -i $O/tok.ncu-rep --page details > $O/tok_details.txt 2>/dev/null
grep -E "Duration|DRAM Throughput|Executed Ipc|No Eligible|Registers Per|Achieved Active Warps" $O/tok_details.txt | head -12
