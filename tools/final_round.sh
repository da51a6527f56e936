mkdir -p gpurun_out/final
python -m pytest tests -m gpu -x -q 2>&1 | tail -2 > gpurun_out/final/gpu_tests.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.txt 2>&1
python bench.py > gpurun_out/final/bench_forward.json 2>gpurun_out/final/bench_forward.err
for m in train embed large moe pretrain; do python bench.py --mode $m --no-cpu-baseline > gpurun_out/final/bench_$m.json 2>gpurun_out/final/bench_$m.err; done
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/final/bench_reference.json 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/moe_launches.csv python bench.py --mode moe --no-cpu-baseline --steps 1 --warmup 1 > /dev/null 2>&1
cat gpurun_out/final/gpu_tests.txt gpurun_out/final/smoke.txt
for f in gpurun_out/final/bench_*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d.get('impl','ours'), d['metric'][:50], round(d['value'],1), round(d['ms_per_step'],3), d.get('clocks',{}).get('sm_mhz'))"; done
