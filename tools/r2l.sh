timeout 900 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2l_tests.log 2>&1; tail -12 gpurun_out/r2l_tests.log
for m in train large; do timeout 300 python bench.py --mode $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2l_$m.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2l_$m.log || tail -5 gpurun_out/r2l_$m.log; done
