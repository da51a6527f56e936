# round-2 re-entry validation: full GPU suite, smoke, bench modes
set -x
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 400 > gpurun_out/r2i_tests.log 2>&1; tail -25 gpurun_out/r2i_tests.log
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -3
timeout 300 python bench.py --steps 10 --warmup 3 > gpurun_out/r2i_bench.log 2>&1; tail -c 3000 gpurun_out/r2i_bench.log
for m in train large embed moe pretrain; do timeout 300 python bench.py --mode $m --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2i_$m.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2i_$m.log || tail -20 gpurun_out/r2i_$m.log; done
