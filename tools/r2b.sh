set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2b_parity.log 2>&1; tail -3 gpurun_out/r2b_parity.log
timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_fx.log 2>&1; tail -c 1500 gpurun_out/r2b_bench_fx.log
SORT_OPTIONS=attn_fx=0 timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2b_bench_old.log 2>&1; tail -c 600 gpurun_out/r2b_bench_old.log
