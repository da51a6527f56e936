set -x
timeout 300 python tools/diag_gemm.py 2>&1 | tail -50
timeout 300 python bench.py --mode train --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/r2j_train.log 2>&1; tail -5 gpurun_out/r2j_train.log
timeout 900 python -m pytest tests -m gpu -q --timeout 400 > gpurun_out/r2j_tests.log 2>&1; tail -25 gpurun_out/r2j_tests.log
