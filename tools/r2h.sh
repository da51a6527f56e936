set -x
timeout 900 python -m pytest tests/test_gpu_gemm.py tests/test_gpu_train.py tests/test_gpu_parity.py tests/test_gpu_exchange.py -q -x --timeout 300 > gpurun_out/r2h_tests.log 2>&1; tail -25 gpurun_out/r2h_tests.log
timeout 200 python bench.py --mode train --steps 5 --warmup 3 > gpurun_out/r2h_train.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2h_train.log
SORT_OPTIONS=attn_bwd_tc=0 timeout 200 python bench.py --mode train --steps 5 --warmup 3 > gpurun_out/r2h_train_mma.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2h_train_mma.log
timeout 200 python bench.py --mode large --steps 10 --warmup 3 > gpurun_out/r2h_large.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2h_large.log
