timeout 300 python tools/diag_gemm.py 2>&1 | grep tf32
timeout 900 python -m pytest tests/test_gpu_train.py tests/test_gpu_gemm.py tests/test_gpu_parity.py -q --timeout 400 > gpurun_out/r2k_tests.log 2>&1; tail -12 gpurun_out/r2k_tests.log
