set -x
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_gemm.py tests/test_gpu_exchange.py -q -x --timeout 240 > gpurun_out/r2f_tests.log 2>&1; tail -15 gpurun_out/r2f_tests.log
for o in "" "attn_fx=0"; do SORT_OPTIONS=$o timeout 200 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2f_bench_$o.log 2>&1; python -c "
import json,sys; l=[json.loads(x) for x in open('gpurun_out/r2f_bench_$o.log') if x.startswith('{')][0]; print('$o', l['ms_per_step'], l['roofline']['stage_ms'])"; done
timeout 600 python -m pytest tests/test_gpu_train.py -q -x --timeout 240 > gpurun_out/r2f_train.log 2>&1; tail -15 gpurun_out/r2f_train.log
for o in "" "train_cublas=1"; do SORT_OPTIONS=$o timeout 200 python bench.py --mode train --steps 5 --warmup 3 > gpurun_out/r2f_train_$o.log 2>&1; grep -o '"ms_per_step": [0-9.]*' gpurun_out/r2f_train_$o.log; done
