set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x > gpurun_out/r2d_parity.log 2>&1; tail -15 gpurun_out/r2d_parity.log
for o in "" "attn_fx=0"; do SORT_OPTIONS=$o timeout 300 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r2d_bench_$o.log 2>&1; python -c "
import json,sys; l=[json.loads(x) for x in open('gpurun_out/r2d_bench_$o.log') if x.startswith('{')][0]; print('$o', l['ms_per_step'], l['roofline']['stage_ms'])"; done
for o in "" "stream_gemm=0"; do SORT_OPTIONS=$o timeout 300 python bench.py --mode large --steps 10 --warmup 3 > gpurun_out/r2d_large_$o.log 2>&1; tail -c 400 gpurun_out/r2d_large_$o.log; done
