#!/usr/bin/env bash
# compute-sanitizer pass over the small GPU cases (run on the GPU box): memcheck on a tiny
# forward / tokenizer / block attention / train step / MoE / pretrain selection, then
# racecheck / synccheck / initcheck on the smoke forward and racecheck on train/MoE/pretrain. Summaries go to gpurun_out/sanitize_*.txt.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL='(tiny and not subtile and not golden) or block_attention or gather_rows or oov or time_buckets or zero_params or two_handles or forward_async or small or train_step_tiny'
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
  tests/test_gpu_parity.py tests/test_gpu_train.py tests/test_gpu_moe.py tests/test_gpu_pretrain.py \
  -k "$SEL" > gpurun_out/sanitize_memcheck.txt 2>&1
echo "memcheck rc=$?" | tee -a gpurun_out/sanitize_memcheck.txt
for tool in racecheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --error-exitcode 9 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/sanitize_$tool.txt 2>&1
  echo "$tool rc=$?" | tee -a gpurun_out/sanitize_$tool.txt
done
timeout 1200 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
  tests/test_gpu_train.py tests/test_gpu_moe.py tests/test_gpu_pretrain.py \
  -k "train_step_tiny or tiny_k2 or small" > gpurun_out/sanitize_racecheck_tests.txt 2>&1
echo "racecheck tests rc=$?" | tee -a gpurun_out/sanitize_racecheck_tests.txt
for f in gpurun_out/sanitize_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|rc=" $f | tail -4; done
