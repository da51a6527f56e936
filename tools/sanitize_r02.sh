#!/usr/bin/env bash
# compute-sanitizer over the round-2 additions: the operator-level entries (facade caller),
# frozen parameters / item-table training, the pre-training backward (small config), the
# exchange; memcheck + racecheck. Summaries in gpurun_out/sanitize_r02_*.txt.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
  tests/test_cpp_reference_api.py tests/test_gpu_frozen.py tests/test_gpu_exchange.py \
  tests/test_gpu_pretrain.py -k "reference_caller or frozen or item_table or transfer or backward_vs_oracle or host_transport or nccl" \
  > gpurun_out/sanitize_r02_memcheck.txt 2>&1
echo "memcheck rc=$?" | tee -a gpurun_out/sanitize_r02_memcheck.txt
timeout 1500 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
  tests/test_gpu_frozen.py tests/test_gpu_pretrain.py -k "dense_parameter or backward_vs_oracle" \
  > gpurun_out/sanitize_r02_racecheck.txt 2>&1
echo "racecheck rc=$?" | tee -a gpurun_out/sanitize_r02_racecheck.txt
for f in gpurun_out/sanitize_r02_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|rc=" $f | tail -4; done
