#!/usr/bin/env bash
# compute-sanitizer over the late round-2 changes: the tensor-core ranking head (3D candidate
# view and the gathered path, in-epilogue row finish), the tokenizer's two-stage gather, the
# coprime attention grids (tiny forward + pruned schedules); memcheck + racecheck.
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
SEL="tensor_core_head and (tiny or n20) or tiny_matches_golden or pruned_schedules or tokenizer_parity"
timeout 1500 $CS --tool memcheck --leak-check no --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
  tests/test_gpu_parity.py -k "$SEL" > gpurun_out/sanitize_r02b_memcheck.txt 2>&1
echo "memcheck rc=$?" | tee -a gpurun_out/sanitize_r02b_memcheck.txt
timeout 1500 $CS --tool racecheck --error-exitcode 9 python -m pytest -q -x -p no:cacheprovider \
  tests/test_gpu_parity.py -k "tensor_core_head and tiny or tiny_matches_golden" > gpurun_out/sanitize_r02b_racecheck.txt 2>&1
echo "racecheck rc=$?" | tee -a gpurun_out/sanitize_r02b_racecheck.txt
for f in gpurun_out/sanitize_r02b_*.txt; do echo "== $f"; grep -E "ERROR SUMMARY|passed|failed|rc=" $f | tail -4; done
