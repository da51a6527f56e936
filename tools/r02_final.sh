#!/usr/bin/env bash
# final round-2 validation: GPU tests + smoke, then the full sweep (tools/r02_sweep.sh)
set -u
mkdir -p gpurun_out/r02f2
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/r02f2/gpu_tests.txt 2>&1
tail -2 gpurun_out/r02f2/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r02f2/smoke.txt 2>&1
tail -1 gpurun_out/r02f2/smoke.txt
SWEEP=r02f2 PTAG=r02b bash tools/r02_sweep.sh
