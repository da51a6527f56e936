#!/usr/bin/env bash
# late round-2 validation: GPU tests + smoke, sanitizers over the late changes, the full sweep
set -u
O=gpurun_out/${FTAG:-r02f3}
mkdir -p $O
timeout 1800 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/gpu_tests.txt 2>&1
tail -2 $O/gpu_tests.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
tail -1 $O/smoke.txt
bash tools/sanitize_r02b.sh
SWEEP=${FTAG:-r02f3} PTAG=${PTAG:-r02c} bash tools/r02_sweep.sh
