#!/usr/bin/env bash
# Round profiling pass (run on the GPU box through gpurun, ONE GPU):
#   1. launch list of two SORT-base forward steps (gpu__time_duration, clocks uncontrolled)
#   2. ncu --set full of one whole step (24 launches) -> raw CSV (per-launch DRAM bytes,
#      pipe utilisation) brought back instead of the large report
#   3. ncu --set full --import-source of layer-1 attention (source/SASS stall analysis)
# Usage: tools/profile_round.sh TAG
set -u
TAG=${1:-r01}
OUT=gpurun_out
mkdir -p $OUT
PER_STEP=16   # kernels per SORT-base forward (tokenizer, 4 x {qkvg(s), attention, block tail},
              # gather at the pruning layer, head)
W=3
ncu --metrics gpu__time_duration.sum --clock-control none -s $((PER_STEP * W)) -c $((PER_STEP * 2)) \
    --csv --log-file $OUT/launches_$TAG.csv \
    python bench.py --profile-launches --steps 2 --warmup $W > $OUT/prof_launch_$TAG.log 2>&1
ncu --set full --clock-control none -s $((PER_STEP * W)) -c $PER_STEP -f -o /tmp/full_$TAG \
    python bench.py --profile-launches --steps 1 --warmup $W > $OUT/prof_full_$TAG.log 2>&1
ncu -i /tmp/full_$TAG.ncu-rep --page raw --csv > $OUT/full_${TAG}_raw.csv 2>>$OUT/prof_full_$TAG.log
ncu --set full --clock-control none --import-source on -k regex:k_attention -s $((4 * W)) -c 1 -f \
    -o $OUT/attn_$TAG python bench.py --profile-launches --steps 1 --warmup $W \
    > $OUT/prof_attn_$TAG.log 2>&1
ls -la $OUT
