#!/usr/bin/env bash
set -u
O=gpurun_out/r02f
mkdir -p $O
timeout 600 python bench.py --mode pretrain_train --steps 10 --warmup 3 > $O/bench_pretrain_train.json 2>$O/bench_pretrain_train.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file $O/pretrain_train_launches.csv python bench.py --mode pretrain_train --steps 1 --warmup 3 > /dev/null 2>&1
tail -1 $O/bench_pretrain_train.json | head -c 700; tail -3 $O/bench_pretrain_train.err
