#!/usr/bin/env bash
# Round-2 measurement sweep on one B200: every bench mode, the reference arm, launch lists, and
# the ncu --set full step capture + layer-1 attention source page (tools/profile_round.sh).
set -u
O=gpurun_out/${SWEEP:-r02s}
mkdir -p $O
timeout 600 python bench.py > $O/bench_forward.json 2>$O/bench_forward.err
for m in train pretrain_train embed large moe pretrain; do
  timeout 600 python bench.py --mode $m --no-cpu-baseline > $O/bench_$m.json 2>$O/bench_$m.err
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 3 > $O/bench_reference.json 2>&1
for m in train large moe pretrain_train; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/${m}_launches.csv python bench.py --mode $m --steps 1 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
bash tools/profile_round.sh ${PTAG:-r02} > $O/profile_round.log 2>&1
for f in $O/bench_*.json; do tail -1 $f | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d.get('impl','ours'), d['metric'][:45], round(d.get('value') or 0,1), round(d.get('ms_per_step') or 0,4), d.get('clocks',{}).get('sm_mhz'))" 2>&1; done
