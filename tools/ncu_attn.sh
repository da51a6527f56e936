# ncu capture of the first attention launch (layer 1) of one SORT-base forward
# usage: bash tools/ncu_attn.sh <tag> [kernel-regex]
tag=$1; re=${2:-k_attn}
ncu --set full --import-source on --clock-control none -k regex:$re -c 1 \
    -o gpurun_out/${tag} python bench.py --profile-launches --steps 1 --warmup 1 > gpurun_out/${tag}_ncu.log 2>&1
ncu -i gpurun_out/${tag}.ncu-rep --page source --csv --print-source sass > gpurun_out/${tag}_source.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page raw --csv > gpurun_out/${tag}_raw.csv 2>/dev/null
ncu -i gpurun_out/${tag}.ncu-rep --page details > gpurun_out/${tag}_details.txt 2>/dev/null
tail -3 gpurun_out/${tag}_ncu.log
