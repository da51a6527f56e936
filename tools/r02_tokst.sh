set -u
L=paper_2603_03988_b200/libsort_b200.so
cp tools/ablib/lib_tokst.so $L; touch $L
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "tokenizer or golden or model_logits or frozen or time_bucket or oov or jsonl or async" 2>&1 | tail -2
for v in ss2 tokst; do cp tools/ablib/lib_$v.so $L; touch $L; timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_tokenize -c 4 --csv --log-file /tmp/tok_$v.csv python bench.py --no-cpu-baseline --steps 2 --warmup 1 > /dev/null 2>&1; echo "$v $(grep gpu__time /tmp/tok_$v.csv | awk -F'","' '{print $NF}' | tr -d '"' | tr '\n' ' ')"; done
ABOUT=r02tokst bash tools/ab_var.sh ss2 tokst
