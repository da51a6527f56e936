set -u
L=paper_2603_03988_b200/libsort_b200.so
for v in e2p h16; do cp tools/ablib/lib_$v.so $L; touch $L; echo "== $v"; timeout 600 python tools/logit_err.py 2>&1 | tail -2; done
cp tools/ablib/lib_h16.so $L; touch $L
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider -k "fused_tail or model_logits or golden or moe or pruned or sampled or geometric or large" 2>&1 | tail -2
ABOUT=r02h16 bash tools/ab_var.sh e2p h16
