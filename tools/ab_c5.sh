#!/bin/bash
# A/B of eval_kernel variants on C5 (tools/build_variants.py): ab_c5.sh "variant..." [kinds] [traces]
V=${1:-""}; K=${2:-"mixed iid"}; T=${3:-100000}
for k in $K; do
  for v in base $V; do
    L=paper_2306_12247_b200/_lib/libcapsim_b200.so; [ $v != base ] && L=paper_2306_12247_b200/_lib/libcapsim_b200_$v.so
    echo "== $v $k"; CAPSIM_B200_LIB=$L timeout 300 python tools/diag_c5.py $T $k 10 | grep kernel
  done
done
