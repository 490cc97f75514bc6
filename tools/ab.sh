#!/bin/bash
# A/B of libcapsim_b200 variants (tools/build_variants.py) on BASELINE configs, kernel-only:
#   tools/ab.sh "variant1 variant2" "C3:10000:mixed C4:1000000:mixed ..."
V=${1:-""}; CFGS=${2:-"C4:1000000:mixed"}
for c in $CFGS; do
  IFS=: read name T kind <<< "$c"
  for v in base $V; do
    L=paper_2306_12247_b200/_lib/libcapsim_b200.so; [ $v != base ] && L=paper_2306_12247_b200/_lib/libcapsim_b200_$v.so
    echo "$v $(CAPSIM_B200_LIB=$L timeout 300 python tools/diag_config.py $name $T $kind | cut -c1-90)"
  done
done
