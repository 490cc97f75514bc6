#!/bin/bash
# A/B of the working-tree library against libcapsim_b200_base.so (the last commit built aside:
# `git stash; python -c "from paper_2306_12247_b200 import build as b; b.build(out=b.LIBDIR/'libcapsim_b200_base.so')"; git stash pop`),
# kernel-only, alternating twice per config:   tools/ab_base.sh ["C3:10000:mixed C4:1000000:mixed ..."]
CFGS=${1:-"C3:10000:mixed C4:1000000:mixed C4:125000:mixed C5:20000:mixed C1:1:solar C2:1:mixed"}
for c in $CFGS; do
  IFS=: read name T kind <<< "$c"
  for r in 1 2; do
    for v in base new; do
      L=paper_2306_12247_b200/_lib/libcapsim_b200.so; [ $v = base ] && L=paper_2306_12247_b200/_lib/libcapsim_b200_base.so
      echo "$v $(CAPSIM_B200_LIB=$L timeout 300 python tools/diag_config.py $name $T $kind | cut -c1-100)"
    done
  done
done
