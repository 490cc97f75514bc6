for k in mixed iid; do
  for cfg in "0 0" "768 0" "768 4" "768 8"; do set -- $cfg
    E="X=1"; [ $1 != 0 ] && E="$E CS_PLAN_THREADS=$1"; [ $2 != 0 ] && E="$E CS_PLAN_WPG=$2"
    echo "threads=$1 wpg=$2 $k: $(env $E timeout 300 python tools/diag_c5.py 100000 $k 5 2>&1 | head -2 | tr '\n' ' ' | cut -c1-330)"
  done
done
