L=paper_2306_12247_b200/_lib/libcapsim_b200_wchunk.so
for cfg in "11 0" "11 16" "10 16" "10 32" "11 32"; do set -- $cfg
  E="CAPSIM_B200_LIB=$L CS_LUT_FORCE_SHIFT=$1"; [ $2 != 0 ] && E="$E CS_PLAN_WPG=$2"
  echo "shift=$1 wpg=$2: $(env $E timeout 300 python tools/diag_config.py C3 10000 mixed | cut -c1-230)"; done
