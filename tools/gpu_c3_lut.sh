# C3 layout probe: LUT shift x worker-group size x CTA histogram (kernel time, 10^4 traces)
for cfg in "12 0 0" "12 0 1" "11 16 1" "11 32 1" "10 32 1" "11 8 1"; do
  set -- $cfg
  E="CS_PLAN_GH_DIRECT=$3"; [ $1 != 12 ] && E="$E CS_LUT_FORCE_SHIFT=$1"; [ $2 != 0 ] && E="$E CS_PLAN_WPG=$2"
  echo "shift=$1 wpg=$2 direct=$3: $(env $E python tools/diag_config.py C3 10000 mixed | cut -c1-260)"
done
