# ncu --set full of the eval kernel per BASELINE config (DRAM traffic per timestep for bench.py's
# roofline.traffic, instruction mix, stalls); summaries (JSON + SASS hot lists) under gpurun_out/ncu/,
# the reports themselves are deleted on the box unless KEEP names them (gpurun_out is capped at 64 MiB)
mkdir -p gpurun_out/ncu
N="ncu --set full --clock-control none --import-source on -k regex:eval_kernel -c 1"
run() {  # name traces steps cmd...
  local n=$1 T=$2 S=$3; shift 3
  timeout 600 $N -o gpurun_out/ncu/$n "$@" > gpurun_out/ncu/$n.log 2>&1
  python tools/ncu_summary.py gpurun_out/ncu/$n.ncu-rep --traces $T --steps $S --out gpurun_out/ncu/$n.json > /dev/null 2>&1
  python tools/sass_hot.py gpurun_out/ncu/$n.ncu-rep $((T * S)) 40 > gpurun_out/ncu/${n}_sass.txt 2>&1
  case " $KEEP " in *" $n "*) ;; *) rm -f gpurun_out/ncu/$n.ncu-rep ;; esac
}
run c4 100000 10080 -s 2 python tools/diag_config.py C4 100000 mixed
run c3 1184 604800 -s 2 python tools/diag_config.py C3 1184 mixed
run c5 20000 10080 -s 3 python tools/diag_c5.py 20000 mixed 1
run c4_f64 50000 10080 -s 2 python tools/diag_f64.py 50000
