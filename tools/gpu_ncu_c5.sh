timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_c5_${1:-v} python tools/diag_c5.py 20000 ${2:-mixed} 1 > gpurun_out/ncu_c5.log 2>&1
