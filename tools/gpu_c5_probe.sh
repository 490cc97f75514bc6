# C5 plan probe: kernel time per forced worker-group size, then ncu --set full of the C5 / C3 kernels
set -x
for w in 0 2 4 8 16; do
  if [ $w = 0 ]; then python tools/diag_c5.py 100000 mixed 5 | head -2; else CS_PLAN_WPG=$w python tools/diag_c5.py 100000 mixed 5 | head -2; fi
done 2>&1 | tee gpurun_out/c5_wpg.log
CS_PLAN_WPG=4 python tools/diag_c5.py 100000 iid 5 | head -2 | tee -a gpurun_out/c5_wpg.log
CS_PLAN_WPG=4 timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 3 -c 1 \
  -o gpurun_out/ncu_c5_wpg4 python tools/diag_c5.py 20000 mixed 1 > gpurun_out/ncu_c5.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:eval_kernel -s 2 -c 1 \
  -o gpurun_out/ncu_c3 python tools/diag_config.py C3 1000 > gpurun_out/ncu_c3.log 2>&1
ls -la gpurun_out
