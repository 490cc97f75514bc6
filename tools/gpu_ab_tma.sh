# TMA bulk-copy A/B (CS_TMA=<stages> variants) on C4/C3 kernel time; NO_BIG = main LUT (room for the rings)
bash tools/ab.sh "tma2 tma4" "C4:200000:mixed C4:200000:iid" > gpurun_out/ab_tma.log 2>&1
echo "--- CS_PLAN_NO_BIG=1" >> gpurun_out/ab_tma.log
CS_PLAN_NO_BIG=1 bash tools/ab.sh "tma2 tma4" "C4:200000:mixed C3:10000:mixed" >> gpurun_out/ab_tma.log 2>&1
