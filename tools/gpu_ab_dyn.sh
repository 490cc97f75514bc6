bash tools/ab_c5.sh "dyn" "mixed iid" 100000 > gpurun_out/ab_dyn.log 2>&1
for a in "2400 10080 mixed" "4800 2305 iid" "4800 1023 mixed" "4800 5 mixed"; do CAPSIM_B200_LIB=paper_2306_12247_b200/_lib/libcapsim_b200_dyn.so python tools/diag_pk_parity.py $a 2>&1 | tail -1; done >> gpurun_out/ab_dyn.log
