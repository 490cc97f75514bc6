set -x
bash tools/ab.sh "pf1 pf2 pf4 roll" "C3:2000:mixed C4:200000:mixed C3:2000:iid" 2>&1 | grep -v Traceback > gpurun_out/ab1.log
python tools/diag_c5.py 100000 mixed 5 2>&1 | head -2 >> gpurun_out/ab1.log
