timeout 900 python -m pytest tests/test_gpu_bench_plans.py -x -q -k "pk or c5" 2>&1 | tail -15 > gpurun_out/pk_tests.log
python tools/diag_pk_parity.py 2400 10080 mixed >> gpurun_out/pk_tests.log 2>&1
for k in mixed iid; do python tools/diag_c5.py 100000 $k 5 2>&1 | head -2; done > gpurun_out/pk_time.log
