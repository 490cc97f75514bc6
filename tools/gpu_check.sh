# full GPU suite + kernel timings of the BASELINE configs (10^4 / 10^5 / 2x10^5 traces)
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/gpu_tests.log 2>&1; echo "rc=$?" >> gpurun_out/gpu_tests.log
for c in "C3 10000 mixed" "C3 3000 iid" "C4 200000 mixed" "C5 100000 mixed" "C2 1 mixed"; do python tools/diag_config.py $c 2>&1 | cut -c1-300; done > gpurun_out/timings.log
