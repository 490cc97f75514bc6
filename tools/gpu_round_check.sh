set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/r2s3_gputests.log 2>&1; echo rc=$? >> gpurun_out/r2s3_gputests.log
for c in C4 C5 C3 C2 C1; do timeout 600 python bench.py --config $c --no-cpu > gpurun_out/r2s3_bench_$c.json 2> gpurun_out/r2s3_bench_$c.err; done
timeout 600 python bench.py --config C4 --dtype f64 --no-cpu > gpurun_out/r2s3_bench_C4_f64.json 2> gpurun_out/r2s3_bench_C4_f64.err
tail -3 gpurun_out/r2s3_gputests.log
