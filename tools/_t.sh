mkdir -p gpurun_out/rb
timeout 900 python bench.py --config C3 > gpurun_out/rb/bench_C3.json 2> gpurun_out/rb/bench_C3.err
timeout 600 python bench.py --config C3 --trace-kind iid --no-cpu --no-e2e > gpurun_out/rb/bench_C3_iid.json 2> gpurun_out/rb/bench_C3_iid.err
