# Round bench pass: every BASELINE config (bench.py lines with clocks, roofline, e2e, CPU baselines),
# the reference arm, iid variants, the fp64 drop-in line and the C4 launch list. Output: gpurun_out/rb/
mkdir -p gpurun_out/rb
R=gpurun_out/rb
timeout 900 python bench.py > $R/bench_C4.json 2> $R/bench_C4.err
timeout 600 python bench.py --impl reference > $R/bench_ref_C4.json 2> $R/bench_ref_C4.err
for c in C1 C2 C3 C5; do timeout 900 python bench.py --config $c > $R/bench_$c.json 2> $R/bench_$c.err; done
timeout 600 python bench.py --config C4 --dtype f64 --no-cpu > $R/bench_C4_f64.json 2> $R/bench_C4_f64.err
for c in C3 C4 C5; do timeout 600 python bench.py --config $c --trace-kind iid --no-cpu --no-e2e > $R/bench_${c}_iid.json 2> $R/bench_${c}_iid.err; done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $R/launches_c4.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu --no-e2e > $R/launches_c4.log 2>&1
