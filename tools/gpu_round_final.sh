# End-of-round GPU pass: compute-sanitizer over small launches of every kernel family, the round
# bench (tools/gpu_round_bench.sh) and the ncu captures (tools/gpu_ncu_configs.sh).
mkdir -p gpurun_out/san
for t in memcheck racecheck synccheck; do
  timeout 600 compute-sanitizer --tool $t python tools/sanitize_small.py > gpurun_out/san/san_$t.log 2>&1
done
bash tools/gpu_round_bench.sh
bash tools/gpu_ncu_configs.sh
