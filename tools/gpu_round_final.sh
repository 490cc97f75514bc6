# End-of-round GPU pass: compute-sanitizer over small launches of every kernel family, the round
# bench (tools/gpu_round_bench.sh) and the ncu captures (tools/gpu_ncu_configs.sh).
bash tools/gpu_sanitize.sh
bash tools/gpu_round_bench.sh
bash tools/gpu_ncu_configs.sh
