timeout 600 python -m pytest tests/test_gpu_multi_rank.py tests/test_gpu_abi_hardening.py -q -x 2>&1 | tail -2
for c in C1 C2; do timeout 300 python bench.py --config $c --no-cpu --no-e2e | python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print(d['config']['workload'], d['value'], d['ms_per_step'], d['gpu_launches'])"; done
