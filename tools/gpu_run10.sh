timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['time_split_ms_per_step'], d['roofline']['sweep_ms'], d['roofline']['frac'], d['residual_kernel']['ms'], d['gpu_launches'])"
