timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for v in 0 1; do PMG_STAR_VARIANT=$v timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('variant', $v, d['ms_per_step'], d['time_split_ms_per_step'], d['roofline']['sweep_ms'], d['roofline']['frac'], d['residual_kernel']['ms'])"; done
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_star_dm -s 24 -c 1 -o gpurun_out/prof_star_dm python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_star_dm.log 2>&1
