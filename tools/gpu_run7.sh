set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print(d['ms_per_step'], d['time_split_ms_per_step'], d['roofline']['sweep_ms'], d['roofline']['frac'], d['residual_kernel']['ms'])"
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_coop -s 1 -c 1 -o gpurun_out/prof_coop python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_coop.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_star_sp -s 24 -c 1 -o gpurun_out/prof_star_sp python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_star_sp.log 2>&1
