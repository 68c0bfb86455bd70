set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r3.json 2> gpurun_out/bench_r3.err; cat gpurun_out/bench_r3.json; tail -3 gpurun_out/bench_r3.err
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r3.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r3.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_star_t -s 24 -c 1 -o gpurun_out/prof_star_t python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_star_t.log 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_elem_apply_t -s 6 -c 1 -o gpurun_out/prof_elem_t python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_elem_t.log 2>&1
