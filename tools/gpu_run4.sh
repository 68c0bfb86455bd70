set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r4.json 2> gpurun_out/bench_r4.err; cat gpurun_out/bench_r4.json; tail -3 gpurun_out/bench_r4.err
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r4.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r4.log 2>&1
