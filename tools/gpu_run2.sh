set -x
./tools/fp64_peaks | tee gpurun_out/fp64_peaks2.jsonl
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -5
PMG_COARSE_MULTIKERNEL=1 timeout 300 python -m pytest tests/test_gpu_parity.py -q -m gpu -x -k "vcycle or solve" 2>&1 | tail -3
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; cat gpurun_out/bench_r2.json; tail -3 gpurun_out/bench_r2.err
timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_r2.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch_r2.log 2>&1
