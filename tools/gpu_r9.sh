set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r9.json 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_star_pf -s 24 -c 1 -o gpurun_out/prof_star_pf3 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_star.log 2>&1
