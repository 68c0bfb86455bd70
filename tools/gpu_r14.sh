set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r14.json 2>&1
PMG_NO_PDL=1 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r14_nopdl.json 2>&1
