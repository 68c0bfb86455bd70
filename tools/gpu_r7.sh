set -x
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q > gpurun_out/pytest_multirank.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_multirank.log; tail -3 gpurun_out/pytest_multirank.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -2 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_r7.json 2> gpurun_out/bench_r7.err; tail -2 gpurun_out/bench_r7.err
