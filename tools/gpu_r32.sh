timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined" > gpurun_out/pytest_ell.log 2>&1; tail -2 gpurun_out/pytest_ell.log
