set -x
timeout 1500 python -m pytest tests/test_gpu_multirank.py tests/test_gpu_parity.py -m gpu -q > gpurun_out/r02x_pytest.log 2>&1; tail -3 gpurun_out/r02x_pytest.log
