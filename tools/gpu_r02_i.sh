set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -k "periodic" > gpurun_out/r02i_pytest_per.log 2>&1; tail -30 gpurun_out/r02i_pytest_per.log
