# round 2, call H: periodic directions on the GPU + regression subset
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q -k "periodic" > gpurun_out/r02h_pytest_per.log 2>&1; tail -30 gpurun_out/r02h_pytest_per.log
timeout 1500 python -m pytest tests -m gpu -x -q -k "not p32 and not periodic" > gpurun_out/r02h_pytest.log 2>&1; tail -4 gpurun_out/r02h_pytest.log
