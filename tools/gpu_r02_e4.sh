set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "residual or operator or solve or hmg" > gpurun_out/r02e4_pytest.log 2>&1; tail -2 gpurun_out/r02e4_pytest.log
timeout 600 python tools/sweep.py --solve --p 2,3,4 > gpurun_out/r02e4_sweep.jsonl 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02e4_bench.json 2>/dev/null
