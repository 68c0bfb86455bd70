set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02e7_pytest.log 2>&1; tail -2 gpurun_out/r02e7_pytest.log
timeout 900 python tools/sweep.py --solve > gpurun_out/r02e7_sweep.jsonl 2>/dev/null
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02e7_bench.json 2>/dev/null
