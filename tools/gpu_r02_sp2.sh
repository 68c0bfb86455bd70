set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "smooth or p2 or periodic or neumann or vcycle" > gpurun_out/r02sp2_pytest.log 2>&1; tail -2 gpurun_out/r02sp2_pytest.log
timeout 600 python tools/sweep.py --p 2 > gpurun_out/r02sp2_sweep.jsonl 2>/dev/null; cut -c1-400 gpurun_out/r02sp2_sweep.jsonl
