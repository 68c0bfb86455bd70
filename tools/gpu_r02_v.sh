set -x
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02v_pytest.log 2>&1; tail -3 gpurun_out/r02v_pytest.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02v_bench.json 2> gpurun_out/r02v_bench.err; tail -1 gpurun_out/r02v_bench.json | cut -c1-600
timeout 900 python tools/sweep.py --solve > gpurun_out/r02v_sweep.jsonl 2> gpurun_out/r02v_sweep.err; tail -2 gpurun_out/r02v_sweep.err
