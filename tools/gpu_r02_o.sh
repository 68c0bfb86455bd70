# grid-layout matrix-free h-multigrid coarse CG: parity + sweep p = 2/4/8 + config-5 bench
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hmg or coarse" > gpurun_out/r02o_pytest.log 2>&1; tail -15 gpurun_out/r02o_pytest.log
timeout 600 python tools/sweep.py --solve --p 2,4,8 > gpurun_out/r02o_sweep.jsonl 2> gpurun_out/r02o_sweep.err; tail -3 gpurun_out/r02o_sweep.err; cut -c1-400 gpurun_out/r02o_sweep.jsonl
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r02o_bench.json 2> gpurun_out/r02o_bench.err; tail -1 gpurun_out/r02o_bench.json | cut -c1-900
