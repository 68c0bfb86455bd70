# k_elem16 edge-stage change: parity (residual / operator / solve, periodic + Neumann) and config-5 timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "residual or operator or solve_parity or neumann or periodic" 2>&1 | tail -4
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e16_bench.json 2> gpurun_out/e16_bench.err; tail -c 1500 gpurun_out/e16_bench.json
