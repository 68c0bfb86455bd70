set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py -q -x -k "condense or solve_parity or periodic" > gpurun_out/r02k_pytest.log 2>&1; tail -3 gpurun_out/r02k_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02k_bench.json 2> gpurun_out/r02k_bench.err; tail -3 gpurun_out/r02k_bench.err
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cr16" -c 2 -o gpurun_out/r02k_cr python tools/cfg5_ops.py --reps 0 --solve > gpurun_out/r02k_ncu.log 2>&1
