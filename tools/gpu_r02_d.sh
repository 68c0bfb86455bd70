# round 2, call D: k_star16 / k_elem16 v2 -- parity subset, bench, ncu
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p12 or p13 or p16 or k333_p8 or k323 or neumann" > gpurun_out/r02d_pytest.log 2>&1; tail -5 gpurun_out/r02d_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_multirank.py -x -q -k "cfg5 or 3-12 or 3-16 or 4-None or config4 or multirank or slab or nccl" > gpurun_out/r02d_pytest_full.log 2>&1; tail -5 gpurun_out/r02d_pytest_full.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02d_bench.json 2> gpurun_out/r02d_bench.err; tail -3 gpurun_out/r02d_bench.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_star16|k_elem16" -c 9 -o gpurun_out/r02d_cfg5 python tools/cfg5_ops.py --reps 1 > gpurun_out/r02d_ncu.log 2>&1
tail -2 gpurun_out/r02d_ncu.log
