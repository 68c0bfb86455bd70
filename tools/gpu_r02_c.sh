# round 2, call C: new p = 9..16 kernels (k_star16, k_elem16): parity, bench, ncu
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "p12 or p13 or p16 or p24 or k333_p8 or k323" > gpurun_out/r02c_pytest.log 2>&1; tail -15 gpurun_out/r02c_pytest.log
timeout 900 python -m pytest tests/test_gpu_fullsize.py -x -q -k "cfg5 or 3-12 or 3-16 or 4-None or config4" > gpurun_out/r02c_pytest_full.log 2>&1; tail -15 gpurun_out/r02c_pytest_full.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02c_bench.json 2> gpurun_out/r02c_bench.err; tail -3 gpurun_out/r02c_bench.err
PMG_NO_STAR16=1 PMG_NO_ELEM16=1 timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02c_bench_old.json 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_star16|k_elem16|k_gather_resid" -c 10 -o gpurun_out/r02c_cfg5 python tools/cfg5_ops.py --reps 1 > gpurun_out/r02c_ncu.log 2>&1
tail -3 gpurun_out/r02c_ncu.log
