# round 2, call F: k_star16 at p = 5..8, k_cr16 v2, skeleton scatter: parity subset, bench configs 5 and 2, ncu
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -x -q -k "not p32 and not p24" > gpurun_out/r02f_pytest.log 2>&1; tail -4 gpurun_out/r02f_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02f_bench.json 2> gpurun_out/r02f_bench.err; tail -3 gpurun_out/r02f_bench.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r02f_bench_cfg2.json 2> gpurun_out/r02f_bench_cfg2.err; tail -3 gpurun_out/r02f_bench_cfg2.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_cr16|k_skel_scatter|k_star16<8>" -c 12 -o gpurun_out/r02f_cfg5 python tools/cfg5_ops.py --reps 1 --solve > gpurun_out/r02f_ncu.log 2>&1
tail -2 gpurun_out/r02f_ncu.log
