# round 2, call A: config-5 baseline bench line + ncu captures of the star / residual kernels at config 5
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv; free -g | head -2; nproc
timeout 600 python bench.py --config 5 --no-cpu-baseline --no-e2e > gpurun_out/r02a_bench_cfg5.json 2> gpurun_out/r02a_bench_cfg5.err
tail -c 600 gpurun_out/r02a_bench_cfg5.json
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_star_pf|k_elem_pf16|k_gather_resid" -c 10 -o gpurun_out/r02a_cfg5 python tools/cfg5_ops.py --reps 1 > gpurun_out/r02a_ncu.log 2>&1
tail -3 gpurun_out/r02a_ncu.log
ls -la gpurun_out
