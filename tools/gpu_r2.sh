set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_r2.json 2> gpurun_out/bench_r2.err; cat gpurun_out/bench_r2.json; tail -3 gpurun_out/bench_r2.err
PMG_COARSE_REG=0 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r2_noreg.json 2>&1; cat gpurun_out/bench_r2_noreg.json | cut -c1-400
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_star_dm -s 0 -c 8 -o gpurun_out/prof_star_sweep python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_star.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_elem_dm -s 0 -c 1 -o gpurun_out/prof_elem python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_elem.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:k_pcg_coop -s 0 -c 1 -o gpurun_out/prof_coarse python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_coarse.log 2>&1
ls -la gpurun_out
