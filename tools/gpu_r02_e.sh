# round 2, call E: hygiene build (A/B kernels removed) + k_cr16 condense/recover: full GPU suite, bench, ncu
set -x
timeout 1500 python -m pytest tests -m gpu -x -q --durations=10 > gpurun_out/r02e_pytest.log 2>&1; tail -16 gpurun_out/r02e_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline > gpurun_out/r02e_bench.json 2> gpurun_out/r02e_bench.err; tail -3 gpurun_out/r02e_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file gpurun_out/r02e_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r02e_ncu_launch.log 2>&1
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_star16|k_elem16|k_cr16" -c 10 -o gpurun_out/r02e_cfg5 python tools/cfg5_ops.py --reps 1 --solve > gpurun_out/r02e_ncu.log 2>&1
tail -2 gpurun_out/r02e_ncu.log
