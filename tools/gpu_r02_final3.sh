# round-2 closing evidence (HEAD after the k_elem16 edge-stage change): GPU suite, smoke, bench lines
# (config 5 default, config 2, reference arm), ncu launch list, ncu full captures of k_elem16 / k_star16
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin3_pytest.log 2>&1; tail -2 gpurun_out/fin3_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin3_bench.json 2> gpurun_out/fin3_bench.err; tail -1 gpurun_out/fin3_bench.json | cut -c1-300
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/fin3_bench_cfg2.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/fin3_bench_reference.json 2>/dev/null
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin3_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin3_ncu_launch.log 2>&1; tail -1 gpurun_out/fin3_ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_star16" -c 8 -o gpurun_out/fin3_star16_c5 python tools/cfg5_ops.py --config 5 --reps 1 > gpurun_out/fin3_ncu_star.log 2>&1; tail -1 gpurun_out/fin3_ncu_star.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_elem16" -c 1 -o gpurun_out/fin3_elem16_c5 python tools/cfg5_ops.py --config 5 --reps 1 > gpurun_out/fin3_ncu_elem.log 2>&1; tail -1 gpurun_out/fin3_ncu_elem.log
ls gpurun_out
