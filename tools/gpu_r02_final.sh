# round-2 evidence: bench lines (config 5 default, configs 2 / 4), reference arm, weak-scaling probe,
# ncu launch list of the bench command, ncu full capture of one config-5 star sweep, h-multigrid traces
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_throttle_reasons.active --format=csv
timeout 900 python bench.py > gpurun_out/fin_bench.json 2> gpurun_out/fin_bench.err; tail -1 gpurun_out/fin_bench.json | cut -c1-300
timeout 600 python bench.py --config 2 --no-cpu-baseline > gpurun_out/fin_bench_cfg2.json 2>/dev/null
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/fin_bench_cfg4.json 2>/dev/null
timeout 900 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/fin_bench_reference.json 2>/dev/null
timeout 900 python tools/weak_probe_cfg5.py > gpurun_out/fin_weak_probe_cfg5.jsonl 2>/dev/null
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 2 > gpurun_out/fin_hmg_trace_p2.txt 2>&1
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 16 5 > gpurun_out/fin_hmg_trace_c5.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/fin_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/fin_ncu_launch.log 2>&1; tail -1 gpurun_out/fin_ncu_launch.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_star16" -c 8 -o gpurun_out/fin_star16_c5 python tools/cfg5_ops.py --config 5 --reps 1 > gpurun_out/fin_ncu_star.log 2>&1; tail -1 gpurun_out/fin_ncu_star.log
