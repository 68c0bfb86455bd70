set -x
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -q -x -k "transfer or restrict or prolong or vcycle or solve or recurrence" > gpurun_out/r02tr_pytest.log 2>&1; tail -2 gpurun_out/r02tr_pytest.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02tr_bench.json 2>/dev/null
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"k_prolong|k_restrict" -c 12 --csv --log-file gpurun_out/r02tr_launches.csv python tools/cfg5_ops.py --config 5 --reps 1 --solve > /dev/null 2>&1
