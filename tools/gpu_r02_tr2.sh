# register-tiled transfer kernels: parity (operators, V-cycle, solve, multirank bitwise), bench, launch list
set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_multirank.py -x -q -m gpu -k "transfer or restrict or prolong or vcycle or solve or operators or neumann or periodic" > gpurun_out/tr2_pytest.log 2>&1; tail -3 gpurun_out/tr2_pytest.log
timeout 600 python bench.py --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tr2_bench.json 2>/dev/null; cut -c1-200 gpurun_out/tr2_bench.json
python -c "import json;d=json.load(open('gpurun_out/tr2_bench.json'));print(d['ms_per_step'],d['solve'],d['time_split_ms_per_step'])"
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -c 3000 --csv --log-file gpurun_out/tr2_launches.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/tr2_ncu_launch.log 2>&1; tail -1 gpurun_out/tr2_ncu_launch.log | cut -c1-100
