set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r21.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_r21.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['time_split_ms_per_step'])"
timeout 900 python tools/sweep.py --solve --steps 3 > gpurun_out/sweep_r6.jsonl 2> gpurun_out/sweep_r6.err; tail -2 gpurun_out/sweep_r6.err
timeout 600 python bench.py --config 5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5c.json 2>&1
timeout 600 python bench.py --config 4 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4c.json 2>&1
