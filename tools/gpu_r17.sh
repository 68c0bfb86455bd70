set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --p 12,16 --steps 5 > gpurun_out/sweep_r3.jsonl 2> gpurun_out/sweep_r3.err; cat gpurun_out/sweep_r3.jsonl | cut -c1-400
timeout 600 python bench.py --config 5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5b.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg5b.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['residual_kernel'], d['time_split_ms_per_step'])"
