timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "hmg" > gpurun_out/pytest_hmg.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_hmg.log; tail -3 gpurun_out/pytest_hmg.log
timeout 600 python bench.py --config 5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5_hmg.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg5_hmg.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['config']['coarse_iters'], d['time_split_ms_per_step'])"
timeout 900 python tools/weak_probe.py > gpurun_out/weak_probe4.jsonl 2>&1; cat gpurun_out/weak_probe4.jsonl
