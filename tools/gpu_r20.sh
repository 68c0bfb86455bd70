set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r20.json 2>&1
PMG_STAR_VARIANT=3 timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r20_pf.json 2>&1
timeout 600 python tools/sweep.py --p 4 --steps 5 > gpurun_out/sweep_r5.jsonl 2>&1
for f in bench_r20 bench_r20_pf; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['time_split_ms_per_step'])"; done
cat gpurun_out/sweep_r5.jsonl | cut -c1-300
