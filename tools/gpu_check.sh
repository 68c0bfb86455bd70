timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -2 gpurun_out/pytest_gpu.log
for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_chk_$i.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_chk_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['gpu_launches'], d['time_split_ms_per_step'])"; done
