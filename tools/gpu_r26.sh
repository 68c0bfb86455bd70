for i in 1 2; do timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r26_$i.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_r26_$i.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'], d['roofline']['sweep_ms'], d['time_split_ms_per_step'])"; done
