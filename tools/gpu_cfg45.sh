timeout 600 python bench.py --config 4 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg4.json 2>&1
timeout 900 python bench.py --config 5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5.json 2>&1
for f in bench_cfg4 bench_cfg5; do python -c "
import json; d=json.loads(open('gpurun_out/$f.json').read().strip().splitlines()[-1]); print('$f', d['value'], d['ms_per_step'], d['config']['cycles'], d['config']['coarse_iters'], d['roofline']['sweep_ms'], d['roofline']['frac'], d['residual_kernel'], d['time_split_ms_per_step'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_cfg4.csv python bench.py --config 4 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_cfg4.log 2>&1
