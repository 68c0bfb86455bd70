timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r40.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_r40.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
for c in 4 5; do timeout 600 python bench.py --config $c --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg${c}_r40.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg${c}_r40.json').read().strip().splitlines()[-1]); print($c, d['value'], d['ms_per_step'], d['config']['coarse_iters'], d['time_split_ms_per_step'])"; done
timeout 900 python tools/sweep.py --solve --steps 3 > gpurun_out/sweep_r10.jsonl 2>&1; python -c "
import json
for l in open('gpurun_out/sweep_r10.jsonl'):
    d=json.loads(l); print(d['p'], round(d['smoother_ms'],3), round(d['residual_ms'],3), round(d.get('solve_ms'),2), d.get('coarse_iters'), d.get('cycles'), round(d['ns_per_unknown'],2))"
timeout 900 python tools/weak_probe.py > gpurun_out/weak_probe5.jsonl 2>&1; cat gpurun_out/weak_probe5.jsonl
