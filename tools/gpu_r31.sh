for v in 0 1; do PMG_NO_L2PERSIST=$v timeout 600 python bench.py --config 5 --steps 3 --no-cpu-baseline --no-e2e > gpurun_out/bench_cfg5_l2_$v.json 2>&1
python -c "
import json; d=json.loads(open('gpurun_out/bench_cfg5_l2_$v.json').read().strip().splitlines()[-1]); print('nopersist=$v', d['value'], d['ms_per_step'], d['time_split_ms_per_step'])"; done
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "pipelined" > gpurun_out/pytest_ell.log 2>&1; tail -2 gpurun_out/pytest_ell.log
