set -x
timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/r02y_c4.json 2>/dev/null; tail -1 gpurun_out/r02y_c4.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['solve']['phase_ms'])"
PMG_NO_L2PERSIST=1 timeout 600 python bench.py --config 4 --no-cpu-baseline --steps 5 > gpurun_out/r02y_c4np.json 2>/dev/null; tail -1 gpurun_out/r02y_c4np.json | python -c "import json,sys; d=json.loads(sys.stdin.read()); print(d['value']/1e9, d['ms_per_step'], d['solve']['phase_ms'])"
