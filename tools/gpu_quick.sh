# parity tests + one bench summary line (used after every kernel change)
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -2
timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>gpurun_out/quick.err | python -c "import json,sys; d=json.load(sys.stdin); print('ms', round(d['ms_per_step'],3), 'Munk/s', round(d['value']/1e6,1), {k: round(v,3) for k,v in d['time_split_ms_per_step'].items()}, 'sweep', round(d['roofline']['sweep_ms'],4), 'frac', round(d['roofline']['frac'],4), 'res', round(d['residual_kernel']['ms'],4))"
