# k_star16 select-free reduce-scatter: smoother parity (all degrees), full-size samples, config-5 / config-2 timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "smooth or vcycle or solve_parity or periodic or deterministic or table" 2>&1 | tail -3
timeout 600 python -m pytest tests/test_gpu_fullsize.py -x -q -m gpu 2>&1 | tail -3
timeout 300 python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sperm_bench.json 2> gpurun_out/sperm_bench.err; head -c 420 gpurun_out/sperm_bench.json; python -c "import json;d=json.load(open('gpurun_out/sperm_bench.json'));print(d['roofline']['frac'],d['roofline']['sweep_ms'],d['time_split_ms_per_step'])"
timeout 300 python bench.py --config 2 --steps 10 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/sperm_bench2.json 2> gpurun_out/sperm_bench2.err; python -c "import json;d=json.load(open('gpurun_out/sperm_bench2.json'));print(d['value'],d['ms_per_step'],d['roofline']['frac'],d['roofline']['sweep_ms'])"
