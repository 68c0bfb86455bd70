# round 2, call B: the widened GPU parity suite, the paper-table / anisotropy probe, the config-5 bench
set -x
timeout 2400 python -m pytest tests -m gpu -x -q --durations=25 > gpurun_out/r02b_pytest.log 2>&1; tail -40 gpurun_out/r02b_pytest.log
timeout 900 python tools/probe_tables.py both > gpurun_out/r02b_tables.jsonl 2> gpurun_out/r02b_tables.err; tail -3 gpurun_out/r02b_tables.err
timeout 900 python bench.py --steps 10 --warmup 3 > gpurun_out/r02b_bench.json 2> gpurun_out/r02b_bench.err; tail -3 gpurun_out/r02b_bench.err; tail -c 1500 gpurun_out/r02b_bench.json
