# re-entry check: full GPU suite + smoke + default bench + degree sweep at HEAD
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/r02n_pytest.log 2>&1; tail -3 gpurun_out/r02n_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 600 python bench.py > gpurun_out/r02n_bench.json 2> gpurun_out/r02n_bench.err; tail -1 gpurun_out/r02n_bench.json | cut -c1-300
timeout 900 python tools/sweep.py --solve > gpurun_out/r02n_sweep.jsonl 2> gpurun_out/r02n_sweep.err; tail -2 gpurun_out/r02n_sweep.err
