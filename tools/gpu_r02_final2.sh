# round-2 evidence refresh after the p = 2 smoother: GPU suite, smoke, bench (config 5), degree sweep
set -x
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/fin2_pytest.log 2>&1; tail -2 gpurun_out/fin2_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -1
timeout 900 python bench.py > gpurun_out/fin2_bench.json 2> gpurun_out/fin2_bench.err; tail -1 gpurun_out/fin2_bench.json | cut -c1-200
timeout 900 python tools/sweep.py --solve > gpurun_out/fin2_sweep.jsonl 2>/dev/null
