# full GPU suite + smoke + degree sweep + one-GPU bench lines for configs 4 and 5 (slab)
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
timeout 900 python tools/sweep.py --solve > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
for f in bench_cfg5 bench_cfg4; do tail -1 gpurun_out/$f.json | cut -c1-200; done
