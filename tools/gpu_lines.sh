# degree sweep + one-GPU bench lines for configs 4 and 5 (slab)
timeout 900 python tools/sweep.py --solve > gpurun_out/sweep.jsonl 2> gpurun_out/sweep.err
timeout 600 python bench.py --config 5 --no-cpu-baseline > gpurun_out/bench_cfg5.json 2> gpurun_out/bench_cfg5.err
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/bench_cfg4.json 2> gpurun_out/bench_cfg4.err
for f in bench_cfg5 bench_cfg4; do tail -1 gpurun_out/$f.json | cut -c1-200; done
