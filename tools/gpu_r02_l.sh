# round 2, call L: gather fix; bench cfg5 + cfg2 + cfg4; degree sweep; config-5 weak probe
set -x
timeout 600 python bench.py --steps 10 --warmup 3 > gpurun_out/r02l_bench.json 2> gpurun_out/r02l_bench.err; tail -3 gpurun_out/r02l_bench.err
timeout 600 python bench.py --config 2 --steps 20 --warmup 5 > gpurun_out/r02l_bench_cfg2.json 2> gpurun_out/r02l_bench_cfg2.err
timeout 600 python bench.py --config 4 --steps 10 --warmup 3 > gpurun_out/r02l_bench_cfg4.json 2> gpurun_out/r02l_bench_cfg4.err
timeout 900 python tools/sweep.py --solve > gpurun_out/r02l_sweep.jsonl 2> gpurun_out/r02l_sweep.err; tail -2 gpurun_out/r02l_sweep.err
timeout 900 python tools/weak_probe_cfg5.py > gpurun_out/r02l_weak_cfg5.jsonl 2> gpurun_out/r02l_weak_cfg5.err; tail -2 gpurun_out/r02l_weak_cfg5.err
