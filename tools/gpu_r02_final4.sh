# degree sweep and config-5 weak probe at the closing commit (after the transfer-kernel change), config-4 bench line
set -x
timeout 900 python tools/sweep.py --solve > gpurun_out/fin4_sweep.jsonl 2> gpurun_out/fin4_sweep.err; wc -l gpurun_out/fin4_sweep.jsonl
timeout 600 python bench.py --config 4 --no-cpu-baseline > gpurun_out/fin4_bench_cfg4.json 2>/dev/null; cut -c1-250 gpurun_out/fin4_bench_cfg4.json
timeout 900 python tools/weak_probe_cfg5.py > gpurun_out/fin4_weak_probe_cfg5.jsonl 2>/dev/null; wc -l gpurun_out/fin4_weak_probe_cfg5.jsonl
