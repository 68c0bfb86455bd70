set -x
timeout 1500 python tools/sweep.py --solve --steps 5 > gpurun_out/sweep_r1.jsonl 2> gpurun_out/sweep_r1.err; tail -5 gpurun_out/sweep_r1.err
cat gpurun_out/sweep_r1.jsonl
