set -x
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --p 8,12,16,24 --solve --steps 5 > gpurun_out/sweep_r2.jsonl 2> gpurun_out/sweep_r2.err; tail -3 gpurun_out/sweep_r2.err
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_star_pf -s 40 -c 1 -o gpurun_out/prof_star16 python tools/sweep.py --p 16 --steps 2 > gpurun_out/ncu_star16.log 2>&1
