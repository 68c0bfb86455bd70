# source-level ncu captures of the config-5 finest-level star and element kernels (one launch each)
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_star16" -s 2 -c 1 -o gpurun_out/src5_star python tools/cfg5_ops.py --reps 1 > gpurun_out/src5_star.log 2>&1; tail -2 gpurun_out/src5_star.log
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_elem16" -c 1 -o gpurun_out/src5_elem python tools/cfg5_ops.py --reps 1 > gpurun_out/src5_elem.log 2>&1; tail -2 gpurun_out/src5_elem.log
ls -la gpurun_out/
