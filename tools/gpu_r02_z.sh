set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_elem16|k_star16|k_gather_resid" -c 4 -o gpurun_out/r02z_c5 python tools/cfg5_ops.py --config 5 --reps 1 > gpurun_out/r02z_ncu.log 2>&1; tail -2 gpurun_out/r02z_ncu.log
