set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_elem16" -c 1 -o gpurun_out/r02z_elem16 python tools/cfg5_ops.py --config 5 --reps 1 > gpurun_out/r02z2_ncu.log 2>&1; tail -2 gpurun_out/r02z2_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_gather_resid" -c 1 -o gpurun_out/r02z_gather python tools/cfg5_ops.py --config 5 --reps 1 > gpurun_out/r02z3_ncu.log 2>&1; tail -2 gpurun_out/r02z3_ncu.log
