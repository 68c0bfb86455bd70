set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_elem_pf" -c 1 -o gpurun_out/r02z_elempf8 python tools/cfg5_ops.py --config 3 --p 8 --reps 1 > gpurun_out/r02z4_ncu.log 2>&1; tail -1 gpurun_out/r02z4_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_elem_pf" -c 1 -o gpurun_out/r02z_elempf4 python tools/cfg5_ops.py --config 3 --p 4 --reps 1 > gpurun_out/r02z5_ncu.log 2>&1; tail -1 gpurun_out/r02z5_ncu.log
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_star" -c 1 -o gpurun_out/r02z_star4 python tools/cfg5_ops.py --config 3 --p 4 --reps 1 > gpurun_out/r02z6_ncu.log 2>&1; tail -1 gpurun_out/r02z6_ncu.log
