# round 2, call J: ncu of the condensation / recovery kernels and the h-multigrid coarse CG at config 5
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cr16|k_pcg_hmg" -c 3 -o gpurun_out/r02j_cr python tools/cfg5_ops.py --reps 0 --solve > gpurun_out/r02j_ncu.log 2>&1
tail -2 gpurun_out/r02j_ncu.log
