# ncu source-level capture of the grid h-multigrid coarse CG at p = 2 (128^3 elements)
set -x
timeout 300 python tools/hmg_p2.py 2
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_hmg -c 1 -o gpurun_out/r02p_hmg python tools/hmg_p2.py 2 > gpurun_out/r02p_ncu.log 2>&1; tail -3 gpurun_out/r02p_ncu.log
