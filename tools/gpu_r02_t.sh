set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_pcg_hmg -c 1 -o gpurun_out/r02t_hmg python tools/hmg_p2.py 2 > gpurun_out/r02t_ncu.log 2>&1; tail -2 gpurun_out/r02t_ncu.log
