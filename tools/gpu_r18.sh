timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_elem_pf16 -s 2 -c 1 -o gpurun_out/prof_elem16 python tools/sweep.py --p 16 --steps 2 > gpurun_out/ncu_elem16.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none --import-source on -k regex:k_star_pf -s 10 -c 1 -o gpurun_out/prof_star16 python tools/sweep.py --p 16 --steps 2 > gpurun_out/ncu_star16.log 2>&1
tail -3 gpurun_out/ncu_elem16.log gpurun_out/ncu_star16.log
