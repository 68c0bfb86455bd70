# one ncu --set full capture with source correlation per hot kernel (config 2, inside a solve)
rm -f gpurun_out/src_*.ncu-rep
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_elem_pf -s 10 -c 1 -o gpurun_out/src_elem python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_src_elem.log 2>&1
timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_star_pf -s 16 -c 1 -o gpurun_out/src_star python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_src_star.log 2>&1
ls -la gpurun_out/src_*
