timeout 300 python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/b_small.log 2>&1 && \
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_pcg_coop_reg -s 1 -c 1 -o gpurun_out/prof_coopreg python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_coopreg.log 2>&1
