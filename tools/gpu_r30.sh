timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct --cache-control none --clock-control none -k regex:k_pcg_gv_ell -c 3 --csv python bench.py --config 5 --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_ell.csv 2>&1
grep -E "k_pcg_gv_ell" gpurun_out/ncu_ell.csv | head -12
