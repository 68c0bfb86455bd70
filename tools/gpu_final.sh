set -x
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; tail -1 gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err; tail -2 gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 3 > gpurun_out/bench_reference.json 2> gpurun_out/bench_reference.err; tail -2 gpurun_out/bench_reference.err
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active --clock-control none --csv --log-file gpurun_out/launches_final.csv python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none -k regex:k_star_pf -s 0 -c 8 -o gpurun_out/prof_star_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_star.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:k_elem_pf -s 10 -c 1 -o gpurun_out/prof_elem_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_elem.log 2>&1
timeout 900 ncu --set full --cache-control none --clock-control none -k regex:k_pcg_gv_p2 -s 2 -c 1 -o gpurun_out/prof_coarse_final python bench.py --steps 1 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/ncu_coarse.log 2>&1
timeout 900 python tools/weak_probe.py > gpurun_out/weak_probe.jsonl 2>&1
du -sh gpurun_out; ls -la gpurun_out
