# A/B of the reduce-scatter variants (experiment builds via PMG_LIB): config 5 and config 2 step, sweep and residual times
for L in libpmg.so libpmg_s2.so libpmg_s1.so libpmg.so libpmg_s2.so; do
  for C in 5 2; do
    PMG_LIB=paper_1808_03595_b200/$L timeout 300 python bench.py --config $C --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/var_$C.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/var_$C.json'));print('$L cfg$C', round(d['ms_per_step'],3), 'sweep', round(d['roofline']['sweep_ms'],4), 'resid', round(d['residual_kernel']['ms'],4), d['time_split_ms_per_step'])"
  done
done
PMG_LIB=paper_1808_03595_b200/libpmg_s2.so timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "smooth_parity or residual_parity or solve_parity" 2>&1 | tail -2
