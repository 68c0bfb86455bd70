# A/B: k_star16 L2 prefetch of the scatter's u blocks (libpmg_pf.so) vs without (libpmg.so)
for L in libpmg.so libpmg_pf.so libpmg.so libpmg_pf.so; do
  for C in 5 2; do
    PMG_LIB=paper_1808_03595_b200/$L timeout 300 python bench.py --config $C --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/pf_$C.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/pf_$C.json'));print('$L cfg$C', round(d['ms_per_step'],3), 'sweep', round(d['roofline']['sweep_ms'],4), 'resid', round(d['residual_kernel']['ms'],4), d['time_split_ms_per_step'])"
  done
done
