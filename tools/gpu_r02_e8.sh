# k_elem16 for p = 5..8 (product build) vs k_elem_pf (libpmg_m9.so): parity, config-5 / config-2 / p = 8 sweep timing
set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -m gpu -k "residual or operator or solve_parity or neumann or periodic or krylov or table" 2>&1 | tail -2
for L in libpmg.so libpmg_m9.so libpmg.so libpmg_m9.so; do
  for C in 5 2; do
    PMG_LIB=paper_1808_03595_b200/$L timeout 300 python bench.py --config $C --steps 6 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/e8_$C.json 2>/dev/null
    python -c "import json;d=json.load(open('gpurun_out/e8_$C.json'));print('$L cfg$C', round(d['ms_per_step'],3), 'sweep', round(d['roofline']['sweep_ms'],4), 'resid', round(d['residual_kernel']['ms'],4), d['time_split_ms_per_step'])"
  done
done
