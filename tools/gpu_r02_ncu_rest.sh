# ncu --set full of the remaining top kernels of the config-5 step: condensation / recovery (k_cr16),
# the p = 8 / p = 4 element operators (k_elem_pf), the residual gather and the h-multigrid coarse CG
set -x
timeout 900 ncu --set full --import-source on --clock-control none -k regex:"k_cr16|k_elem_pf|k_gather_resid|k_pcg_hmg|k_prolong|k_restrict_local" -c 14 -o gpurun_out/rest_c5 python tools/cfg5_ops.py --config 5 --reps 0 --solve > gpurun_out/rest_ncu.log 2>&1; tail -2 gpurun_out/rest_ncu.log
ls -la gpurun_out
