set -x
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_nt64.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "residual" > gpurun_out/r02e6_pytest.log 2>&1; tail -2 gpurun_out/r02e6_pytest.log
for lib in libpmg libpmg_nt64; do PMG_LIB=$PWD/paper_1808_03595_b200/$lib.so timeout 600 python tools/sweep.py --p 3,4 > gpurun_out/r02e6_sweep_$lib.jsonl 2>/dev/null; done
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_elem_pf|k_gather" -c 2 -o gpurun_out/r02e6_p4 python tools/cfg5_ops.py --config 3 --p 4 --reps 1 > /dev/null 2>&1
