set -x
timeout 1200 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -k "p24 or p32 or p20 or 3-24 or 3-32" > gpurun_out/r02m_pytest.log 2>&1; tail -3 gpurun_out/r02m_pytest.log
timeout 900 python tools/sweep.py --solve --p 24,32 > gpurun_out/r02m_sweep.jsonl 2> gpurun_out/r02m_sweep.err; tail -2 gpurun_out/r02m_sweep.err
timeout 600 ncu --set full --import-source on --clock-control none -k regex:"k_elem_pf|k_star16<8>" -c 3 -o gpurun_out/r02m_p8 python tools/cfg5_ops.py --config 2 --reps 1 > gpurun_out/r02m_ncu.log 2>&1
