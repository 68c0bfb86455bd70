set -x
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 2 > gpurun_out/r02r_trace_p2.txt 2>&1; head -14 gpurun_out/r02r_trace_p2.txt
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 16 5 > gpurun_out/r02r_trace_c5.txt 2>&1; head -14 gpurun_out/r02r_trace_c5.txt
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "residual or p2 or hmg or coarse or operator" > gpurun_out/r02r_pytest.log 2>&1; tail -3 gpurun_out/r02r_pytest.log
timeout 600 python tools/sweep.py --solve --p 2,4 > gpurun_out/r02r_sweep.jsonl 2> gpurun_out/r02r_sweep.err; cut -c1-100,600-800 gpurun_out/r02r_sweep.jsonl
