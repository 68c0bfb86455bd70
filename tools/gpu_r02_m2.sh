set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hmg or coarse or p2" > gpurun_out/r02m2_pytest.log 2>&1; tail -2 gpurun_out/r02m2_pytest.log
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 2 > gpurun_out/r02m2_trace_p2.txt 2>&1; head -14 gpurun_out/r02m2_trace_p2.txt
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 16 5 > gpurun_out/r02m2_trace_c5.txt 2>&1; head -14 gpurun_out/r02m2_trace_c5.txt
timeout 600 python tools/sweep.py --solve --p 2,4 > gpurun_out/r02m2_sweep.jsonl 2>/dev/null
