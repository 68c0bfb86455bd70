# h-multigrid per-phase barrier trace (p = 2 and p = 4 sweep meshes, config 5) + p = 2 residual check
set -x
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 2 > gpurun_out/r02q_trace_p2.txt 2>&1; cat gpurun_out/r02q_trace_p2.txt
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so timeout 300 python tools/hmg_trace.py 16 5 > gpurun_out/r02q_trace_c5.txt 2>&1; cat gpurun_out/r02q_trace_c5.txt
timeout 600 python -m pytest tests/test_gpu_parity.py -q -x -k "residual or p2" > gpurun_out/r02q_pytest.log 2>&1; tail -3 gpurun_out/r02q_pytest.log
timeout 600 python tools/sweep.py --solve --p 2 > gpurun_out/r02q_sweep.jsonl 2> gpurun_out/r02q_sweep.err; cut -c1-700 gpurun_out/r02q_sweep.jsonl
