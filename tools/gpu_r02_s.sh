set -x
for v in pmg_trace pmg_trace3; do
PMG_LIB=$PWD/paper_1808_03595_b200/lib${v}.so timeout 300 python tools/hmg_trace.py 2 > gpurun_out/r02s_${v}_p2.txt 2>&1; head -16 gpurun_out/r02s_${v}_p2.txt
PMG_LIB=$PWD/paper_1808_03595_b200/lib${v}.so timeout 300 python tools/hmg_trace.py 16 5 > gpurun_out/r02s_${v}_c5.txt 2>&1; head -16 gpurun_out/r02s_${v}_c5.txt
done
timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "hmg or coarse or p2" > gpurun_out/r02s_pytest.log 2>&1; tail -3 gpurun_out/r02s_pytest.log
