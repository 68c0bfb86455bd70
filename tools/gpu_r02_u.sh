set -x
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so PMG_COARSE_ELL=0 timeout 300 python tools/hmg_trace.py 2 2>&1 | head -14
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_trace.so PMG_NO_L2PERSIST=1 timeout 300 python tools/hmg_trace.py 2 2>&1 | head -14
