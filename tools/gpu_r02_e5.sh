set -x
PMG_LIB=$PWD/paper_1808_03595_b200/libpmg_e5.so timeout 900 python -m pytest tests/test_gpu_parity.py -q -x -k "residual or operator or solve" > gpurun_out/r02e5_pytest.log 2>&1; tail -2 gpurun_out/r02e5_pytest.log
for lib in libpmg libpmg_e5; do
PMG_LIB=$PWD/paper_1808_03595_b200/$lib.so timeout 600 python tools/sweep.py --p 5,6,7,8 > gpurun_out/r02e5_sweep_$lib.jsonl 2>/dev/null
PMG_LIB=$PWD/paper_1808_03595_b200/$lib.so timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r02e5_bench_$lib.json 2>/dev/null
done
