timeout 600 python -m pytest tests/test_gpu_parity.py -x -q -k "neumann" > gpurun_out/pytest_neu.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_neu.log; tail -25 gpurun_out/pytest_neu.log
timeout 600 python -m pytest tests/test_gpu_multirank.py -x -q -k "neumann" > gpurun_out/pytest_neu_mr.log 2>&1; echo "rc=$?" >> gpurun_out/pytest_neu_mr.log; tail -5 gpurun_out/pytest_neu_mr.log
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/bench_r29.json 2>&1; python -c "
import json; d=json.loads(open('gpurun_out/bench_r29.json').read().strip().splitlines()[-1]); print(d['value'], d['ms_per_step'])"
