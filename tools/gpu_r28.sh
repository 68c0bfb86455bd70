timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log; tail -3 gpurun_out/pytest_gpu.log
timeout 900 python tools/sweep.py --p 24,32 --solve --steps 3 > gpurun_out/sweep_r7.jsonl 2> gpurun_out/sweep_r7.err
python -c "
import json
for l in open('gpurun_out/sweep_r7.jsonl'):
    d=json.loads(l); print(d['p'], d['smoother_ms'], d['smoother_fp64_frac'], d['residual_ms'], d.get('solve_ms'))"
