for v in libpmg.so libpmg_minb4.so libpmg_minb6.so; do
  PMG_LIB=$PWD/paper_1808_03595_b200/$v timeout 300 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/ab_$v.json 2>&1
  python -c "
import json; d=json.loads(open('gpurun_out/ab_$v.json').read().strip().splitlines()[-1]); print('$v', d['value'], d['ms_per_step'], d['roofline']['sweep_ms'], d['time_split_ms_per_step'])"
done
