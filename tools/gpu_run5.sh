set -x
timeout 900 python -m pytest tests/test_gpu_parity.py -q -m gpu -x 2>&1 | tail -3
for nb in 32 64 135 296; do PMG_COOP_BLOCKS=$nb timeout 300 python bench.py --no-cpu-baseline --no-e2e --steps 5 2>/dev/null | python -c "import json,sys; d=json.load(sys.stdin); print('coop_blocks', $nb, d['ms_per_step'], d['time_split_ms_per_step'])"; done
