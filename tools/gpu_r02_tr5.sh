# p = 8 / p = 4 sweep solve times: 32-thread (product) vs 64-thread (libpmg_t64.so) transfer blocks at p_f <= 8, alternating
for L in libpmg.so libpmg_t64.so libpmg.so libpmg_t64.so libpmg.so libpmg_t64.so; do
  PMG_LIB=paper_1808_03595_b200/$L timeout 300 python tools/sweep.py --solve --p 8,4 2>/dev/null | python -c "
import sys,json
for l in sys.stdin:
    d=json.loads(l); print('$L', d['p'], round(d['solve_ms'],3))"
done
