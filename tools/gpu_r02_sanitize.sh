# compute-sanitizer memcheck over tiny solves of every kernel family (tools/sanitize_small.py)
set -x
timeout 1500 compute-sanitizer --tool memcheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_memcheck.log 2>&1
echo "memcheck exit $?"
grep -E "ERROR SUMMARY|Invalid|^\(" gpurun_out/sanitize_memcheck.log | tail -30
timeout 900 compute-sanitizer --tool racecheck --print-limit 20 python tools/sanitize_small.py > gpurun_out/sanitize_racecheck.log 2>&1
echo "racecheck exit $?"
grep -E "RACECHECK SUMMARY|hazard|^\(" gpurun_out/sanitize_racecheck.log | tail -30
