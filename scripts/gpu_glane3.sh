set -x
python -m pytest tests/test_chunked.py tests/test_determinism.py -m gpu -x -q > gpurun_out/pytest_glane.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_glane.log
for sm in 2 4 16; do
  ASIM_GLANE_SMAX=$sm python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_gsmax_$sm.txt 2>&1
  tail -1 gpurun_out/prof_gsmax_$sm.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('smax $sm', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done
