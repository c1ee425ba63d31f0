# Walker correctness (chunked, determinism, search parity) and the day-long S3 search profile.
set -x
python -m pytest tests/test_chunked.py tests/test_determinism.py tests/test_search_parity.py -m gpu -x -q > gpurun_out/pytest_part.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_part.log
for r in 1 2; do
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_$r.txt 2>&1
tail -1 gpurun_out/prof_day_$r.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done
