set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
for pr in 1 0; do
  ASIM_PAIR=$pr python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_pair$pr.txt 2>&1
  tail -1 gpurun_out/prof_pair$pr.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('pair $pr', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'], [round(x/1e12,2) for x in d['spec_class_cycles']])"
done
