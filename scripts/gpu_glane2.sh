set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for gw in 0 1 2 4; do
  ASIM_SPLIT=0 ASIM_GLANE_WALK=$gw python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_glane_$gw.txt 2>&1
  tail -1 gpurun_out/prof_glane_$gw.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('glane $gw', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms','walk_critical_chunks')}, d['best_good'])"
done
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python3 -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print('bench', d['ms_per_step'], d['value'], d['roofline']['frac'])"
