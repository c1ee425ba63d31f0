# GPU suite, then the day-long S3 search profile and a short bench.
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day.txt 2>&1
tail -1 gpurun_out/prof_day.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print({k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'], [round(x/1e12,2) for x in d['spec_class_cycles']])"
python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err
python3 -c "import json; d=json.load(open('gpurun_out/bench_quick.json')); print('bench', d['ms_per_step'], d['value'], d['roofline']['frac'])"
