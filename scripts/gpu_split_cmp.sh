# Split steps on vs off in bench mode (no profiling), plus a per-step profile (split off).
set -x
for sp in 0 1; do
  ASIM_SPLIT=$sp python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_split$sp.json 2> gpurun_out/bench_split$sp.err
  python3 -c "import json; d=json.load(open('gpurun_out/bench_split$sp.json')); print('split $sp', d['ms_per_step'], d['value'], d['roofline']['frac'])"
done
ASIM_SPLIT=0 python scripts/search_profile.py 24 --reps 1 --steps > gpurun_out/prof_day_steps.txt 2>&1; head -1 gpurun_out/prof_day_steps.txt | cut -c1-300
