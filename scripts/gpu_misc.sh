# compute-sanitizer over every kernel family; chunk-count sweep of the day search; the 1-h secondary bench line.
set -x
bash tests/sanitize.sh gpurun_out/sanitizer; cat gpurun_out/sanitizer/summary.txt
for mc in 128 192 384; do
  ASIM_MAX_CHUNKS=$mc python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_mc$mc.txt 2>&1
  tail -1 gpurun_out/prof_mc$mc.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('mc $mc', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done
python bench.py --hours 1 --steps 5 --warmup 3 > gpurun_out/bench_1h.json 2> gpurun_out/bench_1h.err
python3 -c "import json; d=json.load(open('gpurun_out/bench_1h.json')); print('1h', d['ms_per_step'], d['value'], d['roofline']['frac'])"
