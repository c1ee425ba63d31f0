# Pass-1 occupancy sensitivity: dynamic shared memory padded to hold 3 / 2 blocks per SM.
for pad in 0 8000 60000; do
  ASIM_P1_PAD=$pad python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_pad_$pad.txt 2>&1
  tail -1 gpurun_out/prof_pad_$pad.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('pad $pad', {k: round(d[k]) for k in ('search_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'], [round(x/1e12,2) for x in d['spec_class_cycles']])"
done
