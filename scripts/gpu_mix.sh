# Speculation source for re-simulated candidates: 0 = mix (default), 1 = own previous states, 2 = base only.
for mm in 1 2 0; do
  ASIM_MIX_MODE=$mm python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_mix$mm.txt 2>&1
  tail -1 gpurun_out/prof_mix$mm.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('mix $mm', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms','walk_critical_chunks','chunk_reruns','walk_candidates')}, d['best_good'])"
done
