# Group-lane walker for S <= 2 vs S <= 4 (ASIM_GLANE_SMAX), twice each, on the day-long S3 search.
for rep in 1 2; do for sm in 2 4; do
  ASIM_GLANE_SMAX=$sm python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_gs_${sm}_$rep.txt 2>&1
  tail -1 gpurun_out/prof_gs_${sm}_$rep.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('smax $sm rep $rep', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done; done
