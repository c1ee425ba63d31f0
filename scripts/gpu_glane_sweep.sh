# Group-lane walker routing sweep on the day-long S3 search: (smallest component in groups, largest stage count).
for cfg in "2 2" "4 4" "2 4" "4 16"; do
  set -- $cfg
  ASIM_GLANE_WALK=$1 ASIM_GLANE_SMAX=$2 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_gl_$1_$2.txt 2>&1
  tail -1 gpurun_out/prof_gl_$1_$2.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('glane $1 smax $2', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done
