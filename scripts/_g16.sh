ASIM_SCALAR_WALK=0 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_coop.txt 2>&1
tail -1 gpurun_out/prof_day_coop.txt
