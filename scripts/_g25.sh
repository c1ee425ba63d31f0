ASIM_SPLIT=1 python scripts/search_profile.py 24 --reps 2 > gpurun_out/prof_day_split256.txt 2>&1
tail -1 gpurun_out/prof_day_split256.txt | cut -c1-600
python scripts/search_profile.py 24 --reps 2 --steps > gpurun_out/prof_day256.txt 2>&1
head -2 gpurun_out/prof_day256.txt | cut -c1-600
