for mc in 128 64 32; do
ASIM_MAX_CHUNKS=$mc python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_mc$mc.txt 2>&1
tail -1 gpurun_out/prof_day_mc$mc.txt | cut -c1-700
done
