for mc in 2048 4096; do
ASIM_MAX_CHUNKS=$mc python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_mc$mc.txt 2>&1
tail -1 gpurun_out/prof_day_mc$mc.txt
done
ASIM_MAX_CHUNKS=4096 python scripts/search_profile.py 24 --reps 1 --chunk 2048 > gpurun_out/prof_day_mc4096_c2048.txt 2>&1
tail -1 gpurun_out/prof_day_mc4096_c2048.txt
