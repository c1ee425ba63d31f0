# One build -> measure iteration: GPU suite, then the day-long S3 search profile (split off and on).
set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
ASIM_SPLIT=0 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_nosplit.txt 2>&1; tail -1 gpurun_out/prof_day_nosplit.txt | cut -c1-1500
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_split.txt 2>&1; tail -1 gpurun_out/prof_day_split.txt | cut -c1-1500
