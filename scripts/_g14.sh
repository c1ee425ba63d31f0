python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day.txt 2>&1
tail -1 gpurun_out/prof_day.txt
ASIM_SPLIT=0 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_nosplit.txt 2>&1
tail -1 gpurun_out/prof_day_nosplit.txt
