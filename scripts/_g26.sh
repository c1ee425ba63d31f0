python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
python scripts/search_profile.py 24 --reps 2 > gpurun_out/prof_day_split.txt 2>&1
tail -1 gpurun_out/prof_day_split.txt | cut -c1-600
