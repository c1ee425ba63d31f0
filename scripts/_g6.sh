python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/search_profile.py 1 --reps 2 > gpurun_out/prof_1h.txt 2>&1
tail -1 gpurun_out/prof_1h.txt
python scripts/search_profile.py 24 --reps 1 --steps > gpurun_out/prof_day.txt 2>&1
head -2 gpurun_out/prof_day.txt
