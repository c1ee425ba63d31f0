python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/search_profile.py 1 --reps 2 > gpurun_out/prof_1h.txt 2>&1
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day.txt 2>&1
ASIM_GROUP_CANDIDATES=0 python scripts/search_profile.py 1 --reps 2 > gpurun_out/prof_1h_nogroup.txt 2>&1
tail -1 gpurun_out/prof_1h.txt; tail -1 gpurun_out/prof_1h_nogroup.txt; tail -1 gpurun_out/prof_day.txt
bash scripts/ncu_heaviest.sh 'chunk_kernelIjLi0' gpurun_out/ncu_p1_1h python scripts/search_profile.py 1 --reps 1
ls gpurun_out/ncu_p1_1h
