python -m pytest tests/test_chunked.py tests/test_search_parity.py tests/test_determinism.py tests/test_fast_heuristic.py -x -q 2>&1 | tail -2
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day.txt 2>&1
tail -1 gpurun_out/prof_day.txt
ASIM_SCALAR_WALK=0 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_coop.txt 2>&1
tail -1 gpurun_out/prof_day_coop.txt
