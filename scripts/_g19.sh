ASIM_SCALAR_WALK=0 python -m pytest tests/test_chunked.py tests/test_search_parity.py tests/test_determinism.py tests/test_shard_emulation.py -x -q 2>&1 | tail -2
ASIM_SCALAR_WALK=0 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_hl.txt 2>&1
tail -1 gpurun_out/prof_day_hl.txt
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day.txt 2>&1
tail -1 gpurun_out/prof_day.txt
