python -m pytest tests/test_determinism.py tests/test_search_parity.py tests/test_shard_emulation.py -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
ASIM_LANE_WALK=1 python -m pytest tests/test_search_parity.py tests/test_shard_emulation.py -x -q 2>&1 | tail -2
ASIM_LANE_WALK=1 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_item.txt 2>&1
tail -1 gpurun_out/prof_day_item.txt
