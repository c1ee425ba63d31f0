cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r16
timeout 900 python -m pytest tests/test_chunked.py tests/test_search_parity.py tests/test_beam.py tests/test_buckets.py -m gpu -q -x > gpurun_out/r16/pytest_gpu.txt 2>&1
ASIM_WALK_LOG=30000000 timeout 300 python scripts/walk_profile.py 1 4096 > gpurun_out/r16/walk_log.txt 2>&1
timeout 300 python scripts/walk_profile.py 1 8192,16384 > gpurun_out/r16/walk_sizes.txt 2>&1
