cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r14
timeout 600 python -m pytest tests/test_chunked.py tests/test_search_parity.py -m gpu -q -x > gpurun_out/r14/pytest_gpu.txt 2>&1
timeout 300 python scripts/walk_profile.py 1 4096 v > gpurun_out/r14/walk_4096.txt 2>&1
timeout 600 python scripts/walk_profile.py 1 1024,2048,8192,16384 > gpurun_out/r14/walk_sizes.txt 2>&1
ASIM_SCALAR_WALK=0 timeout 300 python scripts/walk_profile.py 1 4096 > gpurun_out/r14/walk_noscalar.txt 2>&1
