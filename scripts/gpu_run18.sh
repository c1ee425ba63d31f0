cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r18
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r18/pytest_gpu.txt 2>&1
timeout 300 python scripts/walk_profile.py 1 4096,8192 v > gpurun_out/r18/walk.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/r18/bench.json 2> gpurun_out/r18/bench.err
