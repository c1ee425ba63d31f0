cd $GRAFT_REPO_ROOT
timeout 300 python scripts/debug_search_paths.py > gpurun_out/debug3.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu3.txt
