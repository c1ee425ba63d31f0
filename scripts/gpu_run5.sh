cd $GRAFT_REPO_ROOT
timeout 300 python scripts/debug_paths2.py > gpurun_out/debug5.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -30 > gpurun_out/pytest_gpu5.txt
timeout 900 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench5_s3.txt 2>&1
