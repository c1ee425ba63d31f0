cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_fast_heuristic.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu11a.txt
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu11.txt
timeout 600 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --search fast --no-cpu-baseline --no-e2e > gpurun_out/bench11_fast.txt 2>&1
timeout 900 python bench.py --config S3 --hours 24 --steps 1 --warmup 0 --search fast --no-cpu-baseline --no-e2e > gpurun_out/bench11_fast_day.txt 2>&1
