cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 1200 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu8.txt
timeout 600 python bench.py --config S3 --hours 1 --steps 3 --warmup 3 --search fast --no-cpu-baseline > gpurun_out/bench8_fast.txt 2>&1
bash scripts/gpu_bench_full.sh r1b
