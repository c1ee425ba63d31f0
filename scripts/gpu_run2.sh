set -x
cd $GRAFT_REPO_ROOT
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu2.txt
timeout 600 python bench.py --config S1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench2_s1.txt 2>&1
timeout 600 python bench.py --config S4 --hours 24 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench2_s4.txt 2>&1
timeout 900 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench2_s3.txt 2>&1
ls gpurun_out
