cd $GRAFT_REPO_ROOT
timeout 900 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu7.txt
timeout 900 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench7_s3.txt 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches7.csv python bench.py --config S3 --hours 0.25 --steps 1 --warmup 0 --no-cpu-baseline --no-e2e > /dev/null 2>&1
