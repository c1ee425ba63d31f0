cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r22
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r22/pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r22/bench.json 2> gpurun_out/r22/bench.err
timeout 1500 python bench.py --hours 24 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r22/bench_day.json 2> gpurun_out/r22/bench_day.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r22/launches_day.csv python bench.py --hours 24 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r22/launches_day.json 2>&1
