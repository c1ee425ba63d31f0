python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
python bench.py --steps 3 --warmup 2 > gpurun_out/bench_day.json 2> gpurun_out/bench_day.err; echo rc=$?
tail -c 2500 gpurun_out/bench_day.json
python bench.py --hours 1 --steps 5 --warmup 3 --no-cpu-baseline > gpurun_out/bench_1h.json 2> gpurun_out/bench_1h.err
tail -c 600 gpurun_out/bench_1h.json
