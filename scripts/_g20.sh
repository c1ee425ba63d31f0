python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
# batching: ncu launch list with instruction counts, then its I_eval
mkdir -p gpurun_out/r2batch
timeout 900 ncu --metrics smsp__inst_executed.sum,gpu__time_duration.sum --clock-control none -k regex:batching_kernel --csv --log-file gpurun_out/r2batch/launches.csv python scripts/bench_batching.py --steps 1 --warmup 0 --no-cpu-baseline > gpurun_out/r2batch/bench_ncu.json 2> gpurun_out/r2batch/bench_ncu.err
python scripts/batching_ieval.py gpurun_out/r2batch/launches.csv gpurun_out/r2batch/bench_ncu.json gpurun_out/r2batch/batching_ieval.json
python scripts/bench_batching.py --ieval gpurun_out/r2batch/batching_ieval.json > gpurun_out/r2batch/bench_batching.json 2> gpurun_out/r2batch/bench_batching.err
tail -c 1500 gpurun_out/r2batch/bench_batching.json
