# f4 batching evidence (run under gpurun): parity tests, bench line, ncu launch list and full set.
cd $GRAFT_REPO_ROOT
T=gpurun_out/r1e
mkdir -p $T
timeout 600 python -m pytest tests/test_batching.py -m gpu -x -q > $T/pytest_batching.log 2>&1
timeout 900 python scripts/bench_batching.py > $T/bench_batching.json 2> $T/bench_batching.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $T/launches_batching.csv \
  python scripts/bench_batching.py --steps 1 --warmup 0 --no-cpu-baseline > $T/launches_batching.json 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:batching_kernel -c 1 \
  -o $T/batching python scripts/bench_batching.py --steps 1 --warmup 0 --no-cpu-baseline > $T/ncu_full.log 2>&1
ls -la $T
