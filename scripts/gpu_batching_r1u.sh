cd $GRAFT_REPO_ROOT
T=gpurun_out/r1u
mkdir -p $T
timeout 600 python -m pytest tests/test_batching.py -m gpu -x -q > $T/pytest_batching.log 2>&1
tail -1 $T/pytest_batching.log
timeout 900 python scripts/bench_batching.py > $T/bench_batching.json 2> $T/bench_batching.err
timeout 900 python scripts/bench_batching.py --steps 3 --no-cpu-baseline > $T/bench_batching_again.json 2> $T/bench_batching_again.err
for f in $T/bench_batching.json $T/bench_batching_again.json; do python -c "import json;d=json.load(open('$f'));print('$f', d['ms_per_step'], d['value'])"; done
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,launch__registers_per_thread --clock-control none --csv --log-file $T/launches_batching.csv \
  python scripts/bench_batching.py --steps 1 --warmup 0 --no-cpu-baseline > $T/launches_batching.json 2>&1
