cd $GRAFT_REPO_ROOT
T=gpurun_out/r1k
mkdir -p $T
timeout 600 python -m pytest tests/test_batching.py -m gpu -x -q > $T/pytest_batching.log 2>&1
tail -1 $T/pytest_batching.log
timeout 900 python scripts/bench_batching.py > $T/bench_batching.json 2> $T/bench_batching.err
python -c "import json;d=json.load(open('$T/bench_batching.json'));print(d['ms_per_step'], d['value'], d['cpu_baseline']['value'])"
timeout 600 ncu --metrics gpu__time_duration.sum,smsp__inst_executed.sum --clock-control none --csv --log-file $T/launches_batching.csv \
  python scripts/bench_batching.py --steps 1 --warmup 0 --no-cpu-baseline > $T/launches_batching.json 2>&1
