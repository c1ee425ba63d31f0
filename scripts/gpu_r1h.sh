# Full GPU suite + both bench lines (headline S3 search, f4 batching).
cd $GRAFT_REPO_ROOT
T=gpurun_out/r1h
mkdir -p $T
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $T/pytest_gpu.log 2>&1
tail -2 $T/pytest_gpu.log; tail -1 $T/smoke.log
timeout 900 python scripts/bench_batching.py > $T/bench_batching.json 2> $T/bench_batching.err
head -c 400 $T/bench_batching.json; echo
timeout 1200 python bench.py > $T/bench.json 2> $T/bench.err
head -c 400 $T/bench.json
