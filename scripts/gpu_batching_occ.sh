# Occupancy sweep of the batching kernel (ASIM_BATCH_MINB = 4 / 6 / 8).
cd $GRAFT_REPO_ROOT
T=gpurun_out/r1i
mkdir -p $T
timeout 600 python -m pytest tests/test_batching.py -m gpu -x -q > $T/pytest_batching.log 2>&1
tail -1 $T/pytest_batching.log
for B in 4 6 8; do
  ASIM_BATCH_MINB=$B timeout 600 python scripts/bench_batching.py --steps 3 --no-cpu-baseline > $T/bench_minb$B.json 2>&1
  python -c "import json;d=json.load(open('$T/bench_minb$B.json'));print($B, d['ms_per_step'], d['value'])"
done
ASIM_BATCH_MINB=8 timeout 600 python -m pytest tests/test_batching.py -m gpu -x -q > $T/pytest_batching_minb8.log 2>&1
tail -1 $T/pytest_batching_minb8.log
