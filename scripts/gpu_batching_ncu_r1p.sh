# ncu full set of one batching_kernel launch (the bench command, one step).
cd $GRAFT_REPO_ROOT
T=gpurun_out/r1p
mkdir -p $T
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:batching_kernel -c 1 \
  -o $T/batching python scripts/bench_batching.py --steps 1 --warmup 0 --no-cpu-baseline > $T/ncu_full.log 2>&1
tail -3 $T/ncu_full.log
ls -la $T
