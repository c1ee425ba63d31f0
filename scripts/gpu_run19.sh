cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r19
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r19/launches.csv python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/r19/launches_bench.json 2>&1
timeout 300 python scripts/walk_profile.py 1 4096 v > gpurun_out/r19/walk.txt 2>&1
