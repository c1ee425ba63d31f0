cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/walk2
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:coop_walk_kernel -s 121 -c 1 \
  -o gpurun_out/walk2/walk python bench.py --config S3 --hours 0.25 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/walk2/log.txt 2>&1
