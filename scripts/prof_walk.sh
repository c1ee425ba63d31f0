cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/walk
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:walk_kernel -s 5 -c 1 \
  -o gpurun_out/walk/walk python bench.py --config S3 --hours 0.25 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/walk/log.txt 2>&1
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:chunk_kernel -s 8 -c 1 \
  -o gpurun_out/walk/spec python bench.py --config S3 --hours 0.25 --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/walk/log2.txt 2>&1
