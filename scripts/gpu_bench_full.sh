# Full benchmark + ncu evidence (run under gpurun). Usage: bash scripts/gpu_bench_full.sh <tag>
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}
mkdir -p gpurun_out/$TAG
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/$TAG/gpu.txt 2>&1
timeout 1200 python bench.py > gpurun_out/$TAG/bench.json 2> gpurun_out/$TAG/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > gpurun_out/$TAG/bench_reference.json 2> gpurun_out/$TAG/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/$TAG/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/launches_bench.json 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:coop_walk_kernel -s 151 -c 1 \
  -o gpurun_out/$TAG/walk python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:chunk_kernel -s 151 -c 2 \
  -o gpurun_out/$TAG/chunk python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > /dev/null 2>&1
ls -la gpurun_out/$TAG
