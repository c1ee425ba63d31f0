# ncu evidence for the dominant kernel (run under gpurun, one GPU).
# usage: bash scripts/profile.sh <tag> [bench args...]
set -x
cd $GRAFT_REPO_ROOT
TAG=${1:-r1}; shift
ARGS=${@:---config S3 --hours 0.25}
mkdir -p gpurun_out/$TAG
# 1) launch list of one search (device time per launch, cold-cache, serialised)
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv \
  --log-file gpurun_out/$TAG/launches.csv \
  python bench.py $ARGS --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/$TAG/launches_bench.txt 2>&1
# 2) full section set on a few chunk_kernel launches
timeout 1500 ncu --set full --clock-control none --import-source on -k regex:chunk_kernel -s 4 -c 3 \
  -o gpurun_out/$TAG/prof python bench.py $ARGS --steps 1 --warmup 0 --no-e2e --no-cpu-baseline \
  > gpurun_out/$TAG/prof_bench.txt 2>&1
ls -la gpurun_out/$TAG
