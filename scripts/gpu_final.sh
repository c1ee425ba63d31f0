# Round-end evidence: GPU suite, smoke, the default bench line, the launch list of one bench
# search under ncu (cold-cache, serialised), and ncu --set full of the heaviest pass-1 launch.
set -x
mkdir -p gpurun_out/final
python -m pytest tests -m gpu -q > gpurun_out/final/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/final/pytest_gpu.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/final/smoke.log 2>&1; echo smoke rc=$?; tail -1 gpurun_out/final/smoke.log
python bench.py > gpurun_out/final/bench.json 2> gpurun_out/final/bench.err; echo bench rc=$?
python3 -c "import json; d=json.load(open('gpurun_out/final/bench.json')); print(d['ms_per_step'], d['value'], d['roofline']['frac'], d['e2e']['ms_per_step'], d['cpu_baseline']['value'])"
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/final/launches.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > gpurun_out/final/launches_bench.txt 2>&1; echo ncu list rc=$?
bash scripts/ncu_heaviest.sh chunk_kernelIjLi0 gpurun_out/final/ncu_p1 python scripts/search_profile.py 24 --reps 1
cat gpurun_out/final/ncu_p1/heaviest.txt
