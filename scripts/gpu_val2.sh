set -x
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
for sp in 0 1; do
  ASIM_SPLIT=$sp python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/bench_split$sp.json 2> gpurun_out/bench_split$sp.err
  python3 -c "import json; d=json.load(open('gpurun_out/bench_split$sp.json')); print('split $sp', d['ms_per_step'], d['value'], d['roofline']['frac'])"
done
