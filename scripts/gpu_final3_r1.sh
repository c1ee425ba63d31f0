# Final check at HEAD: smoke, full GPU suite, headline bench, batching bench.
cd $GRAFT_REPO_ROOT
T=gpurun_out/r1final3
mkdir -p $T
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $T/pytest_gpu.log 2>&1
tail -1 $T/pytest_gpu.log; tail -1 $T/smoke.log
timeout 1200 python bench.py > $T/bench.json 2> $T/bench.err
timeout 900 python scripts/bench_batching.py > $T/bench_batching.json 2> $T/bench_batching.err
for f in $T/bench.json $T/bench_batching.json; do python -c "import json;d=json.load(open('$f'));print('$f', d['value'], d['ms_per_step'], d['roofline']['frac'], d['e2e']['value'])"; done
