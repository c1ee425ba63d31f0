# End-of-round evidence: smoke, GPU suite, headline bench + reference arm, other configs, batching.
cd $GRAFT_REPO_ROOT
T=gpurun_out/r1final
mkdir -p $T
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $T/gpu.txt 2>&1
python -c "import __graft_entry__ as g; g.smoke()" > $T/smoke.log 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $T/pytest_gpu.log 2>&1
tail -1 $T/pytest_gpu.log; tail -1 $T/smoke.log
timeout 1200 python bench.py > $T/bench.json 2> $T/bench.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $T/bench_reference.json 2> $T/bench_reference.err
for C in S1 S2 motivating; do
  timeout 900 python bench.py --config $C --no-cpu-baseline > $T/bench_$C.json 2> $T/bench_$C.err
done
timeout 900 python bench.py --config S4 --hours 24 --no-cpu-baseline > $T/bench_S4.json 2> $T/bench_S4.err
timeout 900 python scripts/bench_batching.py > $T/bench_batching.json 2> $T/bench_batching.err
for f in $T/bench*.json; do python -c "import json,sys;d=json.loads(open('$f').read().strip().splitlines()[-1]);print('$f', d.get('value'), d.get('ms_per_step'), (d.get('roofline') or {}).get('frac'))"; done
