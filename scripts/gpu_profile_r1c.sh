# Round-1 evidence set (under gpurun): tests, bench lines, launch list, ncu captures.
cd $GRAFT_REPO_ROOT
O=gpurun_out/r1c
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > $O/gpu.txt 2>&1
echo "host cores: $(nproc)" >> $O/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q > $O/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.txt 2>&1
timeout 900 python bench.py > $O/bench_S3_1h.json 2> $O/bench_S3_1h.err
timeout 900 python bench.py --impl reference --steps 2 --warmup 1 > $O/bench_reference_S3_1h.json 2> $O/bench_reference.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $O/launches_S3_1h.csv \
  python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline > $O/launches_bench.json 2>&1
bash scripts/ncu_heaviest.sh chunk_kernelIjLi0E $O/spec python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline
bash scripts/ncu_heaviest.sh chunk_kernelIjLi1E $O/dual python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline
timeout 1500 python bench.py --hours 24 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > $O/bench_S3_day.json 2> $O/bench_S3_day.err
rm -f $O/*/list.log
ls -la $O
