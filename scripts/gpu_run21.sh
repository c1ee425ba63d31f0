cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r21
timeout 1200 python bench.py --hours 24 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r21/bench_day.json 2> gpurun_out/r21/bench_day.err
timeout 900 python bench.py --config S2 --hours 24 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r21/bench_s2_day.json 2> gpurun_out/r21/bench_s2_day.err
timeout 600 python bench.py --config S1 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r21/bench_s1.json 2> gpurun_out/r21/bench_s1.err
timeout 600 python bench.py --config S4 --hours 24 --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r21/bench_s4.json 2> gpurun_out/r21/bench_s4.err
