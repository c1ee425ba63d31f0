cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r13
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv > gpurun_out/r13/gpu.txt 2>&1
nproc >> gpurun_out/r13/gpu.txt
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r13/pytest_gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r13/smoke.txt 2>&1
timeout 900 python bench.py > gpurun_out/r13/bench.json 2> gpurun_out/r13/bench.err
ASIM_SCALAR_WALK=0 timeout 600 python bench.py --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/r13/bench_coop.json 2>&1
timeout 600 python bench.py --search fast --steps 3 --warmup 3 --no-cpu-baseline --no-e2e > gpurun_out/r13/bench_fast.json 2>&1
ls -la gpurun_out/r13
