cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r20
timeout 1500 python -m pytest tests -m gpu -q -x > gpurun_out/r20/pytest_gpu.txt 2>&1
timeout 600 python bench.py --no-cpu-baseline --no-e2e > gpurun_out/r20/bench.json 2> gpurun_out/r20/bench.err
bash scripts/ncu_heaviest.sh chunk_kernelIjLi0E gpurun_out/r20/spec python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu-baseline
