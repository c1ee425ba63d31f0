cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_chunked.py tests/test_fast_heuristic.py tests/test_search_parity.py -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu12a.txt
timeout 600 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --search fast --no-cpu-baseline --no-e2e > gpurun_out/bench12_fast.txt 2>&1
timeout 600 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench12_greedy.txt 2>&1
ASIM_SCALAR_WALK=0 timeout 600 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench12_greedy_coop.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x 2>&1 | tail -30 > gpurun_out/pytest_gpu12.txt
