set -x
cd $GRAFT_REPO_ROOT
nvidia-smi -L
python -c "import torch;print(torch.cuda.get_device_name(), torch.cuda.get_device_properties(0).multi_processor_count)"
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -40 > gpurun_out/pytest_gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --config S1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_s1.txt 2>&1
timeout 600 python bench.py --config S4 --hours 24 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_s4.txt 2>&1
timeout 900 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e > gpurun_out/bench_s3.txt 2>&1
timeout 900 python bench.py --config S3 --hours 1 --steps 1 --warmup 1 --no-cpu-baseline --no-e2e --dedup > gpurun_out/bench_s3_dedup.txt 2>&1
ls gpurun_out
