python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
bash tests/sanitize.sh gpurun_out/sanitizer
cat gpurun_out/sanitizer/summary.txt
python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo bench rc=$?
tail -c 3000 gpurun_out/bench_default.json
timeout 1200 python scripts/cpu_baseline.py gpurun_out/cpu_baseline.json > gpurun_out/cpu_baseline.log 2>&1; echo cpu rc=$?
tail -30 gpurun_out/cpu_baseline.log
