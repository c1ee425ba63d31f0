set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest rc=$?
tail -3 gpurun_out/pytest_gpu.log
python scripts/search_profile.py 24 --reps 2 > gpurun_out/prof_day.txt 2>&1; tail -1 gpurun_out/prof_day.txt | cut -c1-900
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err; echo bench rc=$?
cat gpurun_out/bench.json | cut -c1-600
