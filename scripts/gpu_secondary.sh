# Secondary bench lines at HEAD: the 1-h opening of the S3 search and the section-5.4 batching evaluator.
set -x
mkdir -p gpurun_out/final2
python bench.py --hours 1 --steps 5 --warmup 3 > gpurun_out/final2/bench_S3_1h.json 2> gpurun_out/final2/bench_S3_1h.err; echo rc=$?
python scripts/bench_batching.py > gpurun_out/final2/bench_batching.json 2> gpurun_out/final2/bench_batching.err; echo rc=$?
cut -c1-300 gpurun_out/final2/bench_S3_1h.json; cut -c1-300 gpurun_out/final2/bench_batching.json
