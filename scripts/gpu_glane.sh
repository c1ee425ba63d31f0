# Group-lane walker: correctness with it forced on, warp-primitive latencies, and search profiles per threshold.
set -x
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/warp_latency scripts/micro/warp_latency.cu && /tmp/warp_latency | tee gpurun_out/warp_latency.txt
ASIM_GLANE_WALK=1 python -m pytest tests/test_chunked.py tests/test_search_parity.py tests/test_determinism.py tests/test_shard_emulation.py tests/test_fullsize_search.py -m gpu -x -q > gpurun_out/pytest_glane.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_glane.log
for gw in 0 2 4 8; do
  ASIM_SPLIT=0 ASIM_GLANE_WALK=$gw python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_glane_$gw.txt 2>&1
  tail -1 gpurun_out/prof_glane_$gw.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('glane $gw', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done
