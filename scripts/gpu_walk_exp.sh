# Walker routing experiment on the day-long S3 search (split off): correctness with the
# shared-memory walker forced on, then search profiles per routing.
set -x
ASIM_SMEM_WALK=1 ASIM_SMEM_WALK_COOP=1 python -m pytest tests/test_chunked.py tests/test_search_parity.py tests/test_determinism.py tests/test_shard_emulation.py -m gpu -x -q > gpurun_out/pytest_smemwalk.log 2>&1; echo pytest rc=$?
tail -2 gpurun_out/pytest_smemwalk.log
for cfg in "0 0" "4 0" "8 0" "1 1" "0 1"; do
  set -- $cfg
  ASIM_SPLIT=0 ASIM_SMEM_WALK=$1 ASIM_SMEM_WALK_COOP=$2 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_walk_$1_$2.txt 2>&1
  tail -1 gpurun_out/prof_walk_$1_$2.txt | python3 -c "import json,sys; d=json.loads(sys.stdin.read()); print('$1 $2', {k: round(d[k]) for k in ('search_ms','sim_ms','spec_busy_ms','pass2_busy_ms','walk_busy_ms')}, d['best_good'])"
done
