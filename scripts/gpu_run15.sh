cd $GRAFT_REPO_ROOT
mkdir -p gpurun_out/r15
ASIM_WALK_LOG=30000000 timeout 300 python scripts/walk_profile.py 1 4096 > gpurun_out/r15/walk_log.txt 2>&1
ASIM_SCALAR_WALK=0 ASIM_WALK_LOG=30000000 timeout 300 python scripts/walk_profile.py 1 4096 > gpurun_out/r15/walk_log_noscalar.txt 2>&1
