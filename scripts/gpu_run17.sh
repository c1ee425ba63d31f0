cd $GRAFT_REPO_ROOT
bash scripts/ncu_heaviest.sh coop_walk_kernelIjLb1E gpurun_out/r17s python scripts/walk_profile.py 1 4096
