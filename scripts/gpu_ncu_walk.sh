# Launch list of the scalar/group-lane walker kernel over the day-long S3 search, then ncu --set full of its heaviest launch.
bash scripts/ncu_heaviest.sh coop_walk_kernelIjLb1 gpurun_out/ncu_walk python scripts/search_profile.py 24 --reps 1
cat gpurun_out/ncu_walk/heaviest.txt; ls -la gpurun_out/ncu_walk
