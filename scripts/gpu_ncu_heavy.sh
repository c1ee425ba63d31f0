# Launch list of the day-long S3 search's pass-1 launches (split off), then ncu --set full of the heaviest.
ASIM_SPLIT=0 bash scripts/ncu_heaviest.sh chunk_kernelIjLi0 gpurun_out/ncu_heavy python scripts/search_profile.py 24 --reps 1
cat gpurun_out/ncu_heavy/heaviest.txt; ls -la gpurun_out/ncu_heavy
