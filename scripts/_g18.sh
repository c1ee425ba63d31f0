bash scripts/ncu_heaviest.sh 'coop_walk_kernelIjLb1' gpurun_out/ncu_walk_scalar_day python scripts/search_profile.py 24 --reps 1
cat gpurun_out/ncu_walk_scalar_day/heaviest.txt
python scripts/ncu_lines.py gpurun_out/ncu_walk_scalar_day/full.ncu-rep 40 > gpurun_out/ncu_walk_scalar_day/lines.md 2>&1
head -30 gpurun_out/ncu_walk_scalar_day/lines.md
