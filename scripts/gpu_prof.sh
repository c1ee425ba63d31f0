# Day-long S3 search diagnostics (split on and off) with per-class pass-1 accounting.
set -x
python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_split.txt 2>&1; tail -1 gpurun_out/prof_day_split.txt | cut -c1-1500
ASIM_SPLIT=0 python scripts/search_profile.py 24 --reps 1 > gpurun_out/prof_day_nosplit.txt 2>&1; tail -1 gpurun_out/prof_day_nosplit.txt | cut -c1-1500
# ncu: one mid-search pass-1 launch (u32 SPEC) of the day search, full set + source lines
mkdir -p gpurun_out/ncu_p1
timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
  -k regex:chunk_kernelIjLi0 -s 150 -c 1 -o gpurun_out/ncu_p1/full \
  python scripts/search_profile.py 24 --reps 1 > gpurun_out/ncu_p1/full.log 2>&1
ls -la gpurun_out/ncu_p1
