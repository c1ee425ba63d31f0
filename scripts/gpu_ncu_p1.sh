# ncu --set full + source lines of one mid-search pass-1 launch (u32 SPEC) of the day-long S3 search (split off).
mkdir -p gpurun_out/ncu_p1b
ASIM_SPLIT=0 timeout 1500 ncu --set full --import-source on --clock-control none --kernel-name-base mangled \
  -k regex:chunk_kernelIjLi0 -s ${1:-70} -c 1 -o gpurun_out/ncu_p1b/full \
  python scripts/search_profile.py 24 --reps 1 > gpurun_out/ncu_p1b/full.log 2>&1
ls -la gpurun_out/ncu_p1b
