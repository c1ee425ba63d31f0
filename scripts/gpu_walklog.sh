# Walk log of the day-long S3 search: a diagnostics build (ASIM_WALK_DIAGNOSTICS) printing every walk
# longer than ASIM_WALK_LOG cycles, step by step.
set -x
python -c "import sys; sys.path.insert(0,'paper_2302_11665_b200'); import build; build.build(force=True, extra=['-DASIM_WALK_DIAGNOSTICS'])" > gpurun_out/build_diag.log 2>&1
ASIM_WALK_LOG=2000000 python scripts/search_profile.py 24 --reps 1 --steps > gpurun_out/walklog_day.txt 2>&1
grep -c "^walk" gpurun_out/walklog_day.txt; gzip -f gpurun_out/walklog_day.txt
