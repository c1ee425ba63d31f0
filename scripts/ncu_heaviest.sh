# Usage (under gpurun): bash scripts/ncu_heaviest.sh <mangled-regex> <outdir> <cmd...>
# 1) launch list of the matching kernels, 2) ncu --set full of the longest one.
RX=$1; OUT=$2; shift 2
mkdir -p $OUT
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --kernel-name-base mangled -k regex:$RX --csv --log-file $OUT/list.csv "$@" > $OUT/list.log 2>&1
IDX=$(python3 - "$OUT/list.csv" <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 14 and r[0].isdigit()]
t = [float(r[14].replace(',', '')) for r in rows]
print(max(range(len(t)), key=lambda i: t[i]) if t else 0)
PY
)
echo "heaviest launch index $IDX" > $OUT/heaviest.txt
timeout 1200 ncu --set full --import-source on --clock-control none --kernel-name-base mangled -k regex:$RX -s $IDX -c 1 -o $OUT/full "$@" > $OUT/full.log 2>&1
