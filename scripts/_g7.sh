bash scripts/ncu_heaviest.sh 'lane_walk_kernel' gpurun_out/ncu_lw_1h python scripts/search_profile.py 1 --reps 1
cat gpurun_out/ncu_lw_1h/heaviest.txt
python3 - <<'PY'
import csv
rows = [r for r in csv.reader(open('gpurun_out/ncu_lw_1h/list.csv')) if len(r) > 14 and r[0].isdigit()]
print(len(rows))
import collections
c=collections.Counter(); t=collections.Counter()
for r in rows:
    c[r[4][:60]]+=1; t[r[4][:60]]+=float(r[14].replace(',',''))
for k in c: print(k, c[k], t[k])
PY
