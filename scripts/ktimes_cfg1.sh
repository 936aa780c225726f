FM_CG_GRAPH=0 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt_cfg1.csv python scripts/cfg1_short.py 1 > /dev/null 2>&1
python3 - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/kt_cfg1.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")))
tot = sum(sum(x) for x in d.values())
print(f"total {tot/1e6:.2f} ms")
for k, x in sorted(d.items(), key=lambda kv: -sum(kv[1]))[:14]:
    print(f"   {k:50s} n={len(x):5d} avg={sum(x)/len(x)/1e3:9.3f} us  sum={sum(x)/1e6:8.3f} ms")
PY
