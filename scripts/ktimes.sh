# per-kernel launch times (ncu, cold-cache, serialised) of a 256^3 MF matvec run under each env setting
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '__')
  env $v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kt_$name.csv python scripts/prof_matvec.py ${KT_N:-256} 3 mf > /dev/null 2>&1
  python3 - "$v" "$name" <<'PY'
import csv, sys, collections
v = sys.argv[1]
rows = [r for r in csv.reader(open(f"gpurun_out/kt_{sys.argv[2]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][:40]].append(float(r[vi].replace(",", "")))
print(v, " | ".join(f"{k}: {sum(x)/len(x)/1e3:.3f} ms x{len(x)}" for k, x in d.items()))
PY
done
