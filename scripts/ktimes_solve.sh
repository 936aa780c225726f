# per-kernel launch times (ncu) of a config-2 matrix-free Newton solve at ${KT_N:-128}^3 under each env setting
for v in "$@"; do
  name=$(echo "$v" | tr ' =' '__')
  env $v ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/kts_$name.csv python scripts/solve_cfg2.py ${KT_N:-128} mf > /dev/null 2>&1
  python3 - "$v" "$name" <<'PY'
import csv, sys, collections
rows = [r for r in csv.reader(open(f"gpurun_out/kts_{sys.argv[2]}.csv")) if len(r) > 10]
h = rows[0]; ki = h.index("Kernel Name"); vi = h.index("Metric Value")
d = collections.defaultdict(list)
for r in rows[1:]:
    d[r[ki].split("(")[0][:48]].append(float(r[vi].replace(",", "")))
tot = sum(sum(x) for x in d.values())
print(sys.argv[1], f"total {tot/1e6:.2f} ms")
for k, x in sorted(d.items(), key=lambda kv: -sum(kv[1])):
    print(f"   {k:50s} n={len(x):5d} avg={sum(x)/len(x)/1e3:9.3f} us  sum={sum(x)/1e6:8.3f} ms")
PY
done
