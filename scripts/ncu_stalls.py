"""Stall-reason attribution from an ncu source page (SASS) CSV:
python scripts/ncu_stalls.py <page-source.csv> [top]"""
import csv
import sys
from collections import Counter

rows = list(csv.reader(open(sys.argv[1])))
# one section per kernel ("Kernel Name" row, header row, data rows): the first
end = next((k for k in range(2, len(rows)) if rows[k] and rows[k][0] == "Kernel Name"), len(rows))
print(rows[0][1][:100])
h, data = rows[1], rows[2:end]
top = int(sys.argv[2]) if len(sys.argv) > 2 else 25
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}
iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
f = lambda r, i: float(r[i] or 0)  # noqa: E731
tot = sum(f(r, iS) for r in data)
agg = Counter({c: sum(f(r, i) for r in data) for c, i in idx.items()})
print("by reason:", [(c[6:], round(v / tot * 100, 1)) for c, v in agg.most_common(8)])
for r in sorted(data, key=lambda r: -f(r, iS))[:top]:
    rs = sorted(((f(r, i), c[6:]) for c, i in idx.items()), reverse=True)[:2]
    print(f"{f(r, iS) / tot * 100:5.1f}% {r[0][-5:]} {r[iSrc][:60]:60s} {rs}")
