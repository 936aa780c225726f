"""Stall samples of an ncu source page (SASS) CSV grouped by opcode, with the
dominant stall reason of each group, plus how many executed instructions the
group holds: python scripts/ncu_stalls_by_op.py <page-source.csv> [skip-regex]"""
import csv
import re
import sys
from collections import Counter, defaultdict

rows = list(csv.reader(open(sys.argv[1])))
end = next((k for k in range(2, len(rows)) if rows[k] and rows[k][0] == "Kernel Name"), len(rows))
h, data = rows[1], rows[2:end]
skip = re.compile(sys.argv[2]) if len(sys.argv) > 2 else None
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
idx = {c: h.index(c) for c in cols}
iS, iSrc = h.index("Warp Stall Sampling (All Samples)"), h.index("Source")
iEx = h.index("Instructions Executed") if "Instructions Executed" in h else None
f = lambda r, i: float(r[i] or 0)  # noqa: E731
samples, execd, reasons = Counter(), Counter(), defaultdict(Counter)
for r in data:
    src = r[iSrc].strip()
    op = src.split()[1] if src.startswith("@") and len(src.split()) > 1 else src.split()[0] if src else "?"
    op = op.split(".")[0]
    if skip and skip.search(src):
        op = "(skipped)"
    samples[op] += f(r, iS)
    if iEx is not None:
        execd[op] += f(r, iEx)
    for c, i in idx.items():
        reasons[op][c[6:]] += f(r, i)
tot = sum(samples.values())
te = sum(execd.values()) or 1
print(f"{'op':10s} {'samples%':>8s} {'exec%':>6s}  top reasons")
for op, s in samples.most_common(24):
    rs = [(k, round(v / max(s, 1) * 100)) for k, v in reasons[op].most_common(3)]
    print(f"{op:10s} {s / tot * 100:8.1f} {execd[op] / te * 100:6.1f}  {rs}")
