"""Summarise an ncu report (--set full) and a launch-list CSV into markdown.
Usage: python scripts/ncu_summary.py <report.ncu-rep> [launches.csv] > out.md"""
import csv
import io
import subprocess
import sys

METRICS = [
    ("gpu__time_duration.sum", "time"),
    ("dram__bytes_read.sum", "DRAM read"),
    ("dram__bytes_write.sum", "DRAM write"),
    ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM %peak"),
    ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
    ("launch__registers_per_thread", "regs"),
    ("launch__occupancy_limit_registers", "occ lim regs"),
    ("launch__occupancy_limit_shared_mem", "occ lim smem"),
    ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem wavefronts"),
    ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smem bank conflicts"),
    ("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "fp64 pipe %"),
]


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    return rows[0], rows[1], rows[2:]


def main():
    rep = sys.argv[1]
    h, units, rows = raw(rep)
    print(f"## ncu --set full: `{rep.split('/')[-1]}`\n")
    print("| kernel | " + " | ".join(n for _, n in METRICS) + " |")
    print("|---|" + "---|" * len(METRICS))
    ki = h.index("Kernel Name")
    for r in rows:
        vals = []
        for m, _ in METRICS:
            if m in h:
                i = h.index(m)
                vals.append(f"{r[i]} {units[i]}".strip())
            else:
                vals.append("n/a")
        print(f"| `{r[ki][:48]}` | " + " | ".join(vals) + " |")
    if len(sys.argv) > 2:
        rows = list(csv.reader(open(sys.argv[2])))
        hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
        hh = rows[hdr]
        ki, vi = hh.index("Kernel Name"), hh.index("Metric Value")
        print(f"\n## launch list (`gpu__time_duration.sum`, ns, cold-cache serialised): `{sys.argv[2].split('/')[-1]}`\n")
        print("| # | kernel | ns |\n|---|---|---|")
        for j, r in enumerate(rows[hdr + 1:]):
            print(f"| {j} | `{r[ki][:60]}` | {r[vi]} |")


if __name__ == "__main__":
    main()
