"""DRAM traffic per voxel of each matvec pass from `ncu --set full` captures,
for bench.py's roofline.traffic (which checks the recorded kernel names
against the kernels it launched).  Usage:
  python scripts/ncu_traffic.py N report.ncu-rep|raw.csv [...] > profiles/r2_traffic_<N>.json"""
import csv
import io
import json
import re
import subprocess
import sys

PASS_OF = [  # (regex on the kernel name, pass key of bench.py)
    (r"k_zf_pipe<\d+, 2, 0", "z_fwd_svk"), (r"k_zf_fast<\d+, 2, 0", "z_fwd_svk"),
    (r"k_zf_fast<\d+, 1, 0", "z_fwd_k4"), (r"k_y_fast<\d+, \d+, \(int\)-1", "y_fwd"),
    (r"k_y_fast<\d+, \d+, 1[,>]", "y_inv"), (r"k_x_(fast|stream|direct)", "x_ghat"), (r"k_zi_(fast|reg)", "z_inv"),
]


def main():
    N = int(sys.argv[1])
    n = N ** 3
    out = {"grid": N, "unit": "DRAM bytes per voxel (dram__bytes_read.sum + dram__bytes_write.sum)",
           "source": [r.split("/")[-1] for r in sys.argv[2:]], "passes": {}, "kernels": {}}
    for rep in sys.argv[2:]:
        if rep.endswith(".csv"):
            txt = open(rep).read()
        else:
            txt = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
        rows = list(csv.reader(io.StringIO(txt)))
        h, units = rows[0], rows[1]
        ki, ri, wi = h.index("Kernel Name"), h.index("dram__bytes_read.sum"), h.index("dram__bytes_write.sum")
        scale = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
        for r in rows[2:]:
            for pat, key in PASS_OF:
                if re.search(pat, r[ki]):
                    b = float(r[ri]) * scale[units[ri]] + float(r[wi]) * scale[units[wi]]
                    out["passes"].setdefault(key, round(b / n, 2))
                    out["kernels"].setdefault(key, r[ki])
                    break
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
