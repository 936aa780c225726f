"""Copies the reference's own golden run records (the outputs its unit tests
left under proj/unit_*_out: snapshot metadata, report.csv, a VTK file) into
tests/golden/reference_records/ so the snapshot/report writers can be pinned
byte-for-byte without /root/reference at test time.  These are data records,
not source.  Run once in the build container:
    python tests/golden/copy_reference_records.py"""
import os
import shutil

SRC = "/root/reference/proj"
DST = os.path.join(os.path.dirname(os.path.abspath(__file__)), "reference_records")
RECORDS = {
    "unit_run_out": ["meta_1.json", "meta_2.json", "report.csv"],
    "unit_snapshot_out": ["meta_7.json"],
    "unit_vtk_out": ["meta_1.json", "report.csv", "snapshot_1.vtk"],
    "unit_det_out1": ["meta_1.json", "meta_2.json", "meta_3.json", "report.csv"],
}
# the CLI smoke-test configurations (proj/tests/data)
DATA = ["hyperelastic_cube_small.json", "bad_poisson.json"]

if __name__ == "__main__":
    for d, files in RECORDS.items():
        os.makedirs(os.path.join(DST, d), exist_ok=True)
        for f in files:
            shutil.copyfile(os.path.join(SRC, d, f), os.path.join(DST, d, f))
            print("copied", d, f)
    os.makedirs(os.path.join(DST, "data"), exist_ok=True)
    for f in DATA:
        shutil.copyfile(os.path.join(SRC, "tests", "data", f), os.path.join(DST, "data", f))
        print("copied data", f)
