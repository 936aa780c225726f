"""`fftmech` CLI (paper_1603_08893_b200/host/tools/fftmech.cpp), the
reference's ctest smoke tests (proj/tests/CMakeLists.txt:5-18) plus a
config-driven run compared with the reference's own run record."""
import json
import os
import subprocess

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
BIN = os.path.join(ROOT, "paper_1603_08893_b200", "lib", "fftmech")
DATA = os.path.join(ROOT, "tests", "golden", "reference_records", "data")
RECORDS = os.path.join(ROOT, "tests", "golden", "reference_records")


def cli(*args, timeout=600):
    return subprocess.run([BIN, *args], capture_output=True, text=True, timeout=timeout)


def test_validate_good_config():
    r = cli("validate", os.path.join(DATA, "hyperelastic_cube_small.json"))
    assert r.returncode == 0 and "configuration OK" in r.stdout, r.stderr


def test_validate_bad_config_reports_path_and_exit_code():
    r = cli("validate", os.path.join(DATA, "bad_poisson.json"))
    assert r.returncode == 2
    assert "config error: model.phases[0].poisson" in r.stderr, r.stderr


def test_set_overrides_take_precedence():
    good = os.path.join(DATA, "hyperelastic_cube_small.json")
    r = cli("validate", good, "--set", "loading.increments=0", "--set", "solver.eta_cg=2")
    assert r.returncode == 2
    assert "loading.increments" in r.stderr and "solver.eta_cg" in r.stderr, r.stderr
    assert cli("validate", good, "--set", "solver.nyquist=identity_equilibrium").returncode == 0
    assert cli("validate", good, "--set", "bogus").returncode == 2


def test_run_section_places_the_gpu_run():
    """device selection and the slab-rank count are config keys
    (`run` section) with command-line shorthands."""
    good = os.path.join(DATA, "hyperelastic_cube_small.json")
    assert cli("validate", good, "--set", "run.device=0", "--set", "run.ranks=2",
               "--set", "run.transpose=nccl").returncode == 0
    assert cli("validate", good, "--device", "1", "--ranks", "4", "--transpose", "peer").returncode == 0
    r = cli("validate", good, "--device", "-1", "--ranks", "0", "--transpose", "mpi")
    assert r.returncode == 2
    for key in ("run.device", "run.ranks", "run.transpose"):
        assert f"config error: {key}" in r.stderr, r.stderr


def test_usage_and_missing_file():
    assert cli("frobnicate", "x").returncode == 1
    r = cli("validate", "/nonexistent/config.json")
    assert r.returncode == 4 and "i/o error" in r.stderr


@pytest.mark.gpu
def test_run_then_info(tmp_path):
    out = tmp_path / "cli_run_small_out"
    r = cli("run", os.path.join(DATA, "hyperelastic_cube_small.json"), "--set", f"output.directory={out}")
    assert r.returncode == 0, r.stdout + r.stderr
    assert (out / "report.csv").exists() and (out / "meta_1.json").exists()
    i = cli("info", str(out))
    assert i.returncode == 0 and "1 snapshot(s)" in i.stdout and "fields F P eq" in i.stdout, i.stdout


@pytest.mark.gpu
@pytest.mark.parametrize("transpose", ["peer", "nccl"])
def test_slab_run_from_the_cli_matches_single_rank(tmp_path, transpose):
    """`fftmech run --ranks 2`: the slab-decomposed kernels (two ranks emulated
    on the device, either transpose arm) write the same converged field and
    the same Newton / CG record as the plain run."""
    import numpy as np
    cfg = {"grid": {"points": [8, 8, 8]}, "microstructure": {"kind": "cube", "volume_fraction": 0.125},
           "model": {"kind": "hyperelastic", "phases": [{"youngs": 1.0, "poisson": 0.3},
                                                       {"youngs": 10.0, "poisson": 0.3}]},
           "loading": {"mode": "simple_shear", "gamma": 0.1, "increments": 1}}
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    outs = []
    for name, extra in (("plain", []), ("slab", ["--device", "0", "--ranks", "2", "--transpose", transpose])):
        out = tmp_path / name
        r = cli("run", str(p), "--set", f"output.directory={out}", *extra)
        assert r.returncode == 0, r.stdout + r.stderr
        outs.append((np.fromfile(out / "F_1.bin", dtype="<f8"), (out / "report.csv").read_text().splitlines()))
    (F1, rep1), (F2, rep2) = outs
    assert np.max(np.abs(F1 - F2)) < 1e-12
    # same Newton and CG counts; the residual is a reduction in another order
    assert [l.split(",")[:3] for l in rep1] == [l.split(",")[:3] for l in rep2]
    assert abs(float(rep1[1].split(",")[3]) - float(rep2[1].split(",")[3])) < 1e-6 * float(rep1[1].split(",")[3])


@pytest.mark.gpu
def test_config_run_reproduces_reference_record(tmp_path):
    """test_config_io.cpp:166-200's configuration through `fftmech run`:
    snapshot metadata byte-identical to proj/unit_run_out, the converged field
    equal to Fbar (homogeneous cell), report rows as recorded."""
    out = tmp_path / "unit_run_out"
    cfg = {"grid": {"points": [4, 4]}, "microstructure": {"kind": "laminate", "fractions": [1.0]},
           "model": {"kind": "hyperelastic", "phases": [{"youngs": 1.0, "poisson": 0.3}]},
           "loading": {"mode": "simple_shear", "gamma": 0.2, "increments": 2},
           "output": {"directory": str(out)}}
    p = tmp_path / "cfg.json"
    p.write_text(json.dumps(cfg))
    r = cli("run", str(p))
    assert r.returncode == 0, r.stdout + r.stderr
    for f in ("meta_1.json", "meta_2.json"):
        assert (out / f).read_bytes() == open(os.path.join(RECORDS, "unit_run_out", f), "rb").read(), f
    import numpy as np
    F = np.fromfile(out / "F_2.bin", dtype="<f8").reshape(4, 16)
    assert np.max(np.abs(F[1] - 0.2)) < 1e-12 and np.max(np.abs(F[0] - 1.0)) < 1e-12
    got = [line.split(",") for line in (out / "report.csv").read_text().splitlines()]
    want = [line.split(",") for line in open(os.path.join(RECORDS, "unit_run_out", "report.csv")).read().splitlines()]
    assert got[0] == want[0] and len(got) == len(want) == 3
    for g, w in zip(got[1:], want[1:]):
        assert g[:4] == w[:4] and abs(float(g[5]) - float(w[5])) <= 1e-14 * float(w[5])
    i = cli("info", str(out))
    assert i.returncode == 0 and "2 snapshot(s)" in i.stdout
