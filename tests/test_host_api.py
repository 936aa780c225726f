"""The drop-in C++ API (paper_1603_08893_b200/host): reference-style client
code compiled against `namespace fftmech` and linked to the CUDA library."""
import os
import subprocess

import pytest

LIB = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_1603_08893_b200", "lib")
BIN = os.path.join(LIB, "test_host_api")
RECORDS = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_records")


def test_host_library_links_the_cuda_library():
    assert os.path.exists(os.path.join(LIB, "libfftmech_host.so")) and os.path.exists(BIN)
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libfftmech_host.so" in out and "libfftmech_b200.so" in out
    syms = subprocess.run(["nm", "-DC", "--defined-only", os.path.join(LIB, "libfftmech_host.so")],
                          capture_output=True, text=True).stdout
    for name in ["fftmech::build_projection", "fftmech::apply_projection", "fftmech::apply_projected_tangent",
                 "fftmech::cg_solve", "fftmech::solve_increment", "fftmech::run_program",
                 "fftmech::HyperelasticModel::evaluate", "fftmech::SimoPlasticityModel::evaluate",
                 "fftmech::make_cubic_inclusion", "fftmech::bind_parameters"]:
        assert name in syms, name


@pytest.mark.gpu
def test_reference_style_cpp_client_passes_on_gpu():
    r = subprocess.run([BIN, RECORDS], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "[FAIL]" not in r.stdout


def test_native_config4_stream_matches_mt19937_64():
    """The host library's std::mt19937_64 filler (large config-4 inputs) and
    the numpy restatement produce the identical stream."""
    import numpy as np
    from paper_1603_08893_b200 import microstructure as M
    pts = (64, 64, 64)
    a = M.uniform_field(pts, 9, seed=4 + 64)  # >= 2^20 entries: native path
    b = 2.0 * M.MT19937_64(4 + 64).uniform(9 * 64 ** 3) - 1.0
    assert M._host_lib() is not None
    assert np.array_equal(a, b)


def test_snapshot_writer_matches_reference_record_on_host():
    """write_snapshot/read_snapshot round trip (test_config_io.cpp:135-164);
    the emitted meta_7.json is byte-identical to proj/unit_snapshot_out's."""
    r = subprocess.run([BIN, RECORDS, "--no-device"], capture_output=True, text=True, timeout=120)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
