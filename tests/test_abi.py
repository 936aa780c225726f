"""CPU-side checks of the drop-in boundary: libfftmech_b200.so loads without a
GPU, exports every entry point include/fftmech_b200.h declares, and the host
setup helpers reproduce the reference's microstructure semantics."""
import ctypes
import subprocess

import numpy as np
import pytest

from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M


def test_library_exports_every_declared_symbol():
    L = abi.lib()
    declared = abi.declared_symbols()
    assert len(declared) >= 35
    missing = [s for s in declared if not hasattr(L, s)]
    assert not missing, missing
    # and nm agrees that they are real dynamic exports
    out = subprocess.run(["nm", "-D", "--defined-only", abi.LIB_PATH], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if " T " in line}
    assert set(declared) <= exported


def test_library_is_sm100a():
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", abi.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out


def test_every_declared_symbol_is_bound():
    assert set(abi.declared_symbols()) == set(abi._SIGS)


def test_invalid_grid_is_rejected_without_touching_the_device():
    L = abi.lib()
    h = ctypes.c_void_p()
    pts = (ctypes.c_int32 * 3)(4, 4, 4)
    ln = (ctypes.c_double * 3)(1, 1, 1)
    assert L.fm_ctx_create(4, pts, ln, 3, 0, 0, ctypes.byref(h)) == 1  # dim 4
    assert L.fm_ctx_create(3, pts, ln, 2, 0, 0, ctypes.byref(h)) == 1  # tdim < dim
    bad = (ctypes.c_int32 * 3)(4, 0, 4)
    assert L.fm_ctx_create(3, bad, ln, 3, 0, 0, ctypes.byref(h)) == 1
    assert L.fm_ctx_create(3, pts, ln, 3, 2, 0, ctypes.byref(h)) == 1  # nyquist mode


def test_cubic_inclusion_matches_reference_rounding():
    # microstructure.cpp:19-49: side = lround(f^(1/d) N), start = (N - side)/2
    pg = M.make_cubic_inclusion((5, 5, 5), (2.0 / 5.0) ** 3)
    lab = pg.labels.reshape(5, 5, 5)
    assert lab.sum() == 8 and lab[1:3, 1:3, 1:3].all()
    pg = M.make_cubic_inclusion((11, 11, 11), (3.0 / 11.0) ** 3)
    assert pg.labels.reshape(11, 11, 11)[4:7, 4:7, 4:7].all() and pg.labels.sum() == 27
    with pytest.raises(ValueError):
        M.make_cubic_inclusion((3, 3, 3), 0.99)


def test_laminate_largest_remainder():
    pg = M.make_laminate((5, 4), [0.4, 0.6])
    assert list(pg.labels.reshape(5, 4)[:, 0]) == [0, 0, 1, 1, 1]
    pg = M.make_laminate((7, 2), [0.5, 0.5])
    assert pg.labels.reshape(7, 2)[:, 0].sum() in (3, 4)


def test_config_generators():
    pg = M.corner_cube((31, 31, 31), 9)
    assert pg.labels.sum() == 729 and pg.labels[0] == 1
    b = M.bernoulli((16, 16, 16), 0.3, seed=2)
    assert 0.25 < b.labels.mean() < 0.35
    b2 = M.bernoulli((16, 16, 16), 0.3, seed=2)
    assert np.array_equal(b.labels, b2.labels)
    s, frac, count = M.random_spheres(64, 6, 0.25, seed=3)
    assert frac >= 0.25 and count > 0
    u = M.uniform_field((4, 4, 4), 9, seed=4)
    assert u.shape == (576,) and np.all(np.abs(u) <= 1.0)


def test_bind_parameters_uses_youngs_poisson():
    pg = M.corner_cube((4, 4, 4), 2)
    lam, mu, ty, h = M.bind_parameters(pg, [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
                                            M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)])
    assert mu[0] == pytest.approx(2.0 / 2.6) and mu[-1] == pytest.approx(1.0 / 2.6)
    assert lam[-1] == pytest.approx(0.3 / (1.3 * 0.4))
    assert ty[0] == 0.006 and h[-1] == 0.003
