"""Debug-mode equivalent of the reference's imaginary-residue check
(projection.cpp:157-169, ComplexResidue): with the half spectrum the residue a
c2c inverse transform would show lives on the self-conjugate kz planes; the
check measures it before the c2r pass.  Real inputs give round-off; a
deliberate Hermitian violation (test hook) raises FM_E_COMPLEX_RESIDUE."""
import os
import subprocess
import sys

import numpy as np
import pytest

from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.mark.parametrize("pts,mode", [((64, 64, 64), 0), ((12, 10, 14), 0), ((16, 16, 16), 1), ((9, 7, 5), 0),
                                       ((256, 32, 32), 0)])
def test_residue_of_real_input_is_roundoff(pts, mode):
    A = M.uniform_field(pts, 9, seed=11)
    rng = np.random.default_rng(4)
    K = rng.uniform(-1, 1, 81 * int(np.prod(pts)))
    with abi.Context(pts, 3, nyquist_mode=mode) as ctx:
        ctx.set_debug(True)
        fa = ctx.field(9, A)
        ctx.projection(fa)
        info = ctx.last_info()
        assert info["status"] == 0 and 0.0 <= info["value"] <= 1e-13 * np.linalg.norm(A), info
        ctx.projected_tangent(ctx.field(81, K), fa)  # the fused operator form is checked too
        assert ctx.last_info()["status"] == 0
        ctx.set_virtual_ranks(2) if pts[0] % 2 == 0 and pts[1] % 2 == 0 else None
        ctx.projection(fa)
        assert ctx.last_info()["value"] <= 1e-13 * np.linalg.norm(A)


def test_hermitian_violation_raises_complex_residue():
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from paper_1603_08893_b200 import abi, microstructure as M\n"
        "pts = (32, 32, 32)\n"
        "A = M.uniform_field(pts, 9, seed=11)\n"
        "with abi.Context(pts, 3) as ctx:\n"
        "    try:\n"
        "        ctx.projection(ctx.field(9, A))\n"
        "        print('NO ERROR')\n"
        "    except abi.FmError as e:\n"
        "        print('STATUS', e.status, e.info['value'])\n" % ROOT)
    env = dict(os.environ, FM_DEBUG_RESIDUE="1", FM_DEBUG_RESIDUE_INJECT="1.0")
    r = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr
    tag, status, value = r.stdout.split()
    assert (tag, int(status)) == ("STATUS", 8), r.stdout
    # Im b(0,0) = 1 at every z of one component: sqrt(Nz) / n
    assert abs(float(value) - np.sqrt(32.0) / 32 ** 3) < 1e-9, value
