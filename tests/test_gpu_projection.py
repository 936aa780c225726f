"""GPU parity of the projection G and the projected tangent G(K : dF^T)
against the CPU oracle (restating projection.cpp:123-194), plus the
reference's own property assertions (test_projection.cpp:96-244) on the GPU."""
import os

import numpy as np
import pytest

from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M

pytestmark = pytest.mark.gpu

# (points, lengths, tdim, nyquist mode) -- odd, even, prime, anisotropic,
# 2-d and plane-strain shapes, both Nyquist modes (test_projection.cpp:109-115)
CASES = [
    ((5, 5, 5), None, 3, 0),
    ((5, 3, 7), (1.0, 2.0, 0.5), 3, 0),
    ((4, 4, 4), None, 3, 0),
    ((4, 4, 4), None, 3, 1),
    ((4, 5, 3), (1.0, 0.7, 1.3), 3, 1),
    ((6, 5), None, 2, 0),
    ((5, 7), None, 3, 0),
    ((4, 5), None, 2, 1),
    ((31, 31, 31), None, 3, 0),
    ((32, 32, 32), None, 3, 0),
    ((12, 10, 14), None, 3, 1),
    ((16, 9, 24), None, 3, 0),
    ((64, 64, 64), None, 3, 0),
    ((128, 64, 32), None, 3, 0),
    ((32, 256, 64), (2.0, 1.0, 0.5), 3, 0),
    ((512, 32, 32), None, 3, 0),
    ((512, 8, 16), (1.0, 0.5, 2.0), 3, 0),
    ((1024, 16, 32), None, 3, 0),
    ((32, 1024, 16), None, 3, 0),
    ((16, 16, 1024), None, 3, 0),
    ((64, 64, 64), None, 3, 1),
    ((1, 1, 1), None, 3, 0),
    ((2, 2, 2), None, 3, 0),
    ((3, 1, 2), None, 3, 0),
]


def _ids(c):
    return "x".join(map(str, c[0])) + f"-t{c[2]}-m{c[3]}"


@pytest.mark.parametrize("case", CASES, ids=[_ids(c) for c in CASES])
def test_projection_matches_oracle(case, oracle):
    pts, lengths, tdim, mode = case
    nc = tdim * tdim
    A = M.uniform_field(pts, nc, seed=11 + len(pts))
    ref, st, _ = oracle.apply_projection(pts, tdim, A, mode=mode, lengths=lengths)
    assert st == 0
    with abi.Context(pts, tdim, lengths=lengths, nyquist_mode=mode) as ctx:
        got = ctx.projection(ctx.field(nc, A)).download()
    scale = max(np.linalg.norm(ref), 1e-300)
    assert np.linalg.norm(got - ref) <= 1e-12 * max(scale, 1.0)


@pytest.mark.parametrize("case", CASES[:12], ids=[_ids(c) for c in CASES[:12]])
def test_projected_tangent_matches_oracle(case, oracle):
    pts, lengths, tdim, mode = case
    nc = tdim * tdim
    n = int(np.prod(pts))
    rng = np.random.default_rng(5)
    K = rng.uniform(-1, 1, nc * nc * n)
    dF = rng.uniform(-1, 1, nc * n)
    ref, st = oracle.apply_projected_tangent(pts, tdim, K, dF, mode=mode, lengths=lengths)
    assert st == 0
    with abi.Context(pts, tdim, lengths=lengths, nyquist_mode=mode) as ctx:
        got = ctx.projected_tangent(ctx.field(nc * nc, K), ctx.field(nc, dF)).download()
    assert np.linalg.norm(got - ref) <= 1e-12 * max(np.linalg.norm(ref), 1.0)


@pytest.mark.parametrize("pts", [(5, 5, 5), (5, 3, 7), (4, 4, 4), (32, 32, 32), (128, 128, 128)])
def test_idempotent_zero_mean_self_adjoint(pts):
    # test_projection.cpp:107-136 with the same 1e-10 / 1e-12 tolerances
    A = M.uniform_field(pts, 9, seed=1)
    B = M.uniform_field(pts, 9, seed=2)
    with abi.Context(pts, 3) as ctx:
        fa, fb = ctx.field(9, A), ctx.field(9, B)
        GA = ctx.projection(fa)
        GGA = ctx.projection(GA)
        GB = ctx.projection(fb)
        ga, gga = GA.download(), GGA.download()
        assert np.linalg.norm(gga - ga) < 1e-10 * max(1.0, np.linalg.norm(ga))
        assert np.all(np.abs(ctx.mean(GA)) < 1e-12)
        lhs, rhs = ctx.dot(fa, GB), ctx.dot(GA, fb)
        assert abs(lhs - rhs) <= 1e-10 * abs(rhs)


def test_constant_field_projects_to_zero():
    # test_projection.cpp:96-105
    pts = (5, 5, 5)
    n = 125
    A = np.zeros(9 * n)
    A[1 * n:2 * n] = 2.0
    A[8 * n:9 * n] = -0.7
    with abi.Context(pts, 3) as ctx:
        out = ctx.projection(ctx.field(9, A)).download()
    assert np.linalg.norm(out) < 1e-12 * np.linalg.norm(A)


def test_fourier_mode_known_answer():
    """Analytic projection of a single Fourier mode (SURVEY.md §8(d) config 4
    known-answer test): A_ij = a_ij cos(2 pi q.x) -> (a xi) (x) xi / |xi|^2 cos."""
    N = 16
    pts = (N, N, N)
    q = np.array([1, 2, 3])
    x = np.stack(np.meshgrid(*[np.arange(N)] * 3, indexing="ij"), axis=-1).reshape(-1, 3) / N
    phase = np.cos(2 * np.pi * x @ q)
    a = np.arange(1.0, 10.0).reshape(3, 3)
    expect_t = (a @ q)[:, None] * q[None, :] / (q @ q)
    A = np.concatenate([a.reshape(-1)[c] * phase for c in range(9)])
    E = np.concatenate([expect_t.reshape(-1)[c] * phase for c in range(9)])
    with abi.Context(pts, 3) as ctx:
        got = ctx.projection(ctx.field(9, A)).download()
    assert np.max(np.abs(got - E)) < 1e-12


def test_plane_strain_stays_in_plane():
    # test_projection.cpp:138-148
    pts = (5, 7)
    n = 35
    A = M.uniform_field(pts, 9, seed=9)
    with abi.Context(pts, 3) as ctx:
        GA = ctx.projection(ctx.field(9, A)).download().reshape(3, 3, n)
    assert np.max(np.abs(GA[:, 2, :])) < 1e-12


def test_linearity_of_projected_tangent():
    # test_projection.cpp:201-228
    pts = (3, 3)
    tdim = 2
    n = 9
    lam, mu = 0.58, 0.38
    C = np.zeros((2, 2, 2, 2))
    for i in range(2):
        for j in range(2):
            for k in range(2):
                for l in range(2):
                    C[i, j, k, l] = lam * (i == j) * (k == l) + mu * ((i == l) * (j == k) + (i == k) * (j == l))
    K = np.repeat(C.reshape(-1, 1), n, axis=1).reshape(-1)
    rng = np.random.default_rng(55)
    x, y = rng.uniform(-1, 1, 4 * n), rng.uniform(-1, 1, 4 * n)
    with abi.Context(pts, tdim) as ctx:
        fk = ctx.field(16, K)
        lhs = ctx.projected_tangent(fk, ctx.field(4, 1.7 * x - 0.3 * y)).download()
        rx = ctx.projected_tangent(fk, ctx.field(4, x)).download()
        ry = ctx.projected_tangent(fk, ctx.field(4, y)).download()
    rhs = 1.7 * rx - 0.3 * ry
    assert np.linalg.norm(lhs - rhs) < 1e-12 * max(1.0, np.linalg.norm(rhs))


def test_shape_mismatch_is_invalid():
    with abi.Context((4, 4, 4), 3) as ctx:
        a = ctx.field(9)
        bad = ctx.field(4)
        with pytest.raises(abi.FmError) as e:
            ctx.projection(bad, a)
        assert e.value.status == 1


@pytest.mark.parametrize("N", [256, 512])
def test_config4_properties_full_size(N):
    """BASELINE.json config 4 at full size: seed 4 + N,
    nine i.i.d. U(-1,1) slabs.  The oracle does not fit at these sizes, so the
    check is by size-independent properties, all evaluated on the device:
    G(G(x)) = G(x), zero mean, self-adjointness <x, G y> = <G x, y>."""
    pts = (N, N, N)
    with abi.Context(pts, 3) as ctx:
        x = ctx.field(9, M.uniform_field(pts, 9, seed=4 + N))
        y = ctx.field(9, M.uniform_field(pts, 9, seed=5 + N))
        Gx = ctx.projection(x)
        GGx = ctx.projection(Gx)
        ngx = ctx.norm(Gx)
        ctx.axpy(-1.0, Gx, GGx)
        assert ctx.norm(GGx) < 1e-10 * ngx
        assert np.all(np.abs(ctx.mean(Gx)) < 1e-12)
        Gy = ctx.projection(y, out=GGx)
        lhs, rhs = ctx.dot(x, Gy), ctx.dot(Gx, y)
        assert abs(lhs - rhs) <= 1e-10 * abs(rhs)


def test_config4_oracle_equality_128():
    """Config 4 at N = 128 (largest size the oracle runs in seconds):
    bitwise-close equality of G(x) against the CPU oracle."""
    N = 128
    pts = (N, N, N)
    x = M.uniform_field(pts, 9, seed=4 + N)
    from oracle import oracle as O
    ref, st, _ = O.apply_projection(pts, 3, x)
    assert st == 0
    with abi.Context(pts, 3) as ctx:
        got = ctx.projection(ctx.field(9, x)).download()
    assert np.linalg.norm(got - ref) <= 1e-12 * np.linalg.norm(ref)


def _digest_child(pts, env):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys, hashlib; sys.path.insert(0, %r)\n"
        "from paper_1603_08893_b200 import abi, microstructure as M\n"
        "pts = %r\n"
        "A = M.uniform_field(pts, 9, seed=21)\n"
        "with abi.Context(pts, 3) as ctx:\n"
        "    out = ctx.projection(ctx.field(9, A)).download()\n"
        "    print(hashlib.sha1(out.tobytes()).hexdigest(), ','.join(ctx.kernel_names))\n" % (root, pts))
    r = subprocess.run([sys.executable, "-c", code], env=dict(os.environ, **env), capture_output=True, text=True,
                       timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.split()


@pytest.mark.parametrize("pts", [(512, 64, 32), (512, 16, 128)])
def test_warp_per_line_x_pass_is_bit_identical_to_the_lockstep_one(pts):
    """The 512-point x pass k_x_warp (one warp per line, TMA in and out,
    projection_xw.cu) against the lane-pair k_x_stream it replaced
    (FM_XDIRECT=4): same butterflies in the same order, so the same bits."""
    new, names_new = _digest_child(pts, {})
    old, names_old = _digest_child(pts, {"FM_XDIRECT": "4"})
    assert "k_x_warp" in names_new and "k_x_stream" in names_old, (names_new, names_old)
    assert new == old


def test_projection_256_matches_oracle_golden():
    """BASELINE config 4 at 256^3 against the CPU oracle (tests/golden/make_golden.py
    proj256 -> proj256.npz: 2^18 fixed samples, norm and per-component checksums of
    G applied to the seeded U(-1,1) field), 1e-12; the 512^3 run of the oracle does
    not fit the CPU container, where the analytic known-answer test
    (test_gpu_config4_known_answer.py) and the idempotence check take over."""
    import sys
    sys.path.insert(0, os.path.dirname(os.path.abspath(__file__)))
    from golden_util import checksums, rel, sample_index
    g = np.load(os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "proj256.npz"))
    pts = (256, 256, 256)
    A = M.uniform_field(pts, 9, 4)
    with abi.Context(pts, 3) as ctx:
        fa = ctx.field(9, A)
        out = ctx.projection(fa)
        x = out.download()
        again = ctx.projection(out).download()  # compatibility: G(G(x)) = G(x)
    idx = sample_index(g["out_samp"].size, x.size)
    assert rel(x[idx], g["out_samp"]) <= 1e-12
    assert abs(np.linalg.norm(x) - g["out_norm"]) <= 1e-12 * g["out_norm"]
    cs, ref = checksums(x, 9), g["out_sums"]
    assert np.all(np.abs(cs[1] - ref[1]) <= 1e-12 * ref[1])
    assert np.all(np.abs(cs[0] - ref[0]) <= 1e-12 * np.sqrt(ref[1] * 256 ** 3))
    assert np.linalg.norm(again - x) <= 1e-13 * np.linalg.norm(x)


def _sample_child(pts, env, path):
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    code = (
        "import sys; sys.path.insert(0, %r)\n"
        "import numpy as np\n"
        "from paper_1603_08893_b200 import abi, microstructure as M\n"
        "pts = %r\n"
        "A = M.uniform_field(pts, 9, seed=23)\n"
        "with abi.Context(pts, 3) as ctx:\n"
        "    out = ctx.projection(ctx.field(9, A)).download()\n"
        "    np.save(%r, out)\n"
        "    print(','.join(ctx.kernel_names))\n" % (root, pts, path))
    r = subprocess.run(["timeout", "300", sys.executable, "-c", code], env=dict(os.environ, **env),
                       capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    return r.stdout.strip()


@pytest.mark.parametrize("pts", [(1024, 8, 16), (1024, 48, 32)])
def test_cluster_x_pass_1024_matches_default(pts, tmp_path):
    """The cluster form of k_x_warp for 1024-point lines (the line split over a
    2-CTA cluster, the outermost radix-2 step through distributed shared
    memory) against k_x_fast4 (FM_XW1024=0): another factorisation of the same
    transform, so equal to round-off, not bit for bit."""
    a, b = str(tmp_path / "a.npy"), str(tmp_path / "b.npy")
    names_def = _sample_child(pts, {"FM_XW1024": "0"}, a)
    names_cl = _sample_child(pts, {}, b)
    assert "k_x_fast4" in names_def and "k_x_warp" in names_cl, (names_def, names_cl)
    x, y = np.load(a), np.load(b)
    assert np.linalg.norm(x - y) <= 1e-14 * np.linalg.norm(x)


@pytest.mark.parametrize("pts", [(8, 1024, 16), (24, 1024, 64)])
def test_cluster_y_pass_1024_matches_k_y_fast(pts, tmp_path):
    """The cluster form of the 1024-point y pass (k_y_warp) against k_y_fast
    (FM_YW1024=0): equal to round-off."""
    a, b = str(tmp_path / "a.npy"), str(tmp_path / "b.npy")
    names_def = _sample_child(pts, {"FM_YW1024": "0"}, a)
    names_cl = _sample_child(pts, {}, b)
    assert "k_y_fast" in names_def and "k_y_warp" in names_cl, (names_def, names_cl)
    x, y = np.load(a), np.load(b)
    assert np.linalg.norm(x - y) <= 1e-14 * np.linalg.norm(x)
