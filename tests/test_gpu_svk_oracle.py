"""Oracle parity of the hot-path pass-1 kernels themselves (SURVEY §8(a)
a7/a11): the matrix-free SVK action in the pipelined z-forward pass
(k_zf_pipe<M, PRO_SVK, ...>, the kernel behind bench.py's `value`) and the
materialised-K4 pass (k_zf_fast<M, PRO_K4>), each against the oracle's
hyperelastic_evaluate K4 followed by apply_projected_tangent
(hyperelastic.cpp:55-63, projection.cpp:173-194).

The template instantiation of pass 1 depends only on Nz (M = Nz/2), so the
thin (a, b, 256) grids run the very instantiation the 256^3 headline runs
(M = 128) at a size the oracle finishes in a second; 64^3 and 128^3 cover
whole cubes.  Tolerance: 1e-12 relative (fp64, different summation order)."""
import numpy as np
import pytest

from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M

pytestmark = pytest.mark.gpu

SHAPES = [(64, 64, 64), (128, 128, 128), (16, 16, 256), (8, 8, 512), (32, 32, 32)]


def _inputs(pts, phases, seed):
    n = int(np.prod(pts))
    if phases == "labels":  # two phases -> 1-byte labels + pair table in pass 1
        lam, mu, _, _ = M.bind_parameters(M.bernoulli(pts, 0.3, seed),
                                          [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
    else:  # > 256 distinct pairs -> per-voxel lambda, mu fields
        rng = np.random.default_rng(seed)
        lam, mu = rng.uniform(0.5, 6.0, n), rng.uniform(0.3, 4.0, n)
    F0 = abi.identity_field(pts, 3) + 0.05 * M.uniform_field(pts, 9, seed + 40)
    dF = M.uniform_field(pts, 9, seed + 41)
    return lam, mu, F0, dF


def _rel(a, b):
    return np.linalg.norm(a - b) / np.linalg.norm(b)


@pytest.mark.parametrize("phases", ["labels", "per_voxel"])
@pytest.mark.parametrize("pts", SHAPES, ids=lambda p: "x".join(map(str, p)))
def test_matrix_free_svk_matvec_matches_oracle(pts, phases, oracle):
    lam, mu, F0, dF0 = _inputs(pts, phases, 3)
    P_ref, K_ref, st, _ = oracle.hyper_evaluate(F0, lam, mu)
    assert st == 0
    ref, st = oracle.apply_projected_tangent(pts, 3, K_ref, dF0)
    assert st == 0
    with abi.Context(pts, 3) as ctx:
        F, dF, P, out = ctx.field(9, F0), ctx.field(9, dF0), ctx.field(9), ctx.field(9)
        model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
        model.evaluate(F, P)
        model.apply(dF, out)
        got, Pg = out.download(), P.download()
        names = ctx.kernel_names
        model.close()
    assert _rel(Pg, P_ref) <= 1e-14
    assert _rel(got, ref) <= 1e-12, _rel(got, ref)
    # the headline pass-1 kernel is the one that ran (the pipelined pass is
    # used up to Nz = 256; longer z-lines take k_zf_fast)
    assert ("k_zf_pipe" if pts[2] <= 256 else "k_zf_fast") in names, names


@pytest.mark.parametrize("pts", SHAPES, ids=lambda p: "x".join(map(str, p)))
def test_k4_matvec_fast_path_matches_oracle(pts, oracle):
    lam, mu, F0, dF0 = _inputs(pts, "labels", 4)
    _, K_ref, st, _ = oracle.hyper_evaluate(F0, lam, mu)
    ref, st = oracle.apply_projected_tangent(pts, 3, K_ref, dF0)
    assert st == 0
    with abi.Context(pts, 3) as ctx:
        F, dF, P, out = ctx.field(9, F0), ctx.field(9, dF0), ctx.field(9), ctx.field(9)
        model = abi.Model(ctx, "hyper", lam, mu, matrix_free=False)
        model.evaluate(F, P)
        K = model.tangent().download()
        model.apply(dF, out)
        got = out.download()
        names = ctx.kernel_names
        model.close()
    assert _rel(K, K_ref) <= 1e-14
    assert _rel(got, ref) <= 1e-12, _rel(got, ref)
    assert "k_zf_fast" in names or "k_zf_pipe" in names, names
