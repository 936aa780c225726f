"""Slab decomposition validated on one B200: P slab ranks
emulated on the device ("virtual ranks": the transpose-fused y and x passes
store across the side-by-side rank buffers)
must reproduce the P = 1 projection bit for bit -- the z / y / x passes
compute the same lines in the same order, only the layouts between them
change -- and the Newton solve must match the single-rank run."""
import numpy as np
import pytest

from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("pts,P", [((64, 64, 64), 2), ((64, 64, 64), 8), ((32, 32, 32), 4),
                                   ((128, 64, 32), 8), ((12, 10, 14), 2), ((16, 24, 9), 4),
                                   ((256, 256, 32), 8),
                                   # long routed x lines (512: direct lane-pair pass, 1024: 4-column tiles) and y lines
                                   # (P = 1 at 512: the warp-per-line TMA pass k_x_warp, one tile per CTA and,
                                   # at 64 x 32, two to three tiles per CTA, against the routed k_x_stream)
                                   ((512, 32, 16), 4), ((512, 64, 32), 2), ((1024, 16, 32), 2), ((1024, 32, 32), 8), ((32, 512, 16), 2),
                                   ((16, 1024, 32), 4)])
def test_virtual_ranks_bitwise_equal(pts, P):
    A = M.uniform_field(pts, 9, seed=3)
    n = int(np.prod(pts))
    K = np.random.default_rng(1).uniform(-1, 1, 81 * n)
    with abi.Context(pts, 3) as ctx:
        fa, fk = ctx.field(9, A), ctx.field(81, K)
        g1 = ctx.projection(fa).download()
        m1 = ctx.projected_tangent(fk, fa).download()
        ctx.set_virtual_ranks(P)
        assert ctx.ranks() == (P, 0, True)
        gp = ctx.projection(fa).download()
        mp = ctx.projected_tangent(fk, fa).download()
    if pts[1] == 1024:
        # P = 1 runs the 2-CTA-cluster y pass (1024 = 2 x 512 across the CTA pair), the slab ranks the
        # 16 x 16 x 4 k_y_fast: two factorisations of the same transform, equal to round-off
        assert np.linalg.norm(g1 - gp) <= 1e-14 * np.linalg.norm(g1)
        assert np.linalg.norm(m1 - mp) <= 1e-14 * np.linalg.norm(m1)
        return
    assert np.array_equal(g1, gp)
    assert np.array_equal(m1, mp)


@pytest.mark.parametrize("pts,P", [((64, 64, 64), 2), ((64, 64, 64), 8), ((12, 10, 14), 2), ((16, 24, 9), 4),
                                   ((128, 64, 32), 8), ((512, 64, 32), 2), ((32, 512, 16), 2)])
def test_staged_all_to_all_bitwise_equal(pts, P):
    """The A/B arm (fm_ctx_set_transpose(ctx, 1), FM_TRANSPOSE=nccl on devices):
    local y and x passes with pack / all-to-all / unpack transposes between
    them.  In the virtual mode the all-to-all is the same block copies on one
    device, so the pack and unpack index maps are checked exactly: bit-equal to
    P = 1 and to the fused peer-store form."""
    A = M.uniform_field(pts, 9, seed=5)
    n = int(np.prod(pts))
    K = np.random.default_rng(2).uniform(-1, 1, 81 * n)
    with abi.Context(pts, 3) as ctx:
        fa, fk = ctx.field(9, A), ctx.field(81, K)
        g1 = ctx.projection(fa).download()
        m1 = ctx.projected_tangent(fk, fa).download()
        ctx.set_transpose(1)
        ctx.set_virtual_ranks(P)
        gs = ctx.projection(fa).download()
        ms = ctx.projected_tangent(fk, fa).download()
        ctx.set_transpose(0)  # back to the fused form on the same context
        gf = ctx.projection(fa).download()
    assert np.array_equal(g1, gs)
    assert np.array_equal(m1, ms)
    assert np.array_equal(g1, gf)


def test_virtual_ranks_solve_matches_single_rank():
    pts = (32, 32, 32)
    pg = M.bernoulli(pts, 0.3, seed=2)
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
    fb = M.simple_shear_program(0.1, 1, 3)[0]
    out = []
    for P in (1, 4):
        with abi.Context(pts, 3) as ctx:
            ctx.set_virtual_ranks(P)
            model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
            F = ctx.field(9, abi.identity_field(pts, 3))
            rep = model.solve_increment(F, fb)
            out.append((F.download(), rep))
            model.close()
    (F1, r1), (F4, r4) = out
    assert r1["passes"] == r4["passes"]
    assert all(abs(a - b) <= 1 for a, b in zip(r1["cg_it"], r4["cg_it"]))
    assert np.linalg.norm(F1 - F4) / np.linalg.norm(F1) < 1e-12


def test_indivisible_grid_is_rejected():
    with abi.Context((10, 12, 8), 3) as ctx:
        with pytest.raises(abi.FmError) as e:
            ctx.set_virtual_ranks(4)
        assert e.value.status == 11
