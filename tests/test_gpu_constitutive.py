"""GPU parity of the per-voxel constitutive kernels against the CPU oracle
(hyperelastic.cpp:10-65, simo.cpp:26-196), including the node-indexed error
semantics (lowest offending node, as the reference's first throw)."""
import numpy as np
import pytest

from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M

pytestmark = pytest.mark.gpu


def _identity(n, tdim=3):
    F = np.zeros(tdim * tdim * n)
    for i in range(tdim):
        F[(i * tdim + i) * n:(i * tdim + i + 1) * n] = 1.0
    return F


@pytest.mark.parametrize("tdim,pts", [(3, (6, 5, 7)), (2, (9, 8)), (3, (32, 32, 32))])
def test_hyper_matches_oracle(oracle, tdim, pts):
    n = int(np.prod(pts))
    rng = np.random.default_rng(3)
    F = _identity(n, tdim) + rng.uniform(-0.2, 0.2, tdim * tdim * n)
    lam = rng.uniform(0.3, 6.0, n)
    mu = rng.uniform(0.2, 4.0, n)
    P_ref, K_ref, st, _ = oracle.hyper_evaluate(F, lam, mu, tdim)
    assert st == 0
    with abi.Context(pts, tdim) as ctx:
        P, K = ctx.hyper_evaluate(ctx.field(tdim * tdim, F), lam, mu)
        P, K = P.download(), K.download()
    assert np.max(np.abs(P - P_ref)) <= 1e-14 * np.max(np.abs(P_ref))
    assert np.max(np.abs(K - K_ref)) <= 1e-14 * np.max(np.abs(K_ref))


def test_hyper_reports_lowest_inverted_node(oracle):
    pts = (8, 8, 8)
    n = 512
    F = _identity(n)
    for q in (300, 77, 401):
        F[0 * n + q] = -1.0
    lam, mu = np.full(n, 0.5), np.full(n, 0.3)
    _, _, st, bad = oracle.hyper_evaluate(F, lam, mu)
    assert st == 4 and bad == 77
    with abi.Context(pts, 3) as ctx:
        with pytest.raises(abi.FmError) as e:
            ctx.hyper_evaluate(ctx.field(9, F), lam, mu)
    assert e.value.status == 4 and e.value.info["node"] == 77


def _random_simo_state(oracle, n, rng, ty_hi=1.0, ty_lo=0.01):
    """Committed states reached by a random pre-deformation (test_simo.cpp:190-196)."""
    e = M.ElasticParams(1.0, 0.3)
    lam, mu = np.full(n, e.lame_lambda), np.full(n, e.lame_mu)
    ty = np.where(np.arange(n) % 2 == 0, ty_hi, ty_lo)
    h = np.full(n, 0.05)
    I = _identity(n)
    Fold = I + rng.uniform(-0.05, 0.05, 9 * n)
    pre = oracle.simo_evaluate(Fold, I, I, np.zeros(n), lam, mu, ty, h, want_K=False)
    F = Fold + rng.uniform(-0.04, 0.04, 9 * n)
    return F, Fold, pre["be"], pre["epsp"], lam, mu, ty, h


@pytest.mark.parametrize("n", [64, 4096])
def test_simo_matches_oracle_both_branches(oracle, n):
    rng = np.random.default_rng(2025 + n)
    F, Fold, be, ep, lam, mu, ty, h = _random_simo_state(oracle, n, rng)
    ref = oracle.simo_evaluate(F, Fold, be, ep, lam, mu, ty, h)
    assert ref["status"] == 0
    plastic = ref["epsp"] > ep
    assert plastic.sum() > 3 and (~plastic).sum() > 3
    with abi.Context((n, 1, 1), 3) as ctx:
        P, K, be_t, ep_t = ctx.simo_evaluate(ctx.field(9, F), ctx.field(9, Fold), be, ep, lam, mu, ty, h)
        P, K, be_t, ep_t = P.download(), K.download(), be_t.download(), ep_t.download()
    rel = lambda a, b: np.max(np.abs(a - b)) / np.max(np.abs(b))
    assert rel(P, ref["P"]) < 1e-12
    assert rel(K, ref["K"]) < 1e-10
    assert rel(be_t, ref["be"]) < 1e-13
    assert np.array_equal(ep_t > ep, plastic)  # identical plastic switch decisions
    assert np.max(np.abs(ep_t - ref["epsp"])) < 1e-14


def test_simo_degenerate_and_virgin_states(oracle):
    # F = I, b_e = I: all eigenvalues equal (the divided-difference branch)
    n = 4
    e = M.ElasticParams(1.0, 0.3)
    lam, mu = np.full(n, e.lame_lambda), np.full(n, e.lame_mu)
    ty, h = np.full(n, 0.01), np.full(n, 0.05)
    I = _identity(n)
    F = I.copy()
    F[1 * n + 1] = 0.004   # elastic shear
    F[1 * n + 2] = 0.05    # plastic shear
    F[4 * n + 3] = 1.02    # uniaxial
    ref = oracle.simo_evaluate(F, I, I, np.zeros(n), lam, mu, ty, h)
    with abi.Context((n, 1, 1), 3) as ctx:
        P, K, be_t, ep_t = ctx.simo_evaluate(ctx.field(9, F), ctx.field(9, I), I, np.zeros(n), lam, mu, ty, h)
        P, K = P.download(), K.download()
    assert np.max(np.abs(P - ref["P"])) < 1e-15
    assert np.max(np.abs(K - ref["K"])) < 1e-12 * np.max(np.abs(ref["K"]))


def test_simo_inverted_node():
    n = 16
    e = M.ElasticParams(1.0, 0.3)
    I = _identity(n)
    F = I.copy()
    F[0 * n + 9] = -2.0
    with abi.Context((n, 1, 1), 3) as ctx:
        with pytest.raises(abi.FmError) as err:
            ctx.simo_evaluate(ctx.field(9, F), ctx.field(9, I), I, np.zeros(n), np.full(n, e.lame_lambda),
                              np.full(n, e.lame_mu), np.full(n, 0.01), np.full(n, 0.05))
    assert err.value.status == 4 and err.value.info["node"] == 9


@pytest.mark.parametrize("tdim,kind", [(3, 0), (3, 1), (3, 2), (2, 0), (2, 1), (2, 2)])
def test_equivalent_stress_matches_oracle(tdim, kind, oracle):
    """fm_equivalent_stress against the restated
    equivalent_stress / inv2 / dot22 (material.cpp:14-31)."""
    pts = (6, 5, 7) if tdim == 3 else (9, 8)
    n = int(np.prod(pts))
    rng = np.random.default_rng(11 + kind)
    F = rng.uniform(-0.2, 0.2, tdim * tdim * n)
    for i in range(tdim):
        F[(i * tdim + i) * n:(i * tdim + i + 1) * n] += 1.0
    P = rng.uniform(-1, 1, tdim * tdim * n)
    ref, st, _ = oracle.equivalent_stress(F, P, n, tdim, kind)
    assert st == 0
    with abi.Context(pts, tdim) as ctx:
        got = ctx.equivalent_stress(ctx.field(tdim * tdim, F), ctx.field(tdim * tdim, P), kind).download()
    assert np.max(np.abs(got - ref) / np.maximum(1.0, np.abs(ref))) < 1e-14


def test_equivalent_stress_singular_reports_first_node():
    pts = (4, 4, 4)
    n = 64
    F = abi.identity_field(pts, 3)
    for node in (37, 9):
        for c in range(9):
            F[c * n + node] = 0.0  # det F = 0 -> SingularTensor(first node)
    P = np.ones(9 * n)
    with abi.Context(pts, 3) as ctx:
        with pytest.raises(abi.FmError) as e:
            ctx.equivalent_stress(ctx.field(9, F), ctx.field(9, P), abi.Context.EQ_PK2)
    assert e.value.status == 6 and e.value.info["node"] == 9
