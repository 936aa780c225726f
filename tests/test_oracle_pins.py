"""Pins the CPU oracle (oracle/fftmech_oracle.cpp) to the reference before it
is trusted as the parity checker:

* golden run records the reference itself wrote (proj/unit_det_out1/report.csv,
  unit_run_out, unit_vtk_out), reproduced through the same setup path
  (make_laminate, bind_parameters, expand_loading, run_program);
* the reference's own unit assertions (test_projection.cpp, test_solver.cpp,
  test_hyperelastic.cpp, test_simo.cpp) re-run against the oracle;
* the restated FFT against an independent O(n^2) DFT (naive_dft.cpp:11-31).
"""
import json
import os

import numpy as np
import pytest

from paper_1603_08893_b200 import microstructure as M

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_reports.json")


def _golden():
    with open(GOLDEN) as f:
        return json.load(f)


def _identity(points, tdim):
    n = int(np.prod(points))
    F = np.zeros(tdim * tdim * n)
    for i in range(tdim):
        F[(i * tdim + i) * n:(i * tdim + i + 1) * n] = 1.0
    return F


# ------------------------------------------------------------ golden records
def test_laminate_report_matches_reference_golden(oracle):
    """proj/unit_det_out1/report.csv (config of test_config_io.cpp:206-217)."""
    g = _golden()["unit_det_out1"]
    pg = M.make_laminate((5, 4), [0.4, 0.6])
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(5.0, 0.25)])
    _, _, reps, st, _ = oracle.run_program((5, 4), 2, 0, lam, mu, M.simple_shear_program(0.15, 3, 2))
    assert st == 0
    for r, row in zip(reps, g["rows"]):
        assert r["passes"] == row["newton_iters"]
        assert sum(r["cg_it"]) == row["cg_iters_total"]
        # last rel_update, printed with 17 digits by write_report_csv
        assert r["rel_update"][-1] == pytest.approx(row["residual"], rel=1e-9)


@pytest.mark.parametrize("name,points,gamma,incs", [("unit_run_out", (4, 4), 0.2, 2),
                                                    ("unit_vtk_out", (3, 3), 0.05, 1)])
def test_homogeneous_reports_match_reference_golden(oracle, name, points, gamma, incs):
    g = _golden()[name]
    pg = M.make_laminate(points, [1.0])
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3)])
    _, _, reps, st, _ = oracle.run_program(points, 2, 0, lam, mu, M.simple_shear_program(gamma, incs, 2))
    assert st == 0
    for r, row in zip(reps, g["rows"]):
        assert r["passes"] == row["newton_iters"] and sum(r["cg_it"]) == row["cg_iters_total"]
        assert r["rel_update"][-1] == row["residual"] == 0.0


def test_mt19937_64_standard_value():
    # [rand.predef]: the 10000th output of a default-constructed mt19937_64
    assert int(M.MT19937_64(5489).raw(10000)[-1]) == 9981545732273789042


# --------------------------------------------------------------------- FFT
def _naive_dft(points, x, sign):
    n = int(np.prod(points))
    idx = np.stack(np.meshgrid(*[np.arange(p) for p in points], indexing="ij"), -1).reshape(n, -1)
    ph = np.zeros((n, n))
    for a, p in enumerate(points):
        ph += np.outer(idx[:, a], idx[:, a]) / p
    return np.exp(sign * 2j * np.pi * ph) @ x


@pytest.mark.parametrize("points", [(5,), (8,), (31,), (12,), (5, 3, 7), (4, 6, 2), (9, 10)])
def test_fft_matches_naive_dft(oracle, points):
    rng = np.random.default_rng(1)
    n = int(np.prod(points))
    x = rng.uniform(-1, 1, n) + 1j * rng.uniform(-1, 1, n)
    for sign in (-1, 1):
        got = oracle.fft(points, x[None, :], sign)[0]
        ref = _naive_dft(points, x, sign)
        assert np.max(np.abs(got - ref)) < 1e-12 * n


# -------------------------------------------------------------- projection
def test_ghat_closed_form(oracle):
    # test_projection.cpp:43-94
    g = oracle.ghat((3, 3, 3), 3).reshape(3, 3, 27)
    assert np.all(g[:, :, 0] == 0.0)
    node = 1 * 9  # q = (1,0,0)
    assert np.allclose(g[:, :, node], np.diag([1.0, 0, 0]))
    g4 = oracle.ghat((4, 4, 4), 3, mode=0).reshape(3, 3, 4, 4, 4)
    assert np.all(g4[:, :, 2] == 0.0)
    gi = oracle.ghat((4, 5), 2, mode=1).reshape(2, 2, 4, 5)
    assert np.allclose(gi[:, :, 2, 1], np.eye(2))
    for mode in (0, 1):
        gs = oracle.ghat((4, 5, 3), 3, mode=mode, lengths=(1.0, 0.7, 1.3)).reshape(3, 3, -1)
        for k in range(gs.shape[2]):
            t = gs[:, :, k]
            assert np.allclose(t, t.T, rtol=1e-14, atol=0)
            assert np.allclose(t @ t, t, rtol=1e-13, atol=1e-15)


@pytest.mark.parametrize("points,lengths,mode", [((5, 5, 5), None, 0), ((5, 3, 7), (1.0, 2.0, 0.5), 0),
                                                 ((4, 4, 4), None, 0), ((4, 4, 4), None, 1),
                                                 ((6, 5), None, 0)])
def test_projection_properties(oracle, points, lengths, mode):
    # test_projection.cpp:107-136
    tdim = len(points)
    rng = np.random.default_rng(1234)
    n = int(np.prod(points))
    A = rng.uniform(-1, 1, tdim * tdim * n)
    B = rng.uniform(-1, 1, tdim * tdim * n)
    GA, st, _ = oracle.apply_projection(points, tdim, A, mode=mode, lengths=lengths)
    GGA, _, _ = oracle.apply_projection(points, tdim, GA, mode=mode, lengths=lengths)
    GB, _, _ = oracle.apply_projection(points, tdim, B, mode=mode, lengths=lengths)
    assert st == 0
    assert np.linalg.norm(GGA - GA) < 1e-10 * max(1.0, np.linalg.norm(GA))
    assert np.all(np.abs(GA.reshape(tdim * tdim, n).mean(axis=1)) < 1e-12)
    assert A @ GB == pytest.approx(GA @ B, rel=1e-10)


def test_projected_tangent_composes(oracle):
    # test_projection.cpp:231-244: G(trans2(ddot42(K, trans2(dF)))) == fused
    rng = np.random.default_rng(99)
    n = 27
    K = rng.uniform(-1, 1, 81 * n)
    dF = rng.uniform(-1, 1, 9 * n)
    K4 = K.reshape(3, 3, 3, 3, n)
    dFt = dF.reshape(3, 3, n).transpose(1, 0, 2)
    # ddot42: C_ij = A_ijkl B_lk
    dd = np.einsum("ijkln,lkn->ijn", K4, dFt)
    composed, _, _ = oracle.apply_projection((3, 3, 3), 3, dd.transpose(1, 0, 2).reshape(-1))
    fused, _ = oracle.apply_projected_tangent((3, 3, 3), 3, K, dF)
    assert np.linalg.norm(fused - composed) < 1e-12 * max(1.0, np.linalg.norm(composed))


# ------------------------------------------------------------ hyperelastic
def _svk_fd(oracle, F, lam, mu, h=1e-6):
    n = lam.size
    K = np.zeros((3, 3, 3, 3, n))
    for k in range(3):
        for l in range(3):
            Fp, Fm = F.copy(), F.copy()
            Fp[(k * 3 + l) * n:(k * 3 + l + 1) * n] += h
            Fm[(k * 3 + l) * n:(k * 3 + l + 1) * n] -= h
            Pp = oracle.hyper_evaluate(Fp, lam, mu, 3, False)[0].reshape(3, 3, n)
            Pm = oracle.hyper_evaluate(Fm, lam, mu, 3, False)[0].reshape(3, 3, n)
            K[:, :, k, l] = ((Pp - Pm) / (2 * h)).transpose(1, 0, 2)  # result(q,i,j,k,l) = dP_ji/dF_kl
    return K.reshape(-1)


def test_hyperelastic_identity_and_fd(oracle):
    # test_hyperelastic.cpp:26-86
    e = M.ElasticParams(1.0, 0.3)
    n = 8
    lam, mu = np.full(n, e.lame_lambda), np.full(n, e.lame_mu)
    P, K, st, _ = oracle.hyper_evaluate(_identity((2, 2, 2), 3), lam, mu)
    assert st == 0 and np.linalg.norm(P) == 0.0
    K = K.reshape(3, 3, 3, 3, n)
    d = np.eye(3)
    C = (e.lame_lambda * np.einsum("ij,kl->ijkl", d, d)
         + e.lame_mu * (np.einsum("il,jk->ijkl", d, d) + np.einsum("ik,jl->ijkl", d, d)))
    assert np.allclose(K, C[..., None], rtol=1e-14, atol=1e-15)
    rng = np.random.default_rng(123)
    F = _identity((2, 2, 1), 3) + rng.uniform(-0.15, 0.15, 36)
    lam4, mu4 = np.full(4, e.lame_lambda), np.full(4, e.lame_mu)
    _, K, _, _ = oracle.hyper_evaluate(F, lam4, mu4)
    Kfd = _svk_fd(oracle, F, lam4, mu4)
    assert np.linalg.norm(K - Kfd) / np.linalg.norm(Kfd) < 1e-6


def test_hyperelastic_inverted_reports_first_node(oracle):
    # test_hyperelastic.cpp:124-135
    n = 4
    F = _identity((4, 1, 1), 3)
    F[0 * n + 2] = -1.0
    F[0 * n + 3] = -1.0
    _, _, st, bad = oracle.hyper_evaluate(F, np.full(n, 0.5), np.full(n, 0.3))
    assert st == 4 and bad == 2


# -------------------------------------------------------------------- Simo
def _simo(oracle, F, Fold=None, be=None, ep=None, ty0=0.01, h=0.05):
    n = F.size // 9
    e = M.ElasticParams(1.0, 0.3)
    I = _identity((n, 1, 1), 3)
    return oracle.simo_evaluate(F, I if Fold is None else Fold, I if be is None else be,
                                np.zeros(n) if ep is None else ep, np.full(n, e.lame_lambda),
                                np.full(n, e.lame_mu), np.full(n, ty0), np.full(n, h))


def test_simo_virgin_state(oracle):
    # test_simo.cpp:75-95
    out = _simo(oracle, _identity((1, 1, 1), 3))
    e = M.ElasticParams(1.0, 0.3)
    d = np.eye(3)
    C = (e.lame_lambda * np.einsum("ij,kl->ijkl", d, d)
         + e.lame_mu * (np.einsum("il,jk->ijkl", d, d) + np.einsum("ik,jl->ijkl", d, d)))
    assert np.linalg.norm(out["P"]) < 1e-14 and out["epsp"][0] == 0.0
    assert np.allclose(out["K"].reshape(3, 3, 3, 3), C, rtol=1e-12, atol=1e-14)


def test_simo_hardening_line(oracle):
    # test_simo.cpp:130-179: after each plastic increment tau_eq == tau_y0 + H eps_p
    e = M.ElasticParams(1.0, 0.3)
    Fold = _identity((1, 1, 1), 3)
    be, ep = _identity((1, 1, 1), 3), np.zeros(1)
    worst, prev = 0.0, 0.0
    for step in range(1, 13):
        F = _identity((1, 1, 1), 3)
        F[1] = 0.01 * step
        out = _simo(oracle, F, Fold, be, ep)
        lb, V = oracle.sym_eig3(out["be"])
        lnb = V @ np.diag(np.log(lb)) @ V.T
        tau = 0.5 * e.lame_lambda * np.trace(lnb) * np.eye(3) + e.lame_mu * lnb
        dev = tau - np.trace(tau) / 3 * np.eye(3)
        taueq = np.sqrt(1.5 * np.sum(dev * dev))
        if out["epsp"][0] > prev:
            worst = max(worst, abs(taueq - (0.01 + 0.05 * out["epsp"][0])))
        assert out["epsp"][0] >= prev
        prev = out["epsp"][0]
        be, ep, Fold = out["be"], out["epsp"], F
    assert worst < 1e-10 and prev > 0.05


def _trial_phi(F, Fold, be, ep, ty0, h=0.05):
    """Elastic-predictor yield value, recomputed independently (test_simo.cpp:36-60)."""
    e = M.ElasticParams(1.0, 0.3)
    f = F.reshape(3, 3) @ np.linalg.inv(Fold.reshape(3, 3))
    btr = f @ be.reshape(3, 3) @ f.T
    w, V = np.linalg.eigh(0.5 * (btr + btr.T))
    eps = 0.5 * (V @ np.diag(np.log(w)) @ V.T)
    tau = e.lame_lambda * np.trace(eps) * np.eye(3) + 2 * e.lame_mu * eps
    dev = tau - np.trace(tau) / 3 * np.eye(3)
    return np.sqrt(1.5 * np.sum(dev * dev)) - (ty0 + h * ep[0]), ty0 + h * ep[0]


def test_simo_tangent_matches_fd(oracle):
    # test_simo.cpp:181-219: every sampled state away from the switch, < 1e-5
    rng = np.random.default_rng(2025)
    seen = {True: 0, False: 0}
    for trial in range(30):
        ty0 = 1.0 if trial % 2 == 0 else 0.01
        Fold = _identity((1, 1, 1), 3) + rng.uniform(-0.05, 0.05, 9)
        pre = _simo(oracle, Fold, ty0=ty0)
        be, ep = pre["be"], pre["epsp"]
        F = Fold + rng.uniform(-0.04, 0.04, 9)
        if np.linalg.det(F.reshape(3, 3)) <= 0.5:
            continue
        phi, scale = _trial_phi(F, Fold, be, ep, ty0)
        if abs(phi) < 0.05 * scale:
            continue
        seen[bool(phi > 0)] += 1
        out = _simo(oracle, F, Fold, be, ep, ty0=ty0)
        Kfd = np.zeros((3, 3, 3, 3))
        hh = 1e-7
        for k in range(3):
            for l in range(3):
                Fp, Fm = F.copy(), F.copy()
                Fp[k * 3 + l] += hh
                Fm[k * 3 + l] -= hh
                Pp = _simo(oracle, Fp, Fold, be, ep, ty0=ty0)["P"].reshape(3, 3)
                Pm = _simo(oracle, Fm, Fold, be, ep, ty0=ty0)["P"].reshape(3, 3)
                Kfd[:, :, k, l] = ((Pp - Pm) / (2 * hh)).T
        K = out["K"].reshape(3, 3, 3, 3)
        assert np.linalg.norm(K - Kfd) / np.linalg.norm(Kfd) < 1e-5
    assert seen[True] > 3 and seen[False] > 3


def test_sym_eig3(oracle):
    rng = np.random.default_rng(7)
    for _ in range(50):
        A = rng.uniform(-1, 1, (3, 3))
        A = A + A.T
        lam, V = oracle.sym_eig3(A)
        assert np.allclose(V @ np.diag(lam) @ V.T, A, atol=1e-13)
        assert np.allclose(V.T @ V, np.eye(3), atol=1e-14)
        assert np.all(np.diff(lam) >= 0)
    lam, V = oracle.sym_eig3(np.eye(3))
    assert np.allclose(lam, 1.0)


# ------------------------------------------------------------------ solver
def test_homogeneous_cell_is_exact(oracle):
    # test_solver.cpp:86-107
    pts = (4, 3, 5)
    n = 60
    e = M.ElasticParams(1.0, 0.3)
    fbar = np.eye(3)
    fbar[0, 1], fbar[0, 0], fbar[2, 0] = 0.37, 1.05, -0.11
    F, _, reps, st, _ = oracle.run_program(pts, 3, 0, np.full(n, e.lame_lambda), np.full(n, e.lame_mu),
                                           fbar[None])
    assert st == 0 and reps[0]["passes"] - 1 == 1
    assert np.max(np.abs(F.reshape(9, n) - fbar.reshape(9, 1))) < 1e-12
    assert reps[0]["drift"] < 1e-12


def test_config0_iteration_counts(oracle):
    """BASELINE config 0 at reduced scale is covered on the GPU; here the
    SURVEY §6 scratch counts of config 0 (3 passes, CG 42/52/54) are pinned
    from the committed golden fixture produced by this oracle."""
    path = os.path.join(os.path.dirname(__file__), "golden", "config0.npz")
    if not os.path.exists(path):
        pytest.skip("config0 golden fixture not generated")
    g = np.load(path)
    assert int(g["passes"][0]) == 3
    assert list(g["cg_it"][0][:3]) == [42, 52, 54]
