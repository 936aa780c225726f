"""Generates the committed golden fixtures of BASELINE.json configs 0 and 1
(31^3) with the CPU oracle (oracle/, restating the reference solver).  The
oracle is itself pinned to the reference's golden run records (see
tests/test_oracle_pins.py).  Run: python tests/golden/make_golden.py [0] [1]"""
import os
import sys
import time

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))
from oracle import oracle as O  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402


def config0():
    pts = (31, 31, 31)
    pg = M.corner_cube(pts, 9)
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
    t = time.time()
    F, P, reps, st, _ = O.run_program(pts, 3, 0, lam, mu, M.simple_shear_program(0.1, 1, 3))
    assert st == 0, st
    np.savez_compressed(os.path.join(HERE, "config0.npz"), F=F, P=P,
                        passes=np.array([r["passes"] for r in reps]),
                        cg_it=np.array([r["cg_it"] + [0] * (64 - len(r["cg_it"])) for r in reps]),
                        rel_update=np.array([r["rel_update"] + [0.0] * (64 - len(r["rel_update"])) for r in reps]),
                        eq_rel=np.array([r["eq_rel"] for r in reps]))
    print("config0", time.time() - t, [r["cg_it"] for r in reps])


def config1():
    pts = (31, 31, 31)
    pg = M.corner_cube(pts, 9)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    t = time.time()
    F, P, reps, st, epsp = O.run_program(pts, 3, 1, lam, mu, M.simple_shear_program(0.1, 20, 3),
                                         ty0=ty, hard=h)
    assert st == 0, st
    np.savez_compressed(os.path.join(HERE, "config1.npz"), F=F, P=P, epsp=epsp,
                        passes=np.array([r["passes"] for r in reps]),
                        cg_it=np.array([r["cg_it"] + [0] * (64 - len(r["cg_it"])) for r in reps]),
                        rel_update=np.array([r["rel_update"] + [0.0] * (64 - len(r["rel_update"])) for r in reps]),
                        eq_rel=np.array([r["eq_rel"] for r in reps]))
    print("config1", time.time() - t, [r["cg_it"] for r in reps])


def config1_band(eps):
    """CG-count sensitivity band of config 1: the oracle re-run with lambda
    scaled by (1 + eps), eps = +-1e-15.  Config 1's J2 passes take ~100-300
    CG iterations, and a 1e-15 relative perturbation alone moves their counts
    by several iterations; GPU counts are checked against this band."""
    pts = (31, 31, 31)
    pg = M.corner_cube(pts, 9)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    _, _, reps, st, _ = O.run_program(pts, 3, 1, lam * (1.0 + eps), mu,
                                      M.simple_shear_program(0.1, 20, 3), ty0=ty, hard=h)
    assert st == 0, st
    tag = "p" if eps > 0 else "m"
    np.savez_compressed(os.path.join(HERE, f"config1_band_{tag}.npz"),
                        passes=np.array([r["passes"] for r in reps]),
                        cg_it=np.array([r["cg_it"] + [0] * (64 - len(r["cg_it"])) for r in reps]))
    print("band", eps, [r["cg_it"] for r in reps])


PERTURB = [("lam", 1e-15), ("lam", -1e-15), ("mu", 1e-15), ("mu", -1e-15), ("lam", 3e-16), ("mu", -3e-16)]


def _simo16_run(args):
    which, eps = args
    pts = (16, 16, 16)
    pg = M.corner_cube(pts, 3)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    if which == "lam":
        lam = lam * (1.0 + eps)
    elif which == "mu":
        mu = mu * (1.0 + eps)
    return O.run_program(pts, 3, 1, lam, mu, M.simple_shear_program(0.02, 4, 3), ty0=ty, hard=h)


def simo16():
    """16^3 J2 case of tests/test_gpu_solver.py: the oracle run plus its
    CG-count envelope under six 1e-15-level perturbations of lambda / mu."""
    from multiprocessing import Pool
    with Pool(7) as pool:
        runs = pool.map(_simo16_run, [("none", 0.0)] + PERTURB)
    F, P, reps, st, epsp = runs[0]
    assert st == 0
    pad = lambda r: r["cg_it"] + [0] * (64 - len(r["cg_it"]))
    np.savez_compressed(os.path.join(HERE, "simo16.npz"), F=F, P=P, epsp=epsp,
                        passes=np.array([r["passes"] for r in reps]),
                        cg_it=np.array([pad(r) for r in reps]),
                        band_passes=np.array([[r["passes"] for r in run[2]] for run in runs[1:]]),
                        band_cg_it=np.array([[pad(r) for r in run[2]] for run in runs[1:]]))
    print("simo16", [r["cg_it"] for r in reps], [[r["cg_it"] for r in run[2]] for run in runs[1:]])


def _simo32_run(args):
    which, eps = args
    pts = (32, 32, 32)
    pg = M.corner_cube(pts, 8)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    if which == "lam":
        lam = lam * (1.0 + eps)
    elif which == "mu":
        mu = mu * (1.0 + eps)
    return O.run_program(pts, 3, 1, lam, mu, M.simple_shear_program(0.01, 2, 3), ty0=ty, hard=h)


def simo32():
    """32^3 J2 case (power-of-two grid: the register-resident passes, fused CG,
    compact tangent) of tests/test_gpu_solver.py, with its CG-count envelope."""
    from multiprocessing import Pool
    with Pool(7) as pool:
        runs = pool.map(_simo32_run, [("none", 0.0)] + PERTURB)
    F, P, reps, st, epsp = runs[0]
    assert st == 0
    pad = lambda r: r["cg_it"] + [0] * (64 - len(r["cg_it"]))
    np.savez_compressed(os.path.join(HERE, "simo32.npz"), F=F, P=P, epsp=epsp,
                        passes=np.array([r["passes"] for r in reps]),
                        cg_it=np.array([pad(r) for r in reps]),
                        band_passes=np.array([[r["passes"] for r in run[2]] for run in runs[1:]]),
                        band_cg_it=np.array([[pad(r) for r in run[2]] for run in runs[1:]]))
    print("simo32", [r["cg_it"] for r in reps], [[r["cg_it"] for r in run[2]] for run in runs[1:]])


if __name__ == "__main__":
    which = sys.argv[1:] or ["0", "1"]
    if "simo32" in which:
        simo32()
    if "simo16" in which:
        simo16()
    if "band+" in which:
        config1_band(1e-15)
    if "band-" in which:
        config1_band(-1e-15)
    if "0" in which:
        config0()
    if "1" in which:
        config1()


def config3_reduced():
    """Config 3's generator on a reduced grid (64^3, radius 2, seed 3, 10
    increments to gamma 0.05), first two increments.  The oracle (like the
    GPU) converges increment 1 and stops with InvertedElement in increment 2
    (DESIGN.md §7b); the run records are kept as the parity fixture."""
    import json
    N, r = 64, 2
    pg, frac, count = M.random_spheres(N, r, 0.25, 3)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    t = time.time()
    _, _, reps, st, _ = O.run_program((N, N, N), 3, 1, lam, mu, M.simple_shear_program(0.05, 10, 3)[:2],
                                      ty0=ty, hard=h)
    rec = {"grid": N, "radius": r, "fraction": frac, "spheres": count, "status": st,
           "increments": [{"passes": rr["passes"], "status": rr["status"], "cg_it": rr["cg_it"],
                           "err_node": rr["err_node"], "converged": rr["converged"]} for rr in reps if rr["passes"]]}
    with open(os.path.join(HERE, "config3_64.json"), "w") as f:
        json.dump(rec, f, indent=1)
    print("config3_64", time.time() - t, rec)


def _config3_64_run(args):
    which, eps = args
    O.set_threads(1)
    N, r = 64, 2
    pg, _, _ = M.random_spheres(N, r, 0.25, 3)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    if which == "lam":
        lam = lam * (1.0 + eps)
    elif which == "mu":
        mu = mu * (1.0 + eps)
    _, _, reps, st, _ = O.run_program((N, N, N), 3, 1, lam, mu, M.simple_shear_program(0.05, 10, 3)[:1],
                                      ty0=ty, hard=h)
    return st, reps[0]["passes"], reps[0]["cg_it"]


def config3_64_band():
    """The oracle's own CG counts of config3_64's increment 1 under four 1e-15
    relative perturbations of lambda / mu, added to config3_64.json as
    `band`: the envelope tests/test_gpu_config3_reduced.py allows on top of
    BASELINE's +-1 is measured on the case itself."""
    import json
    from multiprocessing import Pool
    with Pool(4) as pool:
        runs = pool.map(_config3_64_run, PERTURB[:4])
    path = os.path.join(HERE, "config3_64.json")
    rec = json.load(open(path))
    rec["band"] = [{"perturb": list(pw), "status": st, "passes": npass, "cg_it": cg}
                   for pw, (st, npass, cg) in zip(PERTURB[:4], runs)]
    with open(path, "w") as f:
        json.dump(rec, f, indent=1)
    print("config3_64 band", rec["band"])


if __name__ == "__main__" and "config3" in sys.argv[1:]:
    config3_reduced()
if __name__ == "__main__" and "config3_64_band" in sys.argv[1:]:
    config3_64_band()


# ---------------------------------------------------------------------------
# Large-grid fixtures (BASELINE configs 2 and 3): too big to commit whole, so
# the fixture holds the run record, full-field norms and checksums, and 2^18
# fixed (component, node) samples of each field (tests/golden_util.py).
# The oracle runs threaded here (bit-identical to one thread, see
# oracle/fftmech_oracle.cpp par_for).
NSAMP = 1 << 18


def _record(reps):
    pad = lambda v, z: list(v) + [z] * (64 - len(v))
    return dict(passes=np.array([r["passes"] for r in reps]),
                cg_it=np.array([pad(r["cg_it"], 0) for r in reps]),
                cg_rel=np.array([pad(r["cg_rel"], 0.0) for r in reps]),
                rel_update=np.array([pad(r["rel_update"], 0.0) for r in reps]),
                eq_rel=np.array([r["eq_rel"] for r in reps]),
                drift=np.array([r["drift"] for r in reps]),
                wall=np.array([r["wall"] for r in reps]))


def _fields(prefix, x, ncomp):
    from golden_util import checksums, sample_index
    idx = sample_index(min(NSAMP, x.size), x.size)
    return {f"{prefix}_samp": x[idx], f"{prefix}_norm": np.linalg.norm(x),
            f"{prefix}_sums": checksums(x, ncomp)}


def config2():
    """BASELINE config 2: 256^3 SVK, Bernoulli(0.3) from mt19937_64(2),
    contrast 10, F_bar = I + 0.1 e_x e_y, one increment (~30 GB, ~40 min on 8
    threads)."""
    O.set_threads()
    pts = (256, 256, 256)
    pg = M.bernoulli(pts, 0.3, 2)
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
    t = time.time()
    F, P, reps, st, _ = O.run_program(pts, 3, 0, lam, mu, M.simple_shear_program(0.1, 1, 3))
    assert st == 0, st
    out = _record(reps)
    out.update(_fields("F", F, 9))
    out.update(_fields("P", P, 9))
    np.savez_compressed(os.path.join(HERE, "config2.npz"), **out)
    print("config2", time.time() - t, [r["cg_it"] for r in reps], [r["rel_update"] for r in reps])


def matvec256():
    """One config-2 matvec at 256^3 in the reference operator form: K4 from
    hyperelastic_evaluate at F = I + 0.05 U(-1,1) (seed 41), dF = U(-1,1)
    (seed 42), out = G(K4 : dF^T) (projection.cpp:173-194)."""
    O.set_threads()
    pts = (256, 256, 256)
    pg = M.bernoulli(pts, 0.3, 2)
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
    n = 256 ** 3
    F = 0.05 * M.uniform_field(pts, 9, 41)
    for i in range(3):
        F[(4 * i) * n:(4 * i + 1) * n] += 1.0
    dF = M.uniform_field(pts, 9, 42)
    t = time.time()
    P, K, st, bad = O.hyper_evaluate(F, lam, mu)
    assert st == 0
    del F
    out, st = O.apply_projected_tangent(pts, 3, K, dF)
    assert st == 0
    res = {}
    res.update(_fields("P", P, 9))
    res.update(_fields("out", out, 9))
    np.savez_compressed(os.path.join(HERE, "matvec256.npz"), **res)
    print("matvec256", time.time() - t, res["out_norm"])


def _config3_128_run(args):
    which, eps = args[0], args[1]
    O.set_threads(args[2] if len(args) > 2 else 1)
    N, r = 128, 3
    pg, frac, count = M.random_spheres(N, r, 0.25, 3)
    phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
              M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
    lam, mu, ty, h = M.bind_parameters(pg, phases)
    if which == "lam":
        lam = lam * (1.0 + eps)
    elif which == "mu":
        mu = mu * (1.0 + eps)
    t = time.time()
    F, P, reps, st, epsp = O.run_program((N, N, N), 3, 1, lam, mu, M.simple_shear_program(0.05, 10, 3)[:1],
                                         ty0=ty, hard=h)
    print("config3_128", which, eps, time.time() - t, st, [r["cg_it"] for r in reps], flush=True)
    return F, P, reps, st, epsp, frac, count


def config3_128():
    """Config 3's generator at 128^3 (radius 3 = 12 * 128 / 512, seed 3,
    gamma 0.05 in 10 increments), increment 1: the run record, sampled F, P
    and eps_p, and the CG-count envelope of the oracle itself under four
    1e-15 relative perturbations of lambda / mu (run side by side)."""
    from multiprocessing import Pool
    jobs = [("none", 0.0, 4)] + [(w, e, 1) for w, e in PERTURB[:4]]
    with Pool(len(jobs)) as pool:
        runs = pool.map(_config3_128_run, jobs)
    F, P, reps, st, epsp, frac, count = runs[0]
    assert st == 0, st
    out = _record(reps)
    out.update(_fields("F", F, 9))
    out.update(_fields("P", P, 9))
    out.update(_fields("epsp", epsp, 1))
    pad = lambda r: r["cg_it"] + [0] * (64 - len(r["cg_it"]))
    out.update(fraction=frac, spheres=count,
               band_status=np.array([run[3] for run in runs[1:]]),
               band_passes=np.array([[r["passes"] for r in run[2]] for run in runs[1:]]),
               band_cg_it=np.array([[pad(r) for r in run[2]] for run in runs[1:]]))
    np.savez_compressed(os.path.join(HERE, "config3_128.npz"), **out)
    print("config3_128 band", [[r["cg_it"] for r in run[2]] for run in runs])


def _proj(N):
    """BASELINE config 4: G applied to a seeded i.i.d. U(-1,1) 3x3 tensor field
    (projection.cpp:123-171) at N^3; samples, norm and checksums of the output."""
    O.set_threads()
    pts = (N, N, N)
    A = M.uniform_field(pts, 9, 4)
    t = time.time()
    out, st, _ = O.apply_projection(pts, 3, A)
    assert st == 0
    del A
    res = _fields("out", out, 9)
    np.savez_compressed(os.path.join(HERE, f"proj{N}.npz"), **res)
    print(f"proj{N}", time.time() - t, res["out_norm"])


def proj256():
    _proj(256)  # (512^3 needs more than the 62 GB of this container: the oracle keeps ghat and a complex copy)


if __name__ == "__main__":
    sys.path.insert(0, os.path.dirname(HERE))
    for w in sys.argv[1:]:
        if w in ("config2", "matvec256", "config3_128", "proj256"):
            globals()[w]()
