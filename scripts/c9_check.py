"""Acceptance criterion 9 input (45x45 speckle micrograph, Simo, pure shear to
1.2 in 50 increments) for each contrast chi: GPU vs CPU oracle outcome."""
import math
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1603_08893_b200 import microstructure as M  # noqa: E402


def micrograph():
    n = 45
    modes = [(1, 2), (3, 1), (2, 4), (5, 2), (4, 5), (6, 1), (2, 6), (5, 5)]
    amps = [1.0, 0.8, 0.7, 0.55, 0.5, 0.4, 0.35, 0.3]
    phs = [0.3, 1.7, 2.9, 4.1, 5.3, 0.9, 2.2, 3.6]
    v = np.zeros((n, n))
    for iy in range(n):
        for ix in range(n):
            v[iy, ix] = sum(a * math.cos(2 * math.pi * (mx * ix + my * iy) / n + p)
                            for (mx, my), a, p in zip(modes, amps, phs))
    s = np.sort(v.reshape(-1))
    cut, lo, hi = s[s.size * 30 // 100], s[0], s[-1]
    pix = np.array([[int(math.floor(255.0 * (x - lo) / (hi - lo) + 0.5)) for x in row] for row in v])
    thr = math.floor(255.0 * (cut - lo) / (hi - lo))
    labels = np.zeros(n * n, dtype=np.int32)
    for iy in range(n):
        for ix in range(n):
            labels[ix * n + iy] = 1 if pix[iy, ix] <= thr else 0  # node = ix * Ny + iy
    return M.PhaseGrid((n, n), labels, 2)


def program(incs=50):
    out = np.zeros((incs, 3, 3))
    for t in range(1, incs + 1):
        lam = 1.0 + 0.2 * t / incs
        out[t - 1] = np.diag([lam, 1.0 / lam, 1.0])
    return out


if __name__ == "__main__":
    which = sys.argv[1]
    chis = [float(eval(c)) for c in sys.argv[2:]] or [math.sqrt(2.0), 2.0, 4.0, 8.0]
    pg = micrograph()
    prog = program()
    for chi in chis:
        soft = M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.01)
        hard = M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003 * chi, 0.01 * chi)
        lam, mu, ty, h = M.bind_parameters(pg, [soft, hard])
        if which == "oracle":
            from oracle import oracle as O
            _, _, reps, st, _ = O.run_program((45, 45), 3, 1, lam, mu, prog, ty0=ty, hard=h)
            print("oracle chi", chi, "status", st, "incs", len(reps), "newton", sum(r["passes"] for r in reps),
                  "cg", sum(sum(r["cg_it"]) for r in reps), flush=True)
        else:
            from paper_1603_08893_b200 import abi
            with abi.Context((45, 45), 3) as ctx:
                m = abi.Model(ctx, "simo", lam, mu, ty, h)
                F = ctx.field(9, abi.identity_field((45, 45), 3))
                reps = []
                st = 0
                try:
                    for fb in prog:
                        reps.append(m.solve_increment(F, fb))
                except abi.FmError as e:
                    st = e.status
                print("gpu chi", chi, "status", st, "incs", len(reps), "newton", sum(r["passes"] for r in reps),
                      "cg", sum(sum(r["cg_it"]) for r in reps), flush=True)
