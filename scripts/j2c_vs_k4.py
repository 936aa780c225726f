import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M
for pts in [(16, 16, 512), (16, 16, 256), (8, 8, 1024)]:
    n = int(np.prod(pts))
    rng = np.random.default_rng(0)
    lam = np.full(n, 0.5769); mu = np.full(n, 0.3846); ty = np.full(n, 0.003); h = np.full(n, 0.003)
    F0 = abi.identity_field(pts, 3) + rng.uniform(-0.02, 0.02, 9 * n)
    dF = rng.uniform(-1, 1, 9 * n)
    outs = []
    for compact in (False, True):
        with abi.Context(pts, 3) as ctx:
            m = abi.Model(ctx, "simo", lam, mu, ty, h, compact=compact)
            F = ctx.field(9, F0); P = ctx.field(9)
            m.evaluate(F, P)
            outs.append(m.apply(ctx.field(9, dF), ctx.field(9)).download())
            m.close()
    print(pts, np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[0]), flush=True)
N = 512
pg, frac, count = M.random_spheres(N, 12, 0.25, 3)
lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(2.0, 0.3)])
ctx = abi.Context((N, N, N), 3)
model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
F = ctx.field(9, abi.identity_field((N, N, N), 3))
rep = model.solve_increment(F, M.simple_shear_program(0.05, 10, 3)[0])
print("svk512", rep["passes"], rep["cg_it"], rep["rel_update"], flush=True)
