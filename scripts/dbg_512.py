import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M
from oracle import oracle as O
for pts in [(16, 16, 512), (16, 512, 16), (512, 16, 16), (8, 8, 1024)]:
    A = M.uniform_field(pts, 9, seed=5)
    n = int(np.prod(pts))
    K = np.random.default_rng(2).uniform(-1, 1, 81 * n)
    ref, _, _ = O.apply_projection(pts, 3, A)
    refk, _ = O.apply_projected_tangent(pts, 3, K, A)
    with abi.Context(pts, 3) as ctx:
        g = ctx.projection(ctx.field(9, A)).download()
        gk = ctx.projected_tangent(ctx.field(81, K), ctx.field(9, A)).download()
    print(pts, np.linalg.norm(g - ref) / np.linalg.norm(ref), np.linalg.norm(gk - refk) / np.linalg.norm(refk), flush=True)
N = 512
pg, frac, count = M.random_spheres(N, 12, 0.25, 3)
phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003), M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
lam, mu, ty, h = M.bind_parameters(pg, phases)
ctx = abi.Context((N, N, N), 3)
model = abi.Model(ctx, "simo", lam, mu, ty, h, compact=True)
F = ctx.field(9, abi.identity_field((N, N, N), 3))
A = ctx.field(9, M.uniform_field((N, N, N), 9, seed=1))
GA = ctx.projection(A)
GGA = ctx.projection(GA)
print("512 idempotence", ctx.norm(GGA) , ctx.norm(GA), ctx.dot(GA, GA), flush=True)
try:
    rep = model.solve_increment(F, M.simple_shear_program(0.05, 10, 3)[0], max_newton=8)
    print("ok", rep)
except abi.FmError as e:
    print("FAIL", e, getattr(e, "report", None))
