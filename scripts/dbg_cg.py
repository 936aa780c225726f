import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1603_08893_b200 import abi
from oracle import oracle as O
pts = (6, 6, 6); n = 216
lam, mu = np.full(n, 0.5769), np.full(n, 0.3846)
fb = np.eye(3); fb[0, 1] = 0.1
Fb = np.repeat(fb.reshape(9, 1), n, axis=1).reshape(-1)
P, K, _, _ = O.hyper_evaluate(Fb, lam, mu)
ctx = abi.Context(pts, 3)
fk = ctx.field(81, K)
u = np.repeat((fb - np.eye(3)).reshape(9, 1), n, axis=1).reshape(-1)
rhs = -ctx.projected_tangent(fk, ctx.field(9, u)).download()
print("|rhs|", np.linalg.norm(rhs))
g = ctx.projection(ctx.field(9, rhs)).download()
print("compat |G rhs - rhs|", np.linalg.norm(g - rhs))
rng = np.random.default_rng(0)
for scale in [1.0, 1e-10, 1e-17, 1e-20]:
    b = ctx.projection(ctx.field(9, scale * rng.uniform(-1, 1, 9 * n))).download()
    try:
        x, it, rel = ctx.cg_solve(fk, ctx.field(9, b))
        xr, itr, relr, st = O.cg_solve(pts, 3, K, b)
        print(scale, "gpu", it, rel, "oracle", itr, relr, st)
    except abi.FmError as e:
        print(scale, "gpu FAIL", e)
x = ctx.field(9, ctx.projection(ctx.field(9, rng.uniform(-1, 1, 9 * n))).download())
y = ctx.field(9, ctx.projection(ctx.field(9, rng.uniform(-1, 1, 9 * n))).download())
Ax = ctx.projected_tangent(fk, x); Ay = ctx.projected_tangent(fk, y)
print("sym", ctx.dot(x, Ay), ctx.dot(Ax, y))
try:
    xx, it, rel = ctx.cg_solve(fk, ctx.field(9, rhs))
    print("noise rhs gpu", it, rel)
except abi.FmError as e:
    print("noise rhs FAIL", e)
xr, itr, relr, st = O.cg_solve(pts, 3, K, rhs)
print("noise rhs oracle", itr, relr, st)
