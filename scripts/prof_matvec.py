"""Short matvec driver for ncu captures: N^3 G:K4:dF applications."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1603_08893_b200 import abi
N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
n = N ** 3
ctx = abi.Context((N, N, N), 3)
rng = np.random.default_rng(0)
K = ctx.field(81)
abi.lib().fm_field_fill(ctx.h, K.h, 0.0)
lam = np.full(n, 0.5769); mu = np.full(n, 0.3846)
model = abi.Model(ctx, "hyper", lam, mu, matrix_free=len(sys.argv) > 3 and sys.argv[3] == "mf")
F0 = abi.identity_field((N, N, N), 3); F0[n:2 * n] = 0.1
F = ctx.field(9, F0); P = ctx.field(9)
model.evaluate(F, P)
dF = ctx.field(9, rng.uniform(-1, 1, 9 * n)); out = ctx.field(9)
for _ in range(reps):
    model.apply(dF, out)
ctx.sync()
print("ok", ctx.launches)
