"""Config-2 Newton solve (256^3 SVK Bernoulli) through the C ABI, for profiling."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M
N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
mf = len(sys.argv) > 2 and sys.argv[2] == "mf"
pg = M.bernoulli((N, N, N), 0.3, 2)
lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
ctx = abi.Context((N, N, N), 3)
model = abi.Model(ctx, "hyper", lam, mu, matrix_free=mf)
F = ctx.field(9, abi.identity_field((N, N, N), 3))
fbar = np.eye(3); fbar[0, 1] = 0.1
t = time.perf_counter()
rep = model.solve_increment(F, fbar)
print("solve", time.perf_counter() - t, rep["cg_it"], rep["matvecs"], "launches", ctx.launches)
print("rel_update", rep.get("rel_update"), "F checksum", repr(float(np.sum(F.download()))))
