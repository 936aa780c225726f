import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M
pts = (31, 31, 31)
pg = M.corner_cube(pts, 9)
lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
ctx = abi.Context(pts, 3)
model = abi.Model(ctx, "hyper", lam, mu)
F = ctx.field(9, abi.identity_field(pts, 3))
rep = model.solve_increment(F, M.simple_shear_program(0.1, 1, 3)[0])
print(rep["cg_it"])
import hashlib, time
t = time.perf_counter()
F2 = ctx.field(9, abi.identity_field(pts, 3))
rep = model.solve_increment(F2, M.simple_shear_program(0.1, 1, 3)[0])
print("second solve", time.perf_counter() - t, "F sha1", hashlib.sha1(F2.download().tobytes()).hexdigest()[:16])
