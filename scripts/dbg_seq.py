import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1603_08893_b200 import abi
from paper_1603_08893_b200 import microstructure as M
pts = (31, 31, 31)
with abi.Context(pts, 3) as ctx:
    pg = M.corner_cube(pts, 3)
    lam, mu, ty, h = M.bind_parameters(pg, [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
                                            M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)])
    fb = M.simple_shear_program(0.02, 2, 3)
    for kind, mf, cp in [("hyper", False, False), ("hyper", True, False), ("simo", False, False), ("simo", False, True)]:
        m = abi.Model(ctx, kind, lam, mu, ty, h, matrix_free=mf, compact=cp)
        F = ctx.field(9, abi.identity_field(pts, 3))
        try:
            reps = abi.run_program(m, F, fb)
            print(kind, mf, cp, [r["cg_it"] for r in reps], flush=True)
        except abi.FmError as e:
            print(kind, mf, cp, "FAIL", e, getattr(e, "report", None), flush=True)
        m.close()
        F.free()
