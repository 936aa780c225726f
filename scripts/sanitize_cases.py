"""Small cases exercising every kernel family, for compute-sanitizer runs."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402

for pts in [(31, 31, 31), (32, 32, 32), (12, 10, 14), (5, 7), (64, 32, 16)]:
    tdim = len(pts)
    n = int(np.prod(pts))
    with abi.Context(pts, tdim) as ctx:
        nc = tdim * tdim
        A = ctx.field(nc, M.uniform_field(pts, nc, 1))
        ctx.projection(A)
        ctx.projected_tangent(ctx.field(nc * nc, np.random.default_rng(0).uniform(-1, 1, nc * nc * n)), A)
        pg = M.corner_cube(pts, 9 if pts == (31, 31, 31) else 3) if tdim == 3 else M.make_laminate(pts, [0.5, 0.5])
        lam, mu, ty, h = M.bind_parameters(pg, [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
                                                M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)])
        fb = M.simple_shear_program(0.01, 2, tdim)
        for kind, mf, cp in [("hyper", False, False), ("hyper", True, False), ("simo", False, False),
                             ("simo", False, True)]:
            if kind == "simo" and pts != (31, 31, 31):
                continue  # the config-1 geometry (9^3 inclusion) converges; see DESIGN.md §7b
            m = abi.Model(ctx, kind, lam, mu, ty, h, matrix_free=mf, compact=cp)
            F = ctx.field(nc, abi.identity_field(pts, tdim))
            abi.run_program(m, F, fb)
            m.close()
        if tdim == 3 and pts[0] % 4 == 0 and pts[1] % 4 == 0:
            ctx.set_virtual_ranks(4)
            ctx.projection(A)
print("sanitize cases done")
