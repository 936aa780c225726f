"""Config-2 Newton solve with per-pass CUDA-event timing of every projection
application (fused CG iteration: pass 1 carries the direction/x update and
curvature, pass 5 the residual update)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
pg = M.bernoulli((N, N, N), 0.3, 2)
lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
fbar = np.eye(3)
fbar[0, 1] = 0.1
with abi.Context((N, N, N), 3) as ctx:
    for prof in (False, True):
        model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
        F = ctx.field(9, abi.identity_field((N, N, N), 3))
        ctx.sync()
        if prof:
            ctx.profile(True)
        t = time.perf_counter()
        rep = model.solve_increment(F, fbar)
        ctx.sync()
        wall = time.perf_counter() - t
        out = {"profiled": prof, "wall_s": wall, "device_s": rep["wall"], "cg": rep["cg_it"], "matvecs": rep["matvecs"]}
        if prof:
            ms, calls = ctx.profile_read()
            ctx.profile(False)
            out["passes_ms_per_call"] = [round(m / calls, 4) for m in ms]
            out["calls"] = calls
        print(json.dumps(out), flush=True)
        model.close()
