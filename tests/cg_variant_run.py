"""Helper for test_gpu_solver.py::test_fused_cg_matches_unfused: one config-2
style Newton solve in a fresh process (FM_CG_FUSED / FM_CG_GRAPH are read
once per process); prints the report and a digest of F as JSON."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402

N, kind = int(sys.argv[1]), sys.argv[2]
pg = M.bernoulli((N, N, N), 0.3, 2)
lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
with abi.Context((N, N, N), 3) as ctx:
    model = abi.Model(ctx, "hyper", lam, mu, matrix_free=(kind == "mf"))
    F = ctx.field(9, abi.identity_field((N, N, N), 3))
    fbar = np.eye(3)
    fbar[0, 1] = 0.1
    rep = model.solve_increment(F, fbar)
    f = F.download()
print(json.dumps({"cg": rep["cg_it"], "passes": rep["passes"], "rel": rep["rel_update"],
                  "F_sum": float(f.sum()), "F": f[:: max(1, f.size // 4096)].tolist()}))
