import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np
from paper_1603_08893_b200 import abi
for pts in [(6, 5, 4), (4, 3, 5), (4, 4, 4), (6, 6, 6)]:
    n = int(np.prod(pts))
    ctx = abi.Context(pts, 3)
    m = abi.Model(ctx, "hyper", np.full(n, 0.5769), np.full(n, 0.3846))
    F = ctx.field(9, abi.identity_field(pts, 3))
    fb = np.eye(3); fb[0, 1] = 0.1
    try:
        rep = m.solve_increment(F, fb)
        print(pts, "ok", rep["cg_it"], rep["rel_update"])
    except abi.FmError as e:
        Fh = F.download().reshape(9, n)
        print(pts, "FAIL", e, getattr(e, "report", None))
        print(" F node0", Fh[:, 0], "\n F node1", Fh[:, 1])
    m.close(); ctx.close()
