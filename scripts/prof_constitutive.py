"""Times (CUDA events on the library stream) and drives ncu captures of the
constitutive kernels at N^3: k_hyper<3> (SVK P + K4, hyperelastic.cpp:10-65)
and k_simo (J2 P + K4 or compact tangent + trial history, simo.cpp:26-196).
Prints one JSON line: ms per launch and the fraction of the measured HBM peak
on the algorithmic bytes per voxel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
which = sys.argv[3] if len(sys.argv) > 3 else "all"
pts = (N, N, N)
n = N ** 3
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"] if os.path.exists("MEASURED_PEAKS.json") else 6550.1
pg = M.bernoulli(pts, 0.3, 2)
phases = [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
          M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)]
lam, mu, ty, h = M.bind_parameters(pg, phases)
res = {"grid": N}
with abi.Context(pts, 3) as ctx:
    F = ctx.field(9)
    t = torch.as_tensor(F, device="cuda")
    t.uniform_(-0.004, 0.004)  # mixes elastic and plastic voxels for J2
    for i in range(3):
        t[(4 * i) * n:(4 * i + 1) * n] += 1.0
    torch.cuda.synchronize()
    P = ctx.field(9)
    s = torch.cuda.ExternalStream(ctx.stream)

    def timed(fn):
        fn()
        ctx.sync()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(s)
        for _ in range(reps):
            fn()
        b.record(s)
        b.synchronize()
        return a.elapsed_time(b) / reps

    if which in ("all", "hyper"):
        m = abi.Model(ctx, "hyper", lam, mu, matrix_free=False)
        ms = timed(lambda: m.evaluate(F, P))
        res["k_hyper_K4"] = {"ms": ms, "B_per_voxel": 808, "frac": 808 * n / (ms * 1e-3) / 1e9 / peak}
        m.close()
        m = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
        ms = timed(lambda: m.evaluate(F, P))
        res["k_hyper_P_and_F_copy"] = {"ms": ms, "B_per_voxel": 304, "frac": 304 * n / (ms * 1e-3) / 1e9 / peak}
        m.close()
    if which in ("all", "simo"):
        for compact in (False, True):
            m = abi.Model(ctx, "simo", lam, mu, ty, h, compact=compact)
            ms = timed(lambda: m.evaluate(F, P))
            B = 256 + 72 + 72 + 8 + (360 if compact else 648)
            res["k_simo_" + ("compact" if compact else "K4")] = {"ms": ms, "B_per_voxel": B,
                                                                "frac": B * n / (ms * 1e-3) / 1e9 / peak}
            be, ep = m.history(1)
            res["plastic_fraction" + ("_c" if compact else "")] = float(np.mean(ep > 0))
            m.close()
    res["kernels"] = ctx.kernel_names
print(json.dumps(res))
