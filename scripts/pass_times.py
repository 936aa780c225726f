"""Per-pass CUDA-event times of G (config 4 input) and of the matrix-free SVK
matvec at N^3 (in place for G when --inplace); JSON per N."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402

hbm = 6540.0
try:
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"]
except Exception:
    pass
for N in [int(a) for a in sys.argv[1:]]:
    n = N ** 3
    res = {"N": N}
    with abi.Context((N, N, N), 3) as ctx:
        f = ctx.field(9)
        v = torch.as_tensor(f, device="cuda")
        v.uniform_(-1, 1)
        torch.cuda.synchronize()
        out = f if N >= 1024 else ctx.field(9)
        reps = 3 if N >= 1024 else 10
        ctx.projection(f, out=out)
        ctx.sync()
        ctx.profile(True)
        for _ in range(reps):
            ctx.projection(f, out=out)
        ms, calls = ctx.profile_read()
        ctx.profile(False)
        per = [m / calls for m in ms]
        res["G_passes_ms"] = [round(x, 4) for x in per]
        res["G_ms"] = round(sum(per), 4)
        res["G_frac"] = round(720 * n / (sum(per) * 1e-3) / 1e9 / hbm, 4)
        res["G_pass_frac"] = [round(144 * n / (x * 1e-3) / 1e9 / hbm, 3) for x in per]
        if N <= 512:
            lam = np.full(n, 0.5769)
            mu = np.full(n, 0.3846)
            model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
            F0 = abi.identity_field((N, N, N), 3)
            F0[n:2 * n] = 0.1
            F = ctx.field(9, F0)
            P = ctx.field(9)
            model.evaluate(F, P)
            model.apply(f, out)
            ctx.sync()
            ctx.profile(True)
            for _ in range(reps):
                model.apply(f, out)
            ms, calls = ctx.profile_read()
            ctx.profile(False)
            per = [m / calls for m in ms]
            res["mv_svk_passes_ms"] = [round(x, 4) for x in per]
            res["mv_svk_ms"] = round(sum(per), 4)
            res["mv_svk_frac808"] = round(808 * n / (sum(per) * 1e-3) / 1e9 / hbm, 4)
            model.close()
    print(json.dumps(res), flush=True)
