"""Virtual-rank timing of the transpose-fused slab decomposition on one B200:
the matrix-free SVK matvec at N^3 with P = 1, 2, 4, 8 slab ranks emulated on
the device.  The routed stores of the forward y pass and the x pass then go
to the other ranks' buffers in the same HBM, so the per-pass times show what
the fused transpose costs the kernels themselves (no NVLink in the loop);
also checks the result is bit-for-bit the P = 1 result."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
n = N ** 3
rng = np.random.default_rng(0)
lam = np.where(rng.uniform(size=n) < 0.3, 5.769, 0.5769)
mu = lam * (0.3846 / 0.5769)
F0 = abi.identity_field((N, N, N), 3)
F0[n:2 * n] = 0.1
dF0 = rng.uniform(-1, 1, 9 * n)
res = {}
ref = None
for P in (1, 2, 4, 8):
    with abi.Context((N, N, N), 3) as ctx:
        if P > 1:
            ctx.set_virtual_ranks(P)
        model = abi.Model(ctx, "hyper", lam, mu, matrix_free=True)
        F = ctx.field(9, F0)
        Pf = ctx.field(9)
        model.evaluate(F, Pf)
        dF = ctx.field(9, dF0)
        out = ctx.field(9)
        model.apply(dF, out)
        ctx.sync()
        got = out.download()
        if ref is None:
            ref = got
        ctx.profile(True)
        for _ in range(reps):
            model.apply(dF, out)
        ctx.sync()
        ms, calls = ctx.profile_read()
        ctx.profile(False)
        per = [m / calls for m in ms]
        res[P] = {"passes_ms": [round(x, 4) for x in per], "matvec_ms": round(sum(per), 4),
                  "bitwise_equal_P1": bool(np.array_equal(got, ref))}
        model.close()
    print(P, json.dumps(res[P]), flush=True)
print(json.dumps({"N": N, "virtual_ranks": res}))
