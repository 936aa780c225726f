"""Matrix-free SVK (or, with "k4", materialised-K4) matvec at N^3 (config-2 phases): output checksum and per-pass times
(run under different FM_* switches to A/B pass-1 variants; checksums must agree bitwise)."""
import hashlib
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 256
op = sys.argv[2] if len(sys.argv) > 2 else "svk"  # "k4": materialised SVK tangent, "j2c": compact J2 tangent
mf = op == "svk"
n = N ** 3
pg = M.bernoulli((N, N, N), 0.3, 2)
if op == "j2c":
    lam, mu, ty, hd = M.bind_parameters(pg, [M.PlasticParams(M.ElasticParams(1.0, 0.3), 0.003, 0.003),
                                             M.PlasticParams(M.ElasticParams(2.0, 0.3), 0.006, 0.006)])
else:
    lam, mu, _, _ = M.bind_parameters(pg, [M.ElasticParams(1.0, 0.3), M.ElasticParams(10.0, 0.3)])
with abi.Context((N, N, N), 3) as ctx:
    F0 = abi.identity_field((N, N, N), 3)
    F0[n:2 * n] = 0.1
    F, P, dF, out = ctx.field(9, F0), ctx.field(9), ctx.field(9), ctx.field(9)
    torch.manual_seed(0)
    torch.as_tensor(dF, device="cuda").uniform_(-1, 1)
    model = (abi.Model(ctx, "simo", lam, mu, ty, hd, compact=True) if op == "j2c"
             else abi.Model(ctx, "hyper", lam, mu, matrix_free=mf))
    model.evaluate(F, P)
    model.apply(dF, out)
    ctx.sync()
    h = hashlib.sha1(torch.as_tensor(out, device="cuda").cpu().numpy().tobytes()).hexdigest()[:16]
    ctx.profile(True)
    for _ in range(20):
        model.apply(dF, out)
    ms, calls = ctx.profile_read()
    ctx.profile(False)
    per = [round(m / calls, 4) for m in ms]
    model.close()
print(json.dumps({"N": N, "operator": op, "env": {k: v for k, v in os.environ.items() if k.startswith("FM_")}, "sha1": h,
                  "passes_ms": per, "ms": round(sum(per), 4)}))
