"""512-point x pass check: G and G:K4:dF against the CPU oracle on thin 512-line
grids, virtual-rank bitwise equality, and per-pass times at 512^3.
Run with FM_XDIRECT=0/1 to compare the two 512-point x passes."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from oracle import oracle as O  # noqa: E402
from paper_1603_08893_b200 import abi  # noqa: E402
from paper_1603_08893_b200 import microstructure as M  # noqa: E402

res = {"FM_XDIRECT": os.environ.get("FM_XDIRECT", "1")}
for pts in [(512, 8, 16), (512, 6, 24), (512, 4, 32)]:
    n = int(np.prod(pts))
    A = M.uniform_field(pts, 9, seed=11)
    with abi.Context(pts, 3) as ctx:
        g = ctx.projection(ctx.field(9, A)).download()
    ref, st, _ = O.apply_projection(pts, 3, A)
    res[str(pts)] = float(np.linalg.norm(g - ref) / np.linalg.norm(ref))
pts = (512, 16, 16)
A = M.uniform_field(pts, 9, seed=12)
with abi.Context(pts, 3) as ctx:
    g1 = ctx.projection(ctx.field(9, A)).download()
for P in (2, 4):
    with abi.Context(pts, 3) as ctx:
        ctx.set_virtual_ranks(P)
        gP = ctx.projection(ctx.field(9, A)).download()
    res[f"virtual_P{P}_bitwise"] = bool(np.array_equal(g1, gP))
N = 512
n = N ** 3
with abi.Context((N, N, N), 3) as ctx:
    f = ctx.field(9)
    torch.as_tensor(f, device="cuda").uniform_(-1, 1)
    torch.cuda.synchronize()
    out, out2 = ctx.field(9), ctx.field(9)
    ctx.projection(f, out=out)
    ctx.projection(out, out=out2)
    a, b = torch.as_tensor(out, device="cuda"), torch.as_tensor(out2, device="cuda")
    res["idempotence_512"] = float((a - b).norm() / a.norm())
    ctx.sync()
    ctx.profile(True)
    for _ in range(10):
        ctx.projection(f, out=out)
    ms, calls = ctx.profile_read()
    ctx.profile(False)
    res["G_passes_ms"] = [round(m / calls, 4) for m in ms]
    res["G_ms"] = round(sum(res["G_passes_ms"]), 4)
print(json.dumps(res), flush=True)
