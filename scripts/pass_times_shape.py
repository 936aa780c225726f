"""Per-pass CUDA-event times of G on an (Nx, Ny, Nz) grid: isolates the x-pass
cost of the line length (Nx) from that of the row stride (Ny * Nz / 2 * 16 B)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402

hbm = 6540.0
for arg in sys.argv[1:]:
    pts = tuple(int(v) for v in arg.split("x"))
    n = pts[0] * pts[1] * pts[2]
    with abi.Context(pts, 3) as ctx:
        f = ctx.field(9)
        torch.as_tensor(f, device="cuda").uniform_(-1, 1)
        torch.cuda.synchronize()
        out = ctx.field(9)
        ctx.projection(f, out=out)
        ctx.sync()
        ctx.profile(True)
        for _ in range(10):
            ctx.projection(f, out=out)
        ms, calls = ctx.profile_read()
    per = [m / calls for m in ms]
    print(json.dumps({"grid": arg, "passes_ms": [round(x, 4) for x in per],
                      "pass_frac": [round(144 * n / (x * 1e-3) / 1e9 / hbm, 3) for x in per],
                      "xstride_KB": pts[1] * pts[2] // 2 * 16 // 1024}), flush=True)
