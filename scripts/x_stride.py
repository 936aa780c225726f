"""Does the x pass depend on the x stride (TLB reach) or only on the line
length?  Per-pass CUDA-event times of G at several (Nx, Ny, Nz) shapes with
the same line length but different x strides; one JSON line per shape."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch
from paper_1603_08893_b200 import abi

hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.1
shapes = [tuple(int(x) for x in s.split("x")) for s in sys.argv[1].split(",")]
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 10
for pts in shapes:
    n = pts[0] * pts[1] * pts[2]
    with abi.Context(pts, 3) as ctx:
        f = ctx.field(9)
        g = torch.Generator(device="cuda")
        g.manual_seed(1234)
        torch.as_tensor(f, device="cuda").uniform_(-1, 1, generator=g)
        torch.cuda.synchronize()
        out = ctx.field(9)
        ctx.projection(f, out=out)
        ctx.sync()
        ctx.profile(True)
        for _ in range(reps):
            ctx.projection(f, out=out)
        ms, calls = ctx.profile_read()
        ctx.profile(False)
        per = [m / calls for m in ms]
        fr = [round(144 * n / (p * 1e-3) / 1e9 / hbm, 3) for p in per]
        print(json.dumps({"pts": pts, "xstride_KB": pts[1] * (pts[2] // 2) * 16 / 1024, "mode": os.environ.get("FM_XDIRECT"),
                          "passes_ms": [round(x, 4) for x in per], "pass_frac": fr,
                          "kernels": ctx.kernel_names}), flush=True)
    torch.cuda.empty_cache()
