"""1024-point y pass: the cluster form k_y_warp (FM_YW1024=1) against the default
k_y_fast on the same seeded input -- relative difference of G's output and
per-pass times.  python scripts/y1024_check.py NXxNYxNZ [reps]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(shape, reps, out):
    sys.path.insert(0, ROOT)
    import numpy as np
    import torch
    from paper_1603_08893_b200 import abi
    pts = tuple(int(x) for x in shape.split("x"))
    with abi.Context(pts, 3) as ctx:
        f = ctx.field(9)
        g = torch.Generator(device="cuda")
        g.manual_seed(7)
        torch.as_tensor(f, device="cuda").uniform_(-1, 1, generator=g)
        o = ctx.field(9)
        ctx.projection(f, out=o)
        ctx.sync()
        ctx.profile(True)
        for _ in range(reps):
            ctx.projection(f, out=o)
        ms, calls = ctx.profile_read()
        ctx.profile(False)
        res = torch.as_tensor(o, device="cuda")
        # a fixed strided sample of the output (the fields can be tens of GB)
        samp = res[:: max(1, res.numel() // (1 << 22))].cpu().numpy()
        np.save(out, samp)
        print(json.dumps({"shape": shape, "yw1024": os.environ.get("FM_YW1024", "0"),
                          "passes_ms": [round(m / calls, 4) for m in ms], "kernels": ctx.kernel_names}))


if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(sys.argv[2], int(sys.argv[3]), sys.argv[4])
        sys.exit(0)
    import numpy as np
    shape = sys.argv[1]
    reps = sys.argv[2] if len(sys.argv) > 2 else "3"
    outs = []
    for v in ("0", "1"):
        out = f"/tmp/y1024_{v}.npy"
        r = subprocess.run(["timeout", "300", sys.executable, __file__, "child", shape, reps, out],
                           env=dict(os.environ, FM_YW1024=v), capture_output=True, text=True)
        print(r.stdout.strip() or f"rc {r.returncode}: {r.stderr[-600:]}")
        outs.append(np.load(out) if os.path.exists(out) and r.returncode == 0 else None)
        if os.path.exists(out):
            os.remove(out)
    if outs[0] is not None and outs[1] is not None:
        print("relative difference", float(np.linalg.norm(outs[0] - outs[1]) / np.linalg.norm(outs[0])))
