"""Per-pass CUDA-event times of G with P virtual ranks on one device (what the
routing costs the kernels themselves; all stores land in the same HBM):
python scripts/dist_virtual_passes.py N P[,P...] [reps]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402

N = int(sys.argv[1])
Ps = [int(p) for p in sys.argv[2].split(",")]
reps = int(sys.argv[3]) if len(sys.argv) > 3 else 5
with abi.Context((N, N, N), 3) as ctx:
    f = ctx.field(9)
    torch.as_tensor(f, device="cuda").uniform_(-1, 1)
    out = ctx.field(9)
    for P in Ps:
        for tr in ((0,) if P == 1 else (0, 1)):
            ctx.set_transpose(tr)
            ctx.set_virtual_ranks(P)
            ctx.projection(f, out=out)
            ctx.sync()
            ctx.profile(True)
            for _ in range(reps):
                ctx.projection(f, out=out)
            ms, calls = ctx.profile_read()
            ctx.profile(False)
            print(json.dumps({"N": N, "P": P, "transposes": "staged" if tr else "fused",
                              "passes_ms": [round(m / calls, 3) for m in ms], "G_ms": round(sum(ms) / calls, 3),
                              "kernels": ctx.kernel_names}), flush=True)
        ctx.set_transpose(0)
