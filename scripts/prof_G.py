"""Short driver for ncu captures: `reps` applications of G at N^3 (U(-1,1) input)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

from paper_1603_08893_b200 import abi  # noqa: E402

N = int(sys.argv[1]) if len(sys.argv) > 1 else 512
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 2
with abi.Context((N, N, N), 3) as ctx:
    f = ctx.field(9)
    torch.as_tensor(f, device="cuda").uniform_(-1, 1)
    torch.cuda.synchronize()
    out = f if N >= 1024 else ctx.field(9)
    for _ in range(reps):
        ctx.projection(f, out=out)
    ctx.sync()
print("ok")
