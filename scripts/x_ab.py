"""A/B of the long-line x-pass variants (FM_XDIRECT: 0 staged k_x_fast4,
1 k_x_direct, 2 k_x_stream TW 8, 3 k_x_stream TW 4): per-pass CUDA-event
times of G at N^3 (U(-1,1) input, seed-free torch RNG with a fixed seed) and
a digest of the output, one JSON line per variant.  Variants 0, 2 and 3 run
the same plain N-point transform and must agree bit for bit."""
import hashlib
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def child(N, reps):
    sys.path.insert(0, ROOT)
    import torch
    from paper_1603_08893_b200 import abi
    hbm = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
        if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6550.1
    n = N ** 3
    with abi.Context((N, N, N), 3) as ctx:
        f = ctx.field(9)
        g = torch.Generator(device="cuda")
        g.manual_seed(1234)
        v = torch.as_tensor(f, device="cuda")
        v.uniform_(-1, 1, generator=g)
        torch.cuda.synchronize()
        out = ctx.field(9)
        ctx.projection(f, out=out)
        ctx.sync()
        ctx.profile(True)
        for _ in range(reps):
            ctx.projection(f, out=out)
        ms, calls = ctx.profile_read()
        ctx.profile(False)
        o = torch.as_tensor(out, device="cuda")
        dig = hashlib.sha1(o.cpu().numpy().tobytes()).hexdigest()[:16]
        per = [m / calls for m in ms]
        print(json.dumps({"N": N, "mode": os.environ.get("FM_XDIRECT"), "passes_ms": [round(x, 4) for x in per],
                          "x_ms": round(per[2], 4), "x_frac": round(144 * n / (per[2] * 1e-3) / 1e9 / hbm, 3),
                          "G_ms": round(sum(per), 4), "G_frac": round(720 * n / (sum(per) * 1e-3) / 1e9 / hbm, 3),
                          "digest": dig, "kernels": ctx.kernel_names}), flush=True)


if __name__ == "__main__":
    if sys.argv[1] == "child":
        child(int(sys.argv[2]), int(sys.argv[3]))
        sys.exit(0)
    N = int(sys.argv[1])
    modes = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "3"]
    for m in modes:
        env = dict(os.environ, FM_XDIRECT=m)
        r = subprocess.run([sys.executable, __file__, "child", str(N), "10"], env=env, capture_output=True, text=True,
                           timeout=600)
        print(r.stdout.strip() or json.dumps({"mode": m, "rc": r.returncode, "err": r.stderr[-800:]}), flush=True)
